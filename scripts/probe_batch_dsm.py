"""Dev probe: TFIM-14 mcsolve, batch layout 7 (state in the cluster's DSMEM) vs the default
one-trajectory-per-CTA layout, interleaved; and a coupled-Kerr sweep."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ntraj = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
for rep in range(2):
    for mode in ("clusterdsm", "local1"):
        os.environ["QSG_BATCH_MODE"] = mode
        r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, ntraj, per_traj=True)
        print(json.dumps({"mode": mode, "kernel_ms": r["kernel_ms"], "traj_per_s": ntraj / r["kernel_ms"] * 1e3,
                          "ctas": r["grid_ctas"], "attempts": r["attempts"], "n_ok": r["n_ok"],
                          "mean_last": str(complex(r["block_sum"][0, -1] / r["n_ok"])),
                          "jumps0": r["jumps"][0][:3]}), flush=True)
