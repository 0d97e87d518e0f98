"""Dev: TFIM-14 mcsolve traj/s by batch layout and trajectory count."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
for nt in [int(x) for x in sys.argv[1].split(",")]:
    for mode in sys.argv[2].split(","):
        os.environ["QSG_BATCH_MODE"] = mode
        r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, nt, per_traj=False)
        print(json.dumps({"ntraj": nt, "mode": mode, "s": r["kernel_ms"] / 1e3, "traj_per_s": nt / r["kernel_ms"] * 1e3,
                          "grid": r["grid_ctas"], "mean": round(float((r["block_sum"][0, -1] / r["n_ok"]).real), 9)}), flush=True)
