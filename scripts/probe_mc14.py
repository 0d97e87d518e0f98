"""Dev probe: TFIM-14 mcsolve throughput on one GPU (product model builder)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q

nspin = int(sys.argv[1]) if len(sys.argv) > 1 else 14
ntraj = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
t0 = time.time()
m = q.Model("ising", nspin, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]  # Sz_total
print("build", time.time() - t0, flush=True)
tl = np.linspace(0, 10, 100)
for nt in (64, ntraj):
    r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, nt, per_traj=True)
    nj = np.array([len(j) for j in r["jumps"]])
    att = r["attempts"]
    n = m.dim
    bytes_att = 47 * 16 * n
    print(json.dumps({"ntraj": nt, "kernel_ms": r["kernel_ms"], "traj_per_s": nt / r["kernel_ms"] * 1e3,
                      "attempts": att, "attempts_per_traj": att / nt, "jumps_per_traj": float(nj.mean()),
                      "n_ok": r["n_ok"], "grid": r["grid_ctas"], "GBps_model47": bytes_att * att / r["kernel_ms"] / 1e6,
                      "mean_last": complex(r["block_sum"][0, -1] / r["n_ok"])}, default=str), flush=True)
