"""Dev probe: TFIM-10 mesolve + standalone SpMV timing on the device (operators from the oracle)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import csr_from_oracle, e_ops_csr, rho0_vec, normwise_rel

nspin = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t0 = time.time()
m = O.Model("ising", nspin, 1, 1.0, 0.2, 1.0, 1)
Lc = csr_from_oracle(m, O.L_CONST)
print("build", time.time() - t0, "n", Lc.n_rows, "nnz", Lc.nnz, flush=True)
ctx = q.Context(0)
gen = q.Generator([ctx.op(Lc)])
n, nnz = Lc.n_rows, Lc.nnz
y = torch.randn(n, dtype=torch.complex128, device="cuda")
o = torch.empty_like(y)
res = {}
ms = q.generator_apply_timed(ctx, gen, y, o, reps=20)
b = 20 * nnz + 4 * (n + 1) + 32 * n
res["spmv_sell32"] = (ms, b / ms / 1e6)
print(json.dumps(res), flush=True)
tl = np.linspace(0, 10, 100)
rho0 = rho0_vec(m)
eops = e_ops_csr(m)
for lanes in (1,):
    for grid in (74, 148):
        os.environ["QSG_GRID"] = str(grid)
        r = q.mesolve(ctx, gen, m.dim, rho0, tl, eops)
        batt = 6 * (20 * nnz + 4 * (n + 1)) + 47 * 16 * n
        per = r["kernel_ms"] / r["attempts"]
        print(json.dumps({"lanes": lanes, "grid": grid, "kernel_ms": r["kernel_ms"], "attempts": r["attempts"],
                          "stats": r["stats"], "ms_per_attempt": per, "GBps_model47": batt / per / 1e6,
                          "ctas": r["grid_ctas"], "ex_last": [complex(x) for x in r["expect"][:, -1]]}, default=str), flush=True)
if nspin <= 6:
    ex, st, _ = m.mesolve(tl)
    print("parity", normwise_rel(r["expect"], ex), st)
