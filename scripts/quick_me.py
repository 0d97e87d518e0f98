"""Dev: time TFIM-N mesolve solves (product builder) — kernel ms, attempts, achieved GB/s."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
nspin = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = q.Model("ising", nspin, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
L = m.export(q.SEL_L_CONST)
gen = q.Generator([ctx.op(L)])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
n, nnz = L.n_rows, L.nnz
grids = [int(g) for g in os.environ.get("GRIDS", "0").split(",")]
for g in grids:
    if g: os.environ["QSG_GRID"] = str(g)
    best = 1e9
    for _ in range(3):
        r = q.mesolve(ctx, gen, m.dim, rho0, np.linspace(0, 10, 100), eops)
        best = min(best, r["kernel_ms"])
    b = (6 * (20 * nnz + 4 * (n + 1)) + 47 * 16 * n) * r["attempts"]
    print(json.dumps({"nspin": nspin, "grid": r["grid_ctas"], "ms": best, "attempts": r["attempts"],
                      "GBps": b / best / 1e6, "stats": r["stats"], "ex_last": str(r["expect"][:, -1])}), flush=True)
