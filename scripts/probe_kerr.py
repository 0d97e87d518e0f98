"""Dev: Kerr cutoff mesolve time vs cooperative grid size."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
tl = np.linspace(0, 10, 101)
for N, grids in ((50, (1, 2, 5, 10, 20, 40)), (200, (10, 20, 40, 80, 148)), (400, (40, 79, 148, 296))):
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    out = {}
    for G in grids:
        os.environ["QSG_GRID"] = str(G)
        q.mesolve(ctx, g, m.dim, rho0, tl, eops)
        r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
        out[G] = round(r["kernel_ms"] * 1e3 / r["attempts"], 1)
    print(json.dumps({"N": N, "us_per_attempt_by_grid": out}), flush=True)
