"""Dev probe: Kerr N=20/50/100 mesolve per-attempt time vs grid size (QSG_GRID) and cluster mode."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in (20, 50, 100):
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    for cl in ("0", "1"):
        for G in (1, 2, 4, 8, 16, 32):
            os.environ["QSG_GRID_CLUSTER"] = cl
            os.environ["QSG_GRID"] = str(G)
            os.environ["QSG_GRID_CLUSTER_SIZE"] = str(G)
            if cl == "1" and G > 16: continue
            q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            print(json.dumps({"N": N, "cluster": cl, "G": r["grid_ctas"], "us_per_attempt": r["kernel_ms"] * 1e3 / r["attempts"]}), flush=True)
