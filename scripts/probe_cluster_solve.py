"""Dev probe: the cluster-resident solver (K-cluster, QSG_CLUSTER_SOLVE=1) vs the default grid
engine on small Kerr systems (configs[0], configs[3]) and a small TFIM; agreement and per-attempt time."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
cases = [("kerr", (N, 1.0, 0.01, 2.0, 1.0)) for N in (10, 20, 35, 50, 70, 100)] + [("ising", (5, 1, 1.0, 0.2, 1.0, 1)), ("ising", (6, 1, 1.0, 0.2, 1.0, 1))]
for name, prm in cases:
    m = q.Model(name, *prm)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    res = {}
    for rep in range(2):
        for mode in ("0", "1"):
            os.environ["QSG_CLUSTER_SOLVE"] = mode
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            res[mode] = r
            print(json.dumps({"case": f"{name}{prm[:2]}", "n": m.dim ** 2, "cluster_solve": mode, "ctas": r["grid_ctas"],
                              "ms": r["kernel_ms"], "attempts": r["attempts"],
                              "us_per_attempt": r["kernel_ms"] * 1e3 / r["attempts"], "stats": r["stats"]}), flush=True)
    a, b = res["0"]["expect"], res["1"]["expect"]
    print(json.dumps({"case": f"{name}{prm[:2]}", "max_rel_diff": float(np.max(np.abs(a - b)) / np.max(np.abs(a)))}), flush=True)
