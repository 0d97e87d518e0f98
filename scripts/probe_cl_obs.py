"""Dev probe: K-cluster Kerr mesolve per-attempt time with and without observations
(e_ops / dense tlist), to split the observation cost from the stage passes and controller."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
ctx = q.Context(0)
for N in [int(x) for x in sys.argv[1:]] or [20, 50, 100]:
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    for name, tl, eo in (("full", np.linspace(0.0, 10.0, 101), eops), ("no_eops", np.linspace(0.0, 10.0, 101), []),
                         ("2pts", np.array([0.0, 10.0]), eops), ("2pts_no_eops", np.array([0.0, 10.0]), [])):
        for rep in range(3):
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eo)
        print(json.dumps({"N": N, "case": name, "us_per_attempt": round(r["kernel_ms"] * 1e3 / r["attempts"], 3),
                          "attempts": r["attempts"], "engine": r.get("engine")}), flush=True)
