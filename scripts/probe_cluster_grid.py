"""Dev probe: Kerr cutoff mesolve (configs[0]/[3]) on the grid engine as a cooperative grid (grid
barrier) vs as one thread-block cluster (hardware cluster barrier), interleaved; per-attempt time
and agreement of the two solves."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402

cutoffs = [int(x) for x in sys.argv[1:]] or [20, 50, 100, 150, 200, 300, 400]
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in cutoffs:
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    res = {}
    for rep in range(2):
        for mode, env in (("grid", "0"), ("cluster16", "1"), ("cluster8", "1")):
            os.environ["QSG_GRID_CLUSTER"] = env
            if mode == "cluster8":
                os.environ["QSG_GRID_CLUSTER_SIZE"] = "8"
            else:
                os.environ.pop("QSG_GRID_CLUSTER_SIZE", None)
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            res[mode] = r
            print(json.dumps({"N": N, "mode": mode, "ms": r["kernel_ms"], "attempts": r["attempts"],
                              "us_per_attempt": r["kernel_ms"] * 1e3 / r["attempts"], "ctas": r["grid_ctas"],
                              "stats": r["stats"]}), flush=True)
    a, b = res["grid"]["expect"], res["cluster16"]["expect"]
    print(json.dumps({"N": N, "max_abs_diff": float(np.max(np.abs(a - b)))}), flush=True)
