"""Dev probe: configs[1] TFIM-10 mesolve kernel time (product model builder), 3 timed solves."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
ctx = q.Context(0)
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
tl = np.linspace(0.0, 10.0, 100)
ms = []
for rep in range(4):
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    if rep:
        ms.append(r["kernel_ms"])
print(json.dumps({"lib": os.environ.get("QSG_LIB_PATH", "default"), "ms": [round(x, 3) for x in ms],
                  "stats": r["stats"], "ctas": r["grid_ctas"]}), flush=True)
