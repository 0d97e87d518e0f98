"""Dev: TFIM-10 mesolve kernel time for a grid-engine CTA-size variant library (argv[1] = path to a
libqsim_b200.so built with -DQSG_GRID_THREADS/-DQSG_GRID_MINB; default = the in-tree library)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
if len(sys.argv) > 1:
    q.LIB_PATH = os.path.abspath(sys.argv[1])
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
H = m.export(q.SEL_H_CONST)
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
ctx = q.Context(0)
op = ctx.liouvillian(H, cops)
g = q.Generator([op])
t = np.linspace(0, 10, 100)
ms = []
for it in range(6):
    r = q.mesolve(ctx, g, m.dim, rho0, t, eops)
    ms.append(r["kernel_ms"])
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "default", "kernel_ms": ms[1:],
                  "Sz_end": float(np.asarray(r["expect"])[2, -1].real)}), flush=True)
