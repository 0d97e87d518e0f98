"""Dev: two Kerr N=400 mesolve solves on the grid engine (for an ncu capture of the second)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
m = q.Model("kerr", 400, 1.0, 0.01, 2.0, 1.0)
g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
for _ in range(2):
    r = q.mesolve(ctx, g, m.dim, rho0, np.linspace(0.0, 10.0, 101), eops)
print("kernel_ms", r["kernel_ms"])
