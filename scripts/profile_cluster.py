"""ncu target: one cluster-resident (K-cluster) Kerr mesolve, N from argv (default 50)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ctx = q.Context(0)
m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
tl = np.linspace(0.0, 10.0, 101)
for _ in range(2):
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
print(N, r["kernel_ms"], r["attempts"], r["kernel_ms"] * 1e3 / r["attempts"], r.get("engine"))
