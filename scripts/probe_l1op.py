"""Dev: plain-store entry loads through L1 (__ldg) vs L1::no_allocate: Kerr cutoff solves
(configs[3]), TFIM-10 plain-store solve and SpMV. argv[1] = optional library path."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_21440_b200 as q
if len(sys.argv) > 1:
    q.LIB_PATH = os.path.abspath(sys.argv[1])
ctx = q.Context(0)
out = {"lib": sys.argv[1] if len(sys.argv) > 1 else "default"}
tl = np.linspace(0.0, 10.0, 101)
for N in (50, 100, 200, 400):
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    ms = [q.mesolve(ctx, g, m.dim, rho0, tl, eops)["kernel_ms"] for _ in range(4)]
    out[f"kerr{N}_ms"] = round(min(ms[1:]), 3)
os.environ["QSG_NO_COMPRESS"] = "1"
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
H = m.export(q.SEL_H_CONST)
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
op = ctx.liouvillian(H, cops)
g = q.Generator([op])
t = np.linspace(0, 10, 100)
ms = [q.mesolve(ctx, g, m.dim, rho0, t, eops)["kernel_ms"] for _ in range(3)]
out["tfim10_plain_ms"] = round(min(ms[1:]), 3)
y = torch.randn(m.dim * m.dim, dtype=torch.complex128, device="cuda")
o = torch.empty_like(y)
out["tfim10_spmv_ms"] = round(q.generator_apply_timed(ctx, g, y, o, reps=20), 4)
print(json.dumps(out), flush=True)
