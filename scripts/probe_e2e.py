"""Phase timing of the end-to-end TFIM-10 path: (a) pinned host L CSR -> op store -> solve; (b) host
H + c_ops -> device Liouvillian assembly (qsg_liouvillian_create) -> solve."""
import time
import numpy as np
import torch
import paper_2504_21440_b200 as q

m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
t0 = time.perf_counter()
H = m.export(q.SEL_H_CONST)
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
print(f"host H + c_ops export {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
t0 = time.perf_counter()
L = m.export(q.SEL_L_CONST)
print(f"host L export {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
ctx = q.Context(0)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
Lh = q.CsrMatrix(pin(L.rowptr), pin(L.col), pin(L.val), L.n_rows, L.n_cols)
rho0_h = pin(rho0)
t = np.linspace(0, 10, 100)
for it in range(6):
    t0 = time.perf_counter()
    op = ctx.op(Lh)
    t1 = time.perf_counter()
    r = q.mesolve(ctx, q.Generator([op]), m.dim, rho0_h, t, eops)
    t2 = time.perf_counter()
    op.close()
    print(f"(a) it {it}: op {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms (kernel {r['kernel_ms']:.1f})", flush=True)
for it in range(6):
    t0 = time.perf_counter()
    op = ctx.liouvillian(H, cops)
    t1 = time.perf_counter()
    r = q.mesolve(ctx, q.Generator([op]), m.dim, rho0_h, t, eops)
    t2 = time.perf_counter()
    op.close()
    print(f"(b) it {it}: assemble+store {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms (kernel {r['kernel_ms']:.1f}) "
          f"total {1e3*(t2-t0):.1f} ms", flush=True)
