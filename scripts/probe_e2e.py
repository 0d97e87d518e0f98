"""Phase timing of the end-to-end TFIM-10 path (pinned host CSR -> op store -> solve -> host)."""
import time
import numpy as np
import torch
import paper_2504_21440_b200 as q

m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
L = m.export(q.SEL_L_CONST)
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
ctx = q.Context(0)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
Lh = q.CsrMatrix(pin(L.rowptr), pin(L.col), pin(L.val), L.n_rows, L.n_cols)
rho0_h = pin(rho0)
t = np.linspace(0, 10, 100)
for it in range(8):
    t0 = time.perf_counter()
    op = ctx.op(Lh)
    t1 = time.perf_counter()
    r = q.mesolve(ctx, q.Generator([op]), m.dim, rho0_h, t, eops)
    t2 = time.perf_counter()
    op.close()
    t3 = time.perf_counter()
    print(f"it {it}: op {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms (kernel {r['kernel_ms']:.1f})  close {1e3*(t3-t2):.1f} ms", flush=True)
