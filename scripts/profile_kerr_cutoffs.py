"""Profiling driver (configs[3]): one Kerr mesolve per cutoff N = 50..400 (one dp5_grid_kernel
launch each) — run under ncu with dram__bytes and lts__t_bytes to measure the L2-resident traffic."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402

ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in (50, 100, 150, 200, 300, 400):
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    print(N, r["kernel_ms"], r["attempts"], flush=True)
