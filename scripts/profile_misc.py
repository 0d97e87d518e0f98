"""Profiling driver for ncu: one device Liouvillian assembly (TFIM-10) and one SSE + one SME run (JC N=10)."""
import numpy as np
import paper_2504_21440_b200 as q

ctx = q.Context(0)
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
op = ctx.liouvillian(m.export(q.SEL_H_CONST), [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)])
op.close()
t = np.linspace(0.0, 10.0, 101)
r1 = q.Model("jc_sse", 10, 1.0, 1.0, 0.1, 0.5).ssesolve(t, 5, 2000, dt_max=1e-3)
r2 = q.Model("jc_sme", 10, 1.0, 1.0, 0.1, 0.5, 0.1, 0.05).smesolve(t, 5, 200, n_det=2, dt_max=1e-3)
print("sse_ms", r1["device_ms"], "sme_ms", r2["device_ms"])
