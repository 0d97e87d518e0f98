"""Dev: grid-barrier wait of the TFIM-10 solve, from a library built with -DQSG_BAR_TIMING
(QSG_LIB_PATH=<that lib>): total ns CTAs spent in grid barriers / (CTAs x solve time)."""
import ctypes as C
import numpy as np
import paper_2504_21440_b200 as q

ctx = q.Context(0)
L = q.lib()
L.qsg_debug_barrier_ns.argtypes = [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong), C.c_int, C.c_void_p]
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
op = ctx.liouvillian(m.export(q.SEL_H_CONST), [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)])
g = q.Generator([op])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
tl = np.linspace(0, 10, 100)
q.mesolve(ctx, g, m.dim, rho0, tl, eops)
w, c = C.c_ulonglong(0), C.c_ulonglong(0)
L.qsg_debug_barrier_ns(C.byref(w), C.byref(c), 1, None)
r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
per = np.zeros(1024, np.uint64)
L.qsg_debug_barrier_ns(C.byref(w), C.byref(c), 0, per.ctypes.data)
G = r["grid_ctas"]
print(f"solve {r['kernel_ms']:.2f} ms, {r['attempts']} attempts, {c.value / G:.0f} barriers per CTA, "
      f"mean wait per CTA {w.value / G / 1e6:.2f} ms ({100 * w.value / G / 1e6 / r['kernel_ms']:.1f}% of the solve), "
      f"{w.value / c.value / 1e3:.2f} us per barrier")
pc = per[:G].astype(float) / 1e6
order = np.argsort(pc)
print("per-CTA barrier wait ms: min %.2f (CTA %d) p10 %.2f median %.2f p90 %.2f max %.2f" %
      (pc.min(), order[0], np.percentile(pc, 10), np.median(pc), np.percentile(pc, 90), pc.max()))
print("10 least-waiting (slowest) CTAs:", order[:10].tolist(), np.round(pc[order[:10]], 2).tolist())
print("waits by CTA parity (even/odd):", round(pc[0::2].mean(), 2), round(pc[1::2].mean(), 2))
print("waits by CTA range quarters:", [round(pc[i * G // 4:(i + 1) * G // 4].mean(), 2) for i in range(4)])
