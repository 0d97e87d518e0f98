"""Small invocations of every device kernel, for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): the grid DP5 engine on the plain, dictionary-coded and key-aligned
stores (TMA ring), the store builders, device Liouvillian assembly, the batch engine in its
per-CTA, grid-wide and cluster layouts (mcsolve + device ensemble sums, and a sweep), and the SDE
kernel. Sizes are tiny so the instrumented run stays short; results are checked loosely (the
sanitizer report is the product here)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_21440_b200 as q  # noqa: E402


def rho0(m):
    p = m.psi0()
    return np.outer(p, p.conj()).reshape(-1, order="F").copy()


ctx = q.Context(0)
t = np.linspace(0.0, 1.0, 6)

# grid engine, plain store (Kerr N=8)
m = q.Model("kerr", 8, 1.0, 0.01, 2.0, 1.0)
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
r = q.mesolve(ctx, q.Generator([ctx.op(m.export(q.SEL_L_CONST))]), m.dim, rho0(m), t, eops)
print("grid plain", r["stats"], flush=True)

# dictionary-coded store (built for any size) and the key-aligned store with the TMA ring
os.environ["QSG_COMPRESS_MIN_BYTES"] = "0"
os.environ["QSG_KA_STORE"] = "1"
m = q.Model("ising", 4, 1, 1.0, 0.2, 1.0, 1)
H = m.export(q.SEL_H_CONST)
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
op = ctx.liouvillian(H, cops)  # device Liouvillian assembly + stores
print("stores", q.op_store_info(op), flush=True)
g = q.Generator([op])
r1 = q.mesolve(ctx, g, m.dim, rho0(m), t, eops)
os.environ["QSG_KA_SOLVE"] = "1"
r2 = q.mesolve(ctx, g, m.dim, rho0(m), t, eops)
del os.environ["QSG_KA_SOLVE"], os.environ["QSG_KA_STORE"], os.environ["QSG_COMPRESS_MIN_BYTES"]
print("grid coded/ka", r1["stats"], r2["stats"], r1.get("store"), r2.get("store"),
      float(np.max(np.abs(r1["expect"] - r2["expect"]))), flush=True)

# batch engine: mcsolve (device ensemble sums with ranges) in three layouts, and a sweep
m = q.Model("ising", 4, 1, 1.0, 0.2, 1.0, 1)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
for mode in ("local1", "grid", "cluster1"):
    os.environ["QSG_BATCH_MODE"] = mode
    rr = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), t, 7, 0, 8, ranges=[(0, 4), (4, 8)])
    print("mcsolve", mode, rr["n_ok"], flush=True)
del os.environ["QSG_BATCH_MODE"]
mk = q.Model("coupled_kerr", 3, 0.1, 0.5, 1.0)
ops = [ctx.op(mk.export(q.SEL_L_CONST))] + [ctx.op(mk.export(q.SEL_L_TERM, k)) for k in range(mk.n_terms)]
gk = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0), (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
r0 = np.zeros(mk.dim * mk.dim, complex)
r0[0] = 1.0
rs = q.mesolve_batch(ctx, gk, mk.dim, r0, t, [mk.export(q.SEL_E_OP, 0)], np.array([[0.5, 0.3], [-1.0, 0.8]]))
print("sweep", rs["status"].tolist(), flush=True)

# stochastic (SSE) kernel
ms = q.Model("jc_sse", 4, 1.0, 1.0, 0.1, 0.3)
rsse = ms.ssesolve(t, 3, 4, dt_max=1e-2)
print("sse ok", flush=True)
ctx.close()
print("sanitize cases done")
