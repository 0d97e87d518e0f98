"""Dev: operator-store build time (plain vs coded) and TFIM-10 solve time."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
L = m.export(q.SEL_L_CONST)
ctx = q.Context(0)
for nc in ("1", "0"):
    os.environ["QSG_NO_COMPRESS"] = nc
    t0 = time.perf_counter(); op = ctx.op(L); dt = time.perf_counter() - t0
    t0 = time.perf_counter(); op2 = ctx.op(L); dt2 = time.perf_counter() - t0
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    r = q.mesolve(ctx, q.Generator([op2]), m.dim, rho0, np.linspace(0, 10, 100), eops)
    print(json.dumps({"no_compress": nc, "op_create_s": dt, "op_create_s_2": dt2, "storage": q.op_storage(op2),
                      "solve_ms": r["kernel_ms"], "ex_last": str(r["expect"][:, -1])}), flush=True)
