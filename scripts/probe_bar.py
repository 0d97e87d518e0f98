"""Dev: TFIM-10 / Kerr solves against the instrumented library (_instr/lib) to read barrier ns."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
q.LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "_instr", "lib", "libqsim_b200.so")
ctx = q.Context(0)
for name, prm in (("ising", (10, 1, 1.0, 0.2, 1.0, 1)), ("kerr", (400, 1.0, 0.01, 2.0, 1.0))):
    m = q.Model(name, *prm)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    tl = np.linspace(0, 10, 100)
    q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    print(name, "solve_ms", r["kernel_ms"], "attempts", r["attempts"], flush=True)
