"""Profiling driver: one TFIM-10 mesolve solve (the bench headline kernel) — run under ncu."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
nspin = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = q.Model("ising", nspin, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
gen = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
r = q.mesolve(ctx, gen, m.dim, rho0, np.linspace(0, 10, 100), eops)
print("kernel_ms", r["kernel_ms"], "attempts", r["attempts"], "stats", r["stats"])
