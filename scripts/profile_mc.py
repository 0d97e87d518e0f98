"""Profiling driver: TFIM-14 mcsolve, short tlist (0..2), one full wave of slots — run under ncu."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ntraj = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
r = q.mcsolve(ctx, G, cops, [m.export(q.SEL_E_OP, 2)], m.dim, m.psi0(), np.linspace(0, 2, 21), 2025, 0, ntraj,
              per_traj=False)
print("kernel_ms", r["kernel_ms"], "attempts", r["attempts"], "n_ok", r["n_ok"])
