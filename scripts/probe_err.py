import os, sys, json
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2504_21440_b200 as q
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
n = int(sys.argv[1])
r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, n, per_traj=(sys.argv[2] == '1'))
print(n, r["n_ok"], r["kernel_ms"], flush=True)
