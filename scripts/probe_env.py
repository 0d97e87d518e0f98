"""Dev: TFIM-10 mesolve (device-assembled L) under alternating values of one environment switch,
e.g. `python scripts/probe_env.py QSG_CDICT 0,1`: kernel ms and the difference to the first run."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
var, vals = sys.argv[1], sys.argv[2].split(",")
nspin = int(sys.argv[3]) if len(sys.argv) > 3 else 10
m = q.Model("ising", nspin, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
op = ctx.liouvillian(m.export(q.SEL_H_CONST), [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)])
gen = q.Generator([op])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
ref = None
for rep in range(3):
    for v in vals:
        os.environ[var] = v
        r = q.mesolve(ctx, gen, m.dim, rho0, np.linspace(0, 10, 100), eops)
        if ref is None: ref = r["expect"]
        d = float(np.max(np.abs(r["expect"] - ref)) / np.max(np.abs(ref)))
        print(json.dumps({var: v, "ms": r["kernel_ms"], "attempts": r["attempts"], "stats": r["stats"], "diff": d}), flush=True)
