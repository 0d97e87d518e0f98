"""Dev probe: TFIM-20 sesolve (bench secondary) with the full tlist / e_ops and without
observations, to size the observation cost of the grid engine's sesolve mode."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
ctx = q.Context(0)
m = q.Model("ising", 20, 1, 1.0, 0.2, 0.0, 1)  # as bench.py sesolve_tfim20
g = q.Generator([ctx.op(m.export(q.SEL_SE_GEN))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
for name, tl, eo in (("full", np.linspace(0.0, 10.0, 100), eops), ("2pts", np.array([0.0, 10.0]), eops),
                     ("full_no_eops", np.linspace(0.0, 10.0, 100), [])):
    for rep in range(2):
        r = q.sesolve(ctx, g, m.dim, psi, tl, eo)
    print(json.dumps({"case": name, "ms": round(r["kernel_ms"], 2), "attempts": r["attempts"],
                      "us_per_attempt": round(r["kernel_ms"] * 1e3 / r["attempts"], 1)}), flush=True)
