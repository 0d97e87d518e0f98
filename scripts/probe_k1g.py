"""Dev probe: TFIM-10 mesolve with stage 2 as k1 + (h a21) G k1 (QSG_K1G=1, no x2 pass) vs the
materialised stage-2 input (QSG_K1G=0), interleaved, against the frozen full-solve golden."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_21440_b200 as q  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_golden.json")))["tfim10"]
ref = np.array(g["expect_re"]) + 1j * np.array(g["expect_im"])
t = np.array(g["tlist"])

m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
H = m.export(q.SEL_H_CONST)
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
op = ctx.liouvillian(H, cops)
print(json.dumps(q.op_store_info(op)), flush=True)
gen = q.Generator([op])
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for rep in range(reps):
    for mode in ("k1g", "x2"):
        os.environ["QSG_K1G"] = "1" if mode == "k1g" else "0"
        r = q.mesolve(ctx, gen, m.dim, rho0, t, eops)
        err = max(np.max(np.abs(a - b)) / np.max(np.abs(b)) for a, b in zip(r["expect"], ref))
        print(json.dumps({"mode": mode, "store": r.get("store"), "kernel_ms": r["kernel_ms"],
                          "attempts": r["attempts"], "stats": r["stats"], "err_vs_golden": err,
                          "golden_stats": g["stats"]}), flush=True)
