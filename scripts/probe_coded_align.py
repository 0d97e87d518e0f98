"""Dev probe: TFIM-10 mesolve (configs[1]) and the TFIM-10 coded SpMV with the coded store's
entries in CSR order (QSG_SELL_ALIGN=0) vs slice-aligned order (default), same process."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2504_21440_b200 as q  # noqa: E402
ctx = q.Context(0)
m = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
L = m.export(q.SEL_L_CONST)
gens = {}
for mode in ("0", "1"):
    os.environ["QSG_SELL_ALIGN"] = mode
    gens[mode] = q.Generator([ctx.op(L)])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
tl = np.linspace(0.0, 10.0, 100)
n = m.dim * m.dim
y = torch.randn(n, dtype=torch.complex128, device="cuda")
out = {}
for rep in range(3):
    for mode, g in gens.items():
        r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
        o = torch.empty_like(y)
        sp = q.generator_apply_timed(ctx, g, y, o, reps=20)
        out[mode] = (r, o.clone())
        if rep:
            print(json.dumps({"align": mode, "solve_ms": round(r["kernel_ms"], 3), "spmv_us": round(sp * 1e3, 2),
                              "stats": r["stats"]}), flush=True)
ea, eb = out["0"][0]["expect"], out["1"][0]["expect"]
print(json.dumps({"expect_max_rel": float(np.max(np.abs(ea - eb)) / np.max(np.abs(ea))),
                  "spmv_max_rel": float((out["0"][1] - out["1"][1]).abs().max() / out["0"][1].abs().max())}))
