"""Dev: configs[4] 256-point coupled-Kerr mesolve sweep under each batch layout (QSG_BATCH_MODE)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
m = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
ops = [ctx.op(m.export(q.SEL_L_CONST))] + [ctx.op(m.export(q.SEL_L_TERM, k)) for k in range(m.n_terms)]
g = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0),
                      (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
rho0 = np.zeros(m.dim * m.dim, complex); rho0[0] = 1.0
tl = np.linspace(0.0, 10.0, 101)
ref = None
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["local1", "local2", "local4", "local", "grid", "cluster1"]
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 256
pts = pts[:npts]
for mode in modes:
    if mode == "auto":
        os.environ.pop("QSG_BATCH_MODE", None)
    else:
        os.environ["QSG_BATCH_MODE"] = mode
    q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, pts[:2])
    best = 1e9
    for _ in range(2):
        r = q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, pts)
        best = min(best, r["kernel_ms"])
    ex = np.asarray(r["expect"])
    if ref is None: ref = ex
    print(json.dumps({"mode": mode, "ms": best, "npts": len(pts), "pts_per_s": len(pts) / best * 1e3, "attempts": r["attempts"],
                      "maxdiff": float(np.max(np.abs(ex - ref)))}), flush=True)
