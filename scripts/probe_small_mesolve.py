"""Dev: configs[3] Kerr cutoff solves on the grid engine (q.mesolve) against the batch engine
running the same solve as a one-point batch (q.mesolve_batch) under each batch layout."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "50,100,200,400").split(",")]:
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    ref = np.asarray(r["expect"])
    out = {"N": N, "grid_ms": r["kernel_ms"], "grid_attempts": r["attempts"]}
    for mode in ("local1", "cluster1"):
        for cs in ((1,) if mode == "local1" else (4, 8, 16)):
            os.environ["QSG_BATCH_MODE"] = mode
            os.environ["QSG_CLUSTER"] = str(cs)
            rb = q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, np.zeros((1, 1)))
            rb = q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, np.zeros((1, 1)))
            ex = rb["expect"][0]
            out[f"{mode}_{cs}"] = {"ms": rb["kernel_ms"], "attempts": int(rb["attempts"]),
                                   "maxrel": float(np.max(np.abs(ex - ref)) / np.max(np.abs(ref)))}
    print(json.dumps(out), flush=True)
