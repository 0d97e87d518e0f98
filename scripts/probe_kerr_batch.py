"""Dev: single Kerr-cutoff mesolve (configs[3]) on the grid engine vs one point of the batched
engine in a thread-block cluster (QSG_BATCH_MODE=cluster1, QSG_CLUSTER=c)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in (50, 100, 200, 400):
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0(); rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
    out = {"N": N, "grid_ms": r["kernel_ms"], "grid_att": r["attempts"]}
    for c in (8, 16):
        os.environ["QSG_BATCH_MODE"] = "cluster1"; os.environ["QSG_CLUSTER"] = str(c)
        q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, np.zeros((1, 1)))
        b = q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, np.zeros((1, 1)))
        out[f"cl{c}_ms"] = b["kernel_ms"]; out[f"cl{c}_att"] = b["attempts"]
        out[f"cl{c}_diff"] = float(np.max(np.abs(b["expect"][0] - r["expect"])) / np.max(np.abs(r["expect"])))
    os.environ.pop("QSG_BATCH_MODE"); os.environ.pop("QSG_CLUSTER")
    print(json.dumps(out), flush=True)
