"""Dev probe: K-cluster barrier with a shared-memory-only release (default) vs the full
arrive.release (QSG_CL_FULL_RELEASE=1), interleaved, Kerr mesolve; per-attempt time and agreement.
The switch existed only for this A/B (profiles/r02_cl_release.log) and was removed once the
shared-memory release became the only form: today both modes run the same kernel."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
for N in [int(x) for x in sys.argv[1:]] or [20, 35, 50, 70, 100]:
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    res = {}
    for rep in range(3):
        for mode in ("smem", "full"):
            os.environ["QSG_CL_FULL_RELEASE"] = "1" if mode == "full" else "0"
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            res[mode] = r
            if rep:
                print(json.dumps({"N": N, "mode": mode, "us_per_attempt": r["kernel_ms"] * 1e3 / r["attempts"],
                                  "engine": r.get("engine"), "stats": r["stats"]}), flush=True)
    print(json.dumps({"N": N, "max_abs_diff": float(np.max(np.abs(res["smem"]["expect"] - res["full"]["expect"])))}))
