"""Dev probe: interleaved A/B of K-cluster environment switches on Kerr mesolve.
usage: probe_cl_env.py VAR=a,b [VAR2=c,d ...] -- N1 N2 ...   (every combination, 2 timed reps)"""
import itertools, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
args = sys.argv[1:]
k = args.index("--") if "--" in args else len(args)
axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in args[:k]]
Ns = [int(x) for x in args[k + 1:]] or [20, 50, 100]
ctx = q.Context(0)
tl = np.linspace(0.0, 10.0, 101)
combos = list(itertools.product(*[v for _, v in axes]))
for N in Ns:
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    eops = [m.export(q.SEL_E_OP, j) for j in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    ref = None
    for rep in range(3):
        for combo in combos:
            for (name, _), v in zip(axes, combo):
                os.environ[name] = v
            r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
            if ref is None:
                ref = r["expect"]
            if rep:
                print(json.dumps({"N": N, "env": dict(zip([a for a, _ in axes], combo)),
                                  "us_per_attempt": round(r["kernel_ms"] * 1e3 / r["attempts"], 3),
                                  "engine": r.get("engine"), "stats": r["stats"],
                                  "max_abs_diff_vs_first": float(np.max(np.abs(r["expect"] - ref)))}), flush=True)
