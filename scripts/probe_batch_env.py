"""Dev probe: interleaved A/B of batch-engine environment switches (VAR=a,b ...) on TFIM-14
mcsolve (2,368 trajectories, Sz_total) and the 256-point coupled-Kerr sweep (configs[4])."""
import itertools, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402
axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[1:]]
combos = list(itertools.product(*[v for _, v in axes]))
ctx = q.Context(0)
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
tl = np.linspace(0, 10, 100)
mk = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
ops = [ctx.op(mk.export(q.SEL_L_CONST))] + [ctx.op(mk.export(q.SEL_L_TERM, k)) for k in range(mk.n_terms)]
gk = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0), (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
ek = [mk.export(q.SEL_E_OP, k) for k in range(mk.n_eops)]
pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
rho0 = np.zeros(mk.dim * mk.dim, complex); rho0[0] = 1.0
tk = np.linspace(0.0, 10.0, 101)
ref = {}
for rep in range(2):
    for combo in combos:
        env = dict(zip([a for a, _ in axes], combo))
        os.environ.update(env)
        r = q.mcsolve(ctx, G, cops, [m.export(q.SEL_E_OP, 2)], m.dim, m.psi0(), tl, 2025, 0, 2368)
        mean = r["block_sum"][0] / r["n_ok"]
        ref.setdefault("mc", mean)
        s = q.mesolve_batch(ctx, gk, mk.dim, rho0, tk, ek, pts)
        ex = np.asarray(s["expect"])
        ref.setdefault("sw", ex)
        print(json.dumps({"env": env, "mc_traj_per_s": round(2368 / r["kernel_ms"] * 1e3, 1),
                          "mc_maxdiff": float(np.max(np.abs(mean - ref["mc"]))), "sweep_ms": round(s["kernel_ms"], 2),
                          "sweep_maxdiff": float(np.max(np.abs(ex - ref["sw"])))}), flush=True)
