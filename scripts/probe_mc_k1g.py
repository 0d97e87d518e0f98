"""Dev probe: TFIM-14 mcsolve (default layout) with the stage-2 identity (QSG_K1G=1) vs the
two-vector stage-2 gather (QSG_K1G=0), interleaved; and the 256-point sweep."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ntraj = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
mk = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
ops = [ctx.op(mk.export(q.SEL_L_CONST))] + [ctx.op(mk.export(q.SEL_L_TERM, k)) for k in range(mk.n_terms)]
gk = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0), (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
ek = [mk.export(q.SEL_E_OP, k) for k in range(mk.n_eops)]
pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
r0 = np.zeros(mk.dim * mk.dim, complex); r0[0] = 1.0
tk = np.linspace(0.0, 10.0, 101)
q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, 64, per_traj=False)
for rep in range(2):
    for kg in ("1", "0"):
        os.environ["QSG_K1G"] = kg
        r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, ntraj, per_traj=False)
        s = q.mesolve_batch(ctx, gk, mk.dim, r0, tk, ek, pts)
        print(json.dumps({"k1g": kg, "mc_traj_per_s": ntraj / r["kernel_ms"] * 1e3, "mc_attempts": r["attempts"],
                          "mean_last": str(complex(r["block_sum"][0, -1] / r["n_ok"])),
                          "sweep_ms": s["kernel_ms"], "sweep_attempts": s["attempts"]}), flush=True)
