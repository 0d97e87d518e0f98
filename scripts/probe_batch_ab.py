"""Dev: batch-engine A/B between library builds (argv[1] = optional library path): TFIM-14 mcsolve
traj/s (argv[2] trajectories, default 2368) and the configs[4] 256-point coupled-Kerr sweep."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
if len(sys.argv) > 1 and sys.argv[1]:
    q.LIB_PATH = os.path.abspath(sys.argv[1])
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2368
ctx = q.Context(0)
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, 296, per_traj=False)
r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, nt, per_traj=False)
mk = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
ops = [ctx.op(mk.export(q.SEL_L_CONST))] + [ctx.op(mk.export(q.SEL_L_TERM, k)) for k in range(mk.n_terms)]
g = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0),
                      (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
keops = [mk.export(q.SEL_E_OP, k) for k in range(mk.n_eops)]
pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
rho0 = np.zeros(mk.dim * mk.dim, complex); rho0[0] = 1.0
tlk = np.linspace(0.0, 10.0, 101)
q.mesolve_batch(ctx, g, mk.dim, rho0, tlk, keops, pts[:8])
rs = q.mesolve_batch(ctx, g, mk.dim, rho0, tlk, keops, pts)
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "default", "mc_traj_per_s": round(nt / r["kernel_ms"] * 1e3, 1),
                  "mc_mean_end": float((r["block_sum"][0, -1] / r["n_ok"]).real),
                  "sweep_ms": round(rs["kernel_ms"], 2),
                  "sweep_sum": float(np.abs(np.asarray(rs["expect"])).sum())}), flush=True)
