"""Dev: A/B of the batch engine's per-buffer L2 eviction priorities (QSG_L2HINT=0|1) on TFIM-14
mcsolve and the configs[4] 256-point coupled-Kerr sweep, interleaved to cancel drift."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
ctx = q.Context(0)
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
mk = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
ops = [ctx.op(mk.export(q.SEL_L_CONST))] + [ctx.op(mk.export(q.SEL_L_TERM, k)) for k in range(mk.n_terms)]
g = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0),
                      (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
keops = [mk.export(q.SEL_E_OP, k) for k in range(mk.n_eops)]
pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
rho0 = np.zeros(mk.dim * mk.dim, complex); rho0[0] = 1.0
tlk = np.linspace(0.0, 10.0, 101)
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
ref = {}
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    for hint in ("0", "1"):
        os.environ["QSG_L2HINT"] = hint
        r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, nt, per_traj=False)
        mean = (r["block_sum"][0] / r["n_ok"])
        rs = q.mesolve_batch(ctx, g, mk.dim, rho0, tlk, keops, pts)
        ex = np.asarray(rs["expect"])
        ref.setdefault("mc", mean); ref.setdefault("sw", ex)
        print(json.dumps({"hint": hint, "mc_traj_per_s": nt / r["kernel_ms"] * 1e3,
                          "mc_maxdiff": float(np.max(np.abs(mean - ref["mc"]))),
                          "sweep_ms": rs["kernel_ms"], "sweep_maxdiff": float(np.max(np.abs(ex - ref["sw"])))}), flush=True)
