"""Dev probe: TFIM-14 mcsolve through the batch engine with the generator read from its
key-aligned store (ka_row_slot) vs the plain SELL store, interleaved; same trajectories, so the
means must agree to rounding."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q  # noqa: E402

ntraj = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
os.environ["QSG_KA_STORE"] = "1"
m = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
ctx = q.Context(0)
op = ctx.op(m.export(q.SEL_MC_GEN))
print(json.dumps(q.op_store_info(op)), flush=True)
G = q.Generator([op])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, 2)]
tl = np.linspace(0, 10, 100)
q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, 64, per_traj=False)
for rep in range(2):
    for ka in ("1", "0"):
        os.environ["QSG_BATCH_KA"] = ka
        r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), tl, 2025, 0, ntraj, per_traj=False)
        print(json.dumps({"ka": ka, "kernel_ms": r["kernel_ms"], "traj_per_s": ntraj / r["kernel_ms"] * 1e3,
                          "attempts": r["attempts"], "n_ok": r["n_ok"],
                          "mean_last": str(complex(r["block_sum"][0, -1] / r["n_ok"]))}), flush=True)
