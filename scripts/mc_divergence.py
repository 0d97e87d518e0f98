"""configs[2] per-trajectory parity audit: TFIM-14 mcsolve trajectories [lo, hi) of seed 2025 on the
device (qsg_mcsolve) against the oracle run_ensemble restatement, jump record by jump record.

For every trajectory whose jump record differs, print the first differing jump (index, device and
oracle times / channels) and the device/oracle step statistics, so the cause can be classified.
Usage: python scripts/mc_divergence.py [lo hi] (default 0 256)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_21440_b200 as q  # noqa: E402
from oracle import oracle as O  # noqa: E402

lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 256)
P = (14, 1, 1.0, 0.2, 1.0, 1)
t = np.linspace(0.0, 10.0, 100)
m = q.Model("ising", *P)
ctx = q.Context(0)
G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
t0 = time.time()
dev = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), t, 2025, lo, hi)
t1 = time.time()
om = O.Model("ising", *P)
# the oracle numbers trajectories from 0: run [0, hi) and keep [lo, hi)
ref = om.mcsolve(t, 2025, hi, n_threads=os.cpu_count())
t2 = time.time()
out = {"range": [lo, hi], "device_s": t1 - t0, "oracle_s": t2 - t1, "diverged": []}
worst = 0.0
for i in range(lo, hi):
    dj, rj = dev["jumps"][i - lo], ref["jumps"][i]
    same = len(dj) == len(rj) and all(a[1] == b[1] and abs(a[0] - b[0]) <= 1e-6 for a, b in zip(dj, rj))
    if not same:
        k = next((j for j, (a, b) in enumerate(zip(dj, rj)) if a[1] != b[1] or abs(a[0] - b[0]) > 1e-6),
                 min(len(dj), len(rj)))
        out["diverged"].append({"traj": i, "first_diff": k, "n_dev": len(dj), "n_ref": len(rj),
                                "dev": dj[max(0, k - 1):k + 2], "ref": rj[max(0, k - 1):k + 2],
                                "dev_stats": dev["stats"][i - lo].tolist(), "ref_stats": ref["stats"][i].tolist()})
        continue
    a = dev["per_traj"][i - lo]
    b = ref["per_traj"][i]
    err = max(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300) for x, y in zip(a, b))
    worst = max(worst, err)
    if len(dj):
        out.setdefault("max_jump_dt", 0.0)
        out["max_jump_dt"] = max(out["max_jump_dt"], max(abs(x[0] - y[0]) for x, y in zip(dj, rj)))
out["matched"] = (hi - lo) - len(out["diverged"])
out["worst_expect_normwise_rel"] = worst
print(json.dumps(out, indent=1))
