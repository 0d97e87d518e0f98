"""Generate tests/golden/oracle_golden.json from the CPU oracle (the reference itself cannot be
built here — Eigen3 is absent — so golden vectors are frozen oracle outputs; the oracle is
pinned separately against published RNG vectors and the reference's analytic tests)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

out = {"mesolve": [], "mcsolve": []}
for name, params, tl in [
    ("kerr", [20, 1.0, 0.01, 2.0, 1.0], np.linspace(0, 10, 101)),
    ("ising", [3, 2, 1.0, 0.2, 1.0, 1], np.linspace(0, 10, 100)),
    ("coupled_kerr", [4, 0.1, 0.5, 1.0], np.linspace(0, 10, 101)),
]:
    m = O.Model(name, *params)
    ex, st, _ = m.mesolve(tl)
    out["mesolve"].append({"model": name, "params": params, "tlist": tl.tolist(), "stats": list(map(int, st)),
                           "expect_re": ex.real.tolist(), "expect_im": ex.imag.tolist()})
for name, params, tl, seed, ntraj in [
    ("decay2", [0.25], np.linspace(0, 80, 41), 2025, 64),
    ("jc", [6, 1.0, 1.0, 0.1, 0.05, 0.05], np.linspace(0, 60, 61), 7, 16),
    ("ising", [6, 1, 1.0, 0.2, 1.0, 1], np.linspace(0, 10, 100), 2025, 8),
]:
    m = O.Model(name, *params)
    r = m.mcsolve(tl, seed, ntraj)
    out["mcsolve"].append({"model": name, "params": params, "tlist": tl.tolist(), "seed": seed, "ntraj": ntraj,
                           "jumps": [[list(x) for x in j] for j in r["jumps"]],
                           "mean_re": r["mean"].real.tolist(), "mean_im": r["mean"].imag.tolist(),
                           "stats": r["stats"].tolist()})
os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
with open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json"), "w") as f:
    json.dump(out, f)
print("wrote", sum(len(v) for v in out.values()), "cases")
