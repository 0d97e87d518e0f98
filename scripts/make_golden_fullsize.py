"""Freeze full-size oracle solves as golden fixtures (tests/golden/fullsize_golden.json).

These are the BASELINE.json configurations whose oracle solves are too slow to rerun inside the
GPU test pass (the GPU box has no /root/reference and the tests must finish in minutes):
  * configs[1]: TFIM-10 mesolve, the complete t in [0, 10] solve (81 DP5 attempts);
  * configs[3]: Kerr resonator cutoffs N = 150, 300, 400 (full solves).
The oracle runs with worker threads (orc_set_threads); its results are bit-identical to the
1-thread restatement (tests/test_oracle_pinning.py::test_oracle_threads_bitwise), which is what
the reference's single-threaded mesolve computes.

Usage: python scripts/make_golden_fullsize.py [case ...]   (default: every case)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

PATH = os.path.join(ROOT, "tests", "golden", "fullsize_golden.json")
CASES = {
    "tfim10": ("ising", [10, 1, 1.0, 0.2, 1.0, 1], np.linspace(0.0, 10.0, 100)),
    "kerr150": ("kerr", [150, 1.0, 0.01, 2.0, 1.0], np.linspace(0.0, 10.0, 101)),
    "kerr300": ("kerr", [300, 1.0, 0.01, 2.0, 1.0], np.linspace(0.0, 10.0, 101)),
    "kerr400": ("kerr", [400, 1.0, 0.01, 2.0, 1.0], np.linspace(0.0, 10.0, 101)),
}


def main(names):
    out = json.load(open(PATH)) if os.path.exists(PATH) else {}
    O.set_threads(os.cpu_count() or 1)
    for key in names:
        name, params, tl = CASES[key]
        m = O.Model(name, *params)
        t0 = time.perf_counter()
        m.prepare_liouvillian()
        t1 = time.perf_counter()
        ex, st = m.mesolve_prepared(tl)
        t2 = time.perf_counter()
        out[key] = {"model": name, "params": params, "tlist": tl.tolist(), "stats": list(map(int, st)),
                    "expect_re": ex.real.tolist(), "expect_im": ex.imag.tolist(),
                    "oracle_threads": O.threads(), "build_s": t1 - t0, "solve_s": t2 - t1}
        print(key, st, f"build {t1 - t0:.1f} s, solve {t2 - t1:.1f} s", flush=True)
        with open(PATH, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
