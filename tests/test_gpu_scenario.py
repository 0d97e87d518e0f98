"""`qsim run` end to end on the GPU (tools/qsim.cpp:34-102, scenario.cpp:549-719):
the reference's built-in scenarios ising_mc_2x3 and jc_mcsolve (mcsolve on the batch engine) and
jc_mesolve (the grid engine), checked against the oracle; the CSV must be the reference's table in
"%.17g" and the JSON sidecar nlohmann's dump(2) layout (sorted keys, 2-space indent)."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from tests._helpers import normwise_rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QSIM = os.path.join(ROOT, "paper_2504_21440_b200", "bin", "qsim")


def make_tlist(t0, tf, n):
    """scenario.cpp:378-384: t0 + (tf - t0) * i / (n - 1), not numpy's linspace rounding."""
    return np.array([t0 + (tf - t0) * float(i) / (n - 1) for i in range(n)])


def run(name, tmp_path, *extra):
    r = subprocess.run([QSIM, "run", name, "--out-dir", str(tmp_path), *extra], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    csv = (tmp_path / f"{name}.csv").read_text()
    side = (tmp_path / f"{name}.json").read_text()
    return csv, side


def check_format(csv, side, columns):
    lines = csv.splitlines()
    assert lines[0] == ",".join(columns)
    for ln in lines[1:]:
        for tok in ln.split(","):
            assert tok == "%.17g" % float(tok), tok  # scenario.cpp:399-403
    j = json.loads(side)
    # nlohmann dump(2) + "\n": sorted keys, 2-space indent, ": " separators, shortest doubles
    assert side == json.dumps(j, indent=2, sort_keys=True) + "\n"
    return np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]]), j


def test_qsim_run_ising_mc_2x3(tmp_path):
    csv, side = run("ising_mc_2x3", tmp_path)
    tab, j = check_format(csv, side, ["t", "Sz_total_re", "Sz_total_im"])
    assert j["scenario"]["name"] == "ising_mc_2x3" and j["ntraj"] == 200 and j["seed"] == 2025
    assert j["extras"]["completed_trajectories"] == 200 and j["extras"]["failed_trajectories"] == 0
    t = make_tlist(0.0, 10.0, 100)
    ref = O.Model("ising", 2, 3, 1.0, 0.2, 1.0, 1).mcsolve(t, 2025, 200, n_threads=os.cpu_count() or 1)
    assert np.array_equal(tab[:, 0], t)
    assert normwise_rel(tab[:, 1] + 1j * tab[:, 2], ref["mean"][2]) <= 1e-9
    assert j["extras"]["total_jumps"] == sum(len(x) for x in ref["jumps"])
    st = ref["stats"].sum(axis=0)
    assert j["stats"]["steps"] == st[0] and j["stats"]["rejected"] == st[1]


def test_qsim_run_jc_mcsolve_and_overrides(tmp_path):
    """jc_mcsolve with --ntraj / --seed overrides (run_scenario, scenario.cpp:551-554)."""
    csv, side = run("jc_mcsolve", tmp_path, "--ntraj", "40", "--seed", "7")
    tab, j = check_format(csv, side, ["t", "n_cavity_re", "n_cavity_im"])
    assert j["ntraj"] == 40 and j["seed"] == 7 and j["scenario"]["seed"] == 7
    t = make_tlist(0.0, 314.15926535897933, 1000)
    ref = O.Model("jc", 10, 1.0, 1.0, 0.1, 0.01, 0.01).mcsolve(t, 7, 40, n_threads=os.cpu_count() or 1)
    assert normwise_rel(tab[:, 1] + 1j * tab[:, 2], ref["mean"][0]) <= 1e-6


def test_qsim_run_jc_mesolve(tmp_path):
    csv, side = run("jc_mesolve", tmp_path)
    tab, j = check_format(csv, side, ["t", "n_cavity_re", "n_cavity_im"])
    t = make_tlist(0.0, 314.15926535897933, 1000)
    ex, st, _ = O.Model("jc", 10, 1.0, 1.0, 0.1, 0.01, 0.01).mesolve(t)
    assert normwise_rel(tab[:, 1] + 1j * tab[:, 2], ex[0]) <= 1e-6
    assert j["stats"]["rhs_evals"] == 2 + 6 * (j["stats"]["steps"] + j["stats"]["rejected"])
