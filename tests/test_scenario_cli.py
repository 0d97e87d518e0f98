"""CPU tests of the scenario runner CLI (bin/qsim; the reference's tools/qsim.cpp:34-102 and
scenario.cpp validation, :105-205): built-in list, validation diagnostics and exit codes, and the
loud failure of `run` without a device (no CPU fallback). GPU runs: tests/test_gpu_scenario.py."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QSIM = os.path.join(ROOT, "paper_2504_21440_b200", "bin", "qsim")


def qsim(*args):
    return subprocess.run([QSIM, *args], capture_output=True, text=True, timeout=120)


def spec(tmp_path, **over):
    s = {"name": "t", "model": "ising", "solver": "mcsolve",
         "params": {"nx": 2, "ny": 3, "Jz": 1.0, "hx": 0.2, "gamma": 1.0, "periodic": 1},
         "tlist": {"t0": 0.0, "tf": 1.0, "n_points": 11}, "e_ops": ["Sz_total"], "ntraj": 4, "seed": 1}
    s.update(over)
    p = tmp_path / "s.json"
    p.write_text(json.dumps(s))
    return str(p)


def test_list_builtins():
    r = qsim("list")
    assert r.returncode == 0
    names = r.stdout.split()
    for n in ("ising_mc_2x3", "jc_mcsolve", "jc_mesolve", "jc_sesolve", "sse_homodyne", "sme_homodyne", "optomech_td"):
        assert n in names


def test_validate_builtin_and_json_suffix():
    for arg in ("ising_mc_2x3", "ising_mc_2x3.json"):
        r = qsim("validate", arg)
        assert r.returncode == 0 and json.loads(r.stdout) == {"valid": True, "diagnostics": []}


@pytest.mark.parametrize("over,diag", [
    ({"model": "nope"}, ["unknown_model"]),
    ({"solver": "nope"}, ["unknown_solver"]),
    ({"params": {"nx": 4, "ny": 4, "Jz": 1.0, "hx": 0.2, "gamma": 1.0, "periodic": 1}}, ["bad_param:lattice_too_large"]),
    ({"params": {"nx": 2, "ny": 3, "Jz": 1.0, "hx": 0.2, "periodic": 1}}, ["missing_param:gamma"]),
    ({"e_ops": ["n_cavity"]}, ["unknown_observable:n_cavity"]),
    ({"tlist": {"t0": 1.0, "tf": 1.0, "n_points": 1}}, ["nonpositive_time_span", "bad_n_points"]),
    ({"ntraj": 0}, ["bad_param:ntraj"]),
    ({"solver": "sesolve"}, ["unsupported_model_solver"]),
])
def test_validate_diagnostics(tmp_path, over, diag):
    """scenario.cpp:157-205 diagnostics, in order; `validate` exits 2, `run` exits 2 with the
    machine-readable error (first diagnostic's code) before touching a device."""
    p = spec(tmp_path, **over)
    r = qsim("validate", p)
    assert r.returncode == 2
    assert json.loads(r.stdout) == {"valid": False, "diagnostics": diag}
    r = qsim("run", p, "--out-dir", str(tmp_path / "o"))
    assert r.returncode == 2
    err = json.loads(r.stderr)
    assert err["diagnostics"] == diag and err["error"] == diag[0].split(":")[0]


def test_malformed_and_missing_specs(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{\"name\": ")
    r = qsim("validate", str(bad))
    assert r.returncode == 2 and json.loads(r.stderr)["error"] == "InvalidScenario"
    r = qsim("run", "no_such_scenario")
    assert r.returncode == 2 and "no such scenario" in json.loads(r.stderr)["message"]


def test_run_without_device_fails_loudly(tmp_path):
    """No CUDA device here: the solve must fail with exit 3 (no CPU fallback) and write no CSV."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    out = tmp_path / "o"
    r = qsim("run", spec(tmp_path), "--out-dir", str(out))
    assert r.returncode == 3
    assert json.loads(r.stderr)["error"] in ("exception", "IntegrationFailure")
    assert not (out / "t.csv").exists()
