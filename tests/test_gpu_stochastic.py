"""GPU parity of the stochastic solvers (qsg_ssesolve / qsg_smesolve, trajectories.cpp:251-503)
against the oracle, trajectory by trajectory on the same RngStream(seed, i).

The device draws the same uniforms (bit-exact RNG) but its log/sin/cos in Box-Muller may differ
from glibc in the last ulp, and it contracts FMAs, so per-trajectory results agree to ~1e-12, far
inside the 1e-6 bar; the current record J = e + dW/dt holds exactly (trajectories.cpp:351).
"""
import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import csr_from_oracle, e_ops_csr, normwise_rel, oracle_generator, rho0_vec

pytestmark = pytest.mark.gpu
TOL = 1e-8


def _sse(ctx, m, t, seed, ntraj, dt_max, store=False):
    G = oracle_generator(ctx, m, "se")
    sc = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    return q.ssesolve(ctx, G, sc, e_ops_csr(m), m.dim, m.psi0(), t, seed, 0, ntraj, dt_max=dt_max,
                      store_measurement=store)


@pytest.mark.parametrize("name,params", [("jc_sse", (6, 1.0, 1.0, 0.1, 0.3)),
                                         ("jc_sme", (5, 1.0, 1.0, 0.2, 0.4, 0.2, 0.1))])
def test_ssesolve_matches_oracle(ctx, name, params):
    """single-channel fast path (jc_sse) and the 3-channel general path (jc_sme's ops as sc_ops)."""
    m = O.Model(name, *params)
    t = np.linspace(0.0, 0.5, 6)
    dev = _sse(ctx, m, t, 31, 8, 1e-3, store=True)
    ref = m.ssesolve(t, 31, 8, dt_max=1e-3, store_measurement=True)
    assert dev["n_steps"] == ref["n_steps"] and dev["dt"] == ref["dt"]
    for i in range(8):
        assert normwise_rel(dev["per_traj"][i], ref["per_traj"][i]) <= TOL, i
    assert np.max(np.abs(dev["increments"] - ref["increments"])) <= 1e-13 * np.max(np.abs(ref["increments"]))
    assert np.max(np.abs(dev["expectation"] - ref["expectation"])) <= TOL
    assert np.max(np.abs(dev["current"] - (dev["expectation"] + dev["increments"] / dev["dt"]))) == 0.0
    assert normwise_rel(dev["mean"], ref["mean"]) <= TOL


def test_smesolve_matches_oracle(ctx):
    """jc_sme: c_ops {sqrt(gamma) sm, sqrt(kphi) n} deterministic, sqrt(kappa) a measured."""
    m = O.Model("jc_sme", 4, 1.0, 1.0, 0.1, 1.0, 0.1, 0.05)
    t = np.linspace(0.0, 1.0, 11)
    L = oracle_generator(ctx, m, "me")  # liouvillian(H, c_ops + sc_ops)
    sc = [csr_from_oracle(m, O.C_OP, 2)]
    dev = q.smesolve(ctx, L, sc, e_ops_csr(m), m.dim, rho0_vec(m), t, 7, 0, 6, dt_max=2e-3, store_measurement=True)
    ref = m.smesolve(t, 7, 6, n_det=2, dt_max=2e-3, store_measurement=True)
    for i in range(6):
        assert normwise_rel(dev["per_traj"][i], ref["per_traj"][i]) <= TOL, i
    assert np.max(np.abs(dev["increments"] - ref["increments"])) <= 1e-13 * np.max(np.abs(ref["increments"]))
    assert normwise_rel(dev["mean"], ref["mean"]) <= TOL


def test_sse_deterministic_limit_and_uniform_grid(ctx):
    """test_trajectories.cpp:205-216 on the device; a non-uniform tlist is rejected."""
    m = O.Model("jc_sse", 8, 1.0, 1.0, 0.1, 0.0)
    t = np.linspace(0.0, 5.0, 26)
    dev = _sse(ctx, m, t, 11, 1, 1e-4)
    se, _, _ = O.Model("jc", 8, 1.0, 1.0, 0.1, 0.0, 0.0).sesolve(t)
    assert np.max(np.abs(dev["mean"][0] - se[0])) < 5e-4
    with pytest.raises(q.QsgError) as ei:
        _sse(ctx, m, np.array([0.0, 0.1, 0.3]), 11, 1, 1e-3)
    assert ei.value.code == 11


def test_sse_ensemble_matches_oracle_and_converges(ctx):
    """64 trajectories: the device ensemble mean equals the oracle's (same trajectories), and the
    X-quadrature mean approaches mesolve (test_trajectories.cpp:320-344)."""
    m = O.Model("jc_sse", 4, 1.0, 1.0, 0.1, 1.0)
    t = np.linspace(0.0, 2.0, 21)
    dev = _sse(ctx, m, t, 2024, 64, 2e-3)
    ref = m.ssesolve(t, 2024, 64, dt_max=2e-3)
    assert normwise_rel(dev["mean"], ref["mean"]) <= TOL
    me, _, _ = m.mesolve(t)
    assert np.max(np.abs(dev["mean"][2] - me[2])) < 0.25


def test_cpp_ssesolve_smesolve_match_oracle():
    """qsim::ssesolve / qsim::smesolve of the C++ host API (zoo models) against the oracle."""
    t = np.linspace(0.0, 0.5, 6)
    dev = q.Model("jc_sse", 6, 1.0, 1.0, 0.1, 0.3).ssesolve(t, 31, 8, dt_max=1e-3, store_measurement=True)
    ref = O.Model("jc_sse", 6, 1.0, 1.0, 0.1, 0.3).ssesolve(t, 31, 8, dt_max=1e-3, store_measurement=True)
    assert normwise_rel(dev["mean"], ref["mean"]) <= TOL
    assert np.max(np.abs(dev["increments"] - ref["increments"])) <= 1e-13 * np.max(np.abs(ref["increments"]))
    prm = (4, 1.0, 1.0, 0.1, 1.0, 0.1, 0.05)
    t2 = np.linspace(0.0, 1.0, 11)
    dev = q.Model("jc_sme", *prm).smesolve(t2, 7, 6, n_det=2, dt_max=2e-3)
    ref = O.Model("jc_sme", *prm).smesolve(t2, 7, 6, n_det=2, dt_max=2e-3)
    for i in range(6):
        assert normwise_rel(dev["per_traj"][i], ref["per_traj"][i]) <= TOL, i


def test_ssesolve_without_e_ops(ctx):
    """Empty e_ops is legal (the reference stores nothing per trajectory): the call must not write
    past the caller's zero-length buffers, and the measurement records still match the oracle."""
    m = O.Model("jc_sse", 6, 1.0, 1.0, 0.1, 0.3)
    t = np.linspace(0.0, 0.5, 6)
    G = oracle_generator(ctx, m, "se")
    sc = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    guard = np.full(64, 7.25)
    dev = q.ssesolve(ctx, G, sc, [], m.dim, m.psi0(), t, 31, 0, 8, dt_max=1e-3, store_measurement=True)
    assert dev["per_traj"].size == 0 and np.all(guard == 7.25)
    ref = m.ssesolve(t, 31, 8, dt_max=1e-3, store_measurement=True)
    assert np.max(np.abs(dev["increments"] - ref["increments"])) <= 1e-13 * np.max(np.abs(ref["increments"]))
