"""GPU parity of the batched Monte-Carlo engine (qsg_mcsolve) and the parameter-sweep engine
(qsg_mesolve_batch) against the CPU oracle, plus the reference's statistical assertions.

Per-trajectory parity: trajectory i draws from RngStream(seed, i) on both sides, so jump
channels must agree exactly and jump times / observables within the integrator tolerance.
"""
import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import assert_stats_close, csr_from_oracle, e_ops_csr, normwise_rel, oracle_generator

pytestmark = pytest.mark.gpu


def _mc(ctx, m, tlist, seed, b, e, **kw):
    gen = oracle_generator(ctx, m, "mc")
    cops = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    return q.mcsolve(ctx, gen, cops, e_ops_csr(m), m.dim, m.psi0(), tlist, seed, b, e, **kw)


def _compare_trajectories(dev, ref, lo=0, jt_tol=1e-6, ex_tol=1e-6, allow_diverged=0):
    diverged = 0
    for i in range(min(len(dev["jumps"]), len(ref["jumps"]) - lo)):
        dj, rj = dev["jumps"][i], ref["jumps"][lo + i]
        same = len(dj) == len(rj) and all(a[1] == b[1] and abs(a[0] - b[0]) <= jt_tol * max(1, abs(b[0]))
                                          for a, b in zip(dj, rj))
        if not same:
            diverged += 1
            continue
        assert normwise_rel(dev["per_traj"][i], ref["per_traj"][lo + i]) <= ex_tol, i
    assert diverged <= allow_diverged, diverged


def test_mc_threshold_crossing_located(ctx):
    """test_trajectories.cpp:66-88 on the device: |exp(-g t_jump) - r| < 5e-10."""
    m = O.Model("decay2", 0.8)
    r = _mc(ctx, m, np.linspace(0, 30, 31), 99, 0, 64, abstol=1e-13, reltol=1e-12)
    assert r["n_ok"] == 64
    for i in range(64):
        assert len(r["jumps"][i]) == 1
        u = O.rng(99, i, 2, 1)[0]
        assert abs(np.exp(-0.8 * r["jumps"][i][0][0]) - u) < 5e-10


def test_mc_decay_law_and_oracle_parity(ctx):
    """test_trajectories.cpp:40-64 statistics + per-trajectory parity with the oracle."""
    m = O.Model("decay2", 0.25)
    t = np.linspace(0, 80, 41)
    dev = _mc(ctx, m, t, 2025, 0, 2000)
    times = np.array([j[0][0] for j in dev["jumps"]])
    assert all(len(j) == 1 for j in dev["jumps"])
    assert abs(times.mean() - 4.0) / 4.0 < 0.05
    ref = m.mcsolve(t, 2025, 256)
    _compare_trajectories(dev, ref)


def test_mc_disjoint_seeds_ks(ctx):
    """test_trajectories.cpp:186-203 on the device: first-jump times of 400 decaying-qubit
    trajectories from seeds 1000 and 2000 pass a two-sample KS test (p > 0.01, scipy's ks_2samp
    for the reference's test::ks_two_sample_pvalue), and each sample passes a one-sample KS test
    against the exact first-jump law 1 - exp(-gamma t), truncated at t = 40."""
    from scipy.stats import ks_2samp, kstest
    m = O.Model("decay2", 0.5)
    t = np.linspace(0.0, 40.0, 21)
    samples = []
    for seed in (1000, 2000):
        r = _mc(ctx, m, t, seed, 0, 400)
        assert r["n_ok"] == 400
        samples.append(np.array([j[0][0] for j in r["jumps"] if len(j)]))
        ref = m.mcsolve(t, seed, 32)  # the same draws as the restatement, trajectory by trajectory
        _compare_trajectories(r, ref)
    assert ks_2samp(samples[0], samples[1]).pvalue > 0.01
    for x in samples:
        assert kstest(x, lambda v: (1.0 - np.exp(-0.5 * v)) / (1.0 - np.exp(-20.0))).pvalue > 0.01


def test_mc_jc_per_trajectory_parity(ctx):
    m = O.Model("jc", 6, 1.0, 1.0, 0.1, 0.05, 0.05)
    t = np.linspace(0, 60, 61)
    dev = _mc(ctx, m, t, 7, 0, 16)
    ref = m.mcsolve(t, 7, 16)
    _compare_trajectories(dev, ref)
    for i in range(16):
        assert_stats_close(dev["stats"][i], ref["stats"][i], restarts=len(ref["jumps"][i]))


def test_mc_ising_trajectory_block_independent(ctx):
    """Any partition of the trajectory range gives identical per-trajectory results."""
    m = O.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    full = _mc(ctx, m, t, 2025, 0, 24)
    part = _mc(ctx, m, t, 2025, 8, 16)
    assert part["jumps"] == full["jumps"][8:16]
    assert np.array_equal(part["per_traj"], full["per_traj"][8:16])
    ref = m.mcsolve(t, 2025, 24)
    _compare_trajectories(full, ref)


def test_mc_mean_matches_mesolve_4sigma(ctx):
    """test_trajectories.cpp:90-114: |mc - me| <= 4 sigma/sqrt(N) + 1e-3 at every grid point."""
    m = O.Model("jc", 10, 1.0, 1.0, 0.1, 0.01, 0.01)
    t = np.linspace(0, 10 * np.pi / 0.1, 101)
    n = 400
    dev = _mc(ctx, m, t, 7, 0, n)
    me, _, _ = m.mesolve(t)
    mean = dev["block_sum"] / dev["n_ok"]
    sd = np.std(dev["per_traj"][:, 0, :].real, axis=0, ddof=1)
    assert np.all(np.abs(mean[0].real - me[0].real) <= 4 * sd / np.sqrt(n) + 1e-3)


def test_mc_zero_collapse_reduces_to_sesolve(ctx):
    m = O.Model("jc", 8, 1.0, 1.0, 0.1, 0.0, 0.0)
    t = np.linspace(0, 25, 26)
    dev = _mc(ctx, m, t, 5, 0, 3, abstol=1e-12, reltol=1e-11)
    se, _, _ = m.sesolve(t, abstol=1e-12, reltol=1e-11)
    assert all(len(j) == 0 for j in dev["jumps"])
    assert np.max(np.abs(dev["block_sum"] / 3 - se)) < 1e-9


def test_ensemble_combine_matches_pairwise(ctx):
    """Blocks [0,5000) [5000,10000)-style tiling reproduces the single-block bracket bitwise."""
    m = O.Model("jc", 6, 1.0, 1.0, 0.1, 0.05, 0.05)
    t = np.linspace(0, 20, 21)
    full = _mc(ctx, m, t, 11, 0, 64)
    blocks = [(0, 16), (16, 32), (32, 48), (48, 64)]
    parts = [_mc(ctx, m, t, 11, b, e) for b, e in blocks]
    mean = q.ensemble_combine(blocks, [p["block_sum"] for p in parts], 64)
    ref = full["block_sum"] / 64
    assert np.array_equal(mean.view(np.float64), ref.view(np.float64))


def test_mesolve_batch_sweep_parity(ctx):
    """Parameter sweep (a14): per-point device results vs one oracle mesolve per point."""
    m = O.Model("coupled_kerr", 4, 0.1, 0.5, 1.0)
    gen = oracle_generator(ctx, m, "me")
    t = np.linspace(0, 10, 101)
    pts = np.array([[d, f] for d in (-2.0, 0.0, 1.3) for f in (0.1, 0.55, 1.0)])
    rho0 = np.zeros(m.dim * m.dim, complex)
    rho0[0] = 1.0
    res = q.mesolve_batch(ctx, gen, m.dim, rho0, t, e_ops_csr(m), pts)
    assert np.all(res["status"] == 0)
    for p, prm in enumerate(pts):
        ex, st, _ = m.mesolve(t, params=prm)
        assert normwise_rel(res["expect"][p], ex) <= 1e-6, p
        assert_stats_close(res["stats"][p], st)


MODES = ["local1", "local2", "local4", "local", "grid", "cluster1", "cluster2"]


@pytest.fixture(params=MODES)
def batch_mode(request, monkeypatch):
    """Every batch-engine layout: 1/2/4/8 slots per CTA, the grid-wide 32-slot batch and 1/2 slots
    per 16-CTA cluster."""
    monkeypatch.setenv("QSG_BATCH_MODE", request.param)
    return request.param


def test_both_modes_jc_parity(ctx, batch_mode):
    m = O.Model("jc", 6, 1.0, 1.0, 0.1, 0.05, 0.05)
    t = np.linspace(0, 60, 61)
    dev = _mc(ctx, m, t, 7, 0, 40)
    ref = m.mcsolve(t, 7, 40)
    _compare_trajectories(dev, ref)


def test_both_modes_threshold_crossing(ctx, batch_mode):
    m = O.Model("decay2", 0.8)
    r = _mc(ctx, m, np.linspace(0, 30, 31), 99, 0, 48, abstol=1e-13, reltol=1e-12)
    for i in range(48):
        u = O.rng(99, i, 2, 1)[0]
        assert abs(np.exp(-0.8 * r["jumps"][i][0][0]) - u) < 5e-10


def test_both_modes_ising_identical(ctx, monkeypatch):
    """All layouts give the same per-trajectory records (TFIM-7 chain)."""
    m = O.Model("ising", 7, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    out = {}
    for mode in MODES:
        monkeypatch.setenv("QSG_BATCH_MODE", mode)
        out[mode] = _mc(ctx, m, t, 2025, 0, 40)
    # same trajectories; only the reduction order differs (jump times agree to ~1e-13)
    for mode in MODES[1:]:
        _compare_trajectories(out[mode], out["local1"], jt_tol=1e-9, ex_tol=1e-9)
    ref = m.mcsolve(t, 2025, 40)
    _compare_trajectories(out["grid"], ref)


def test_both_modes_sweep(ctx, batch_mode):
    m = O.Model("coupled_kerr", 4, 0.1, 0.5, 1.0)
    gen = oracle_generator(ctx, m, "me")
    t = np.linspace(0, 10, 101)
    pts = np.array([[-1.0, 0.3], [0.5, 0.9], [2.0, 0.1]])
    rho0 = np.zeros(m.dim * m.dim, complex)
    rho0[0] = 1.0
    res = q.mesolve_batch(ctx, gen, m.dim, rho0, t, e_ops_csr(m), pts)
    for p, prm in enumerate(pts):
        ex, st, _ = m.mesolve(t, params=prm)
        assert normwise_rel(res["expect"][p], ex) <= 1e-6


# ---- ensembles through the reference-facing C++ API (qsim::mcsolve) ------------------------------

def test_mcsolve_duplicate_devices_bitwise(ctx):
    """qsim::mcsolve over devices (0, 0): two shards, one context each (no shared stream or events),
    combined in the bracket. Bitwise equal to the single-device run."""
    m = q.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    a = m.mcsolve(t, 2025, 96, devices=(0,))
    b = m.mcsolve(t, 2025, 96, devices=(0, 0))
    assert a["jumps"] == b["jumps"]
    assert np.array_equal(a["mean"].view(np.float64), b["mean"].view(np.float64))
    assert np.array_equal(a["per_traj"].view(np.float64), b["per_traj"].view(np.float64))


def test_mcsolve_three_shards_bitwise(ctx):
    """A non-power-of-two shard count: bracket-subtree shards (ensemble_shards) still combine into
    the single-device mean bit for bit."""
    m = q.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    a = m.mcsolve(t, 2025, 100, devices=(0,))
    b = m.mcsolve(t, 2025, 100, devices=(0, 0, 0))
    assert np.array_equal(a["mean"].view(np.float64), b["mean"].view(np.float64))


def test_mcsolve_nccl_path_single_rank(ctx, monkeypatch):
    """The NCCL all-gather path of qsim::mcsolve (qsg_comm_init_all + qsg_comm_allgather), forced
    on one device: same mean, bit for bit."""
    import ctypes
    assert q.lib().qsg_nccl_version() > 0
    m = q.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    a = m.mcsolve(t, 2025, 64, devices=(0,))
    monkeypatch.setenv("QSG_MC_NCCL", "1")
    b = m.mcsolve(t, 2025, 64, devices=(0,))
    assert np.array_equal(a["mean"].view(np.float64), b["mean"].view(np.float64))


def test_mcsolve_long_jump_logs_kept(ctx, monkeypatch):
    """Trajectories with more jumps than the batch buffers hold are re-run with room for the whole
    list (the reference keeps every jump, trajectories.cpp:189-200): capacity forced to 4 on the
    driven-dissipative TFIM-6 chain, whose spins decay and are re-excited many times."""
    monkeypatch.setenv("QSG_MC_JUMP_CAP", "4")
    t = np.linspace(0, 10, 100)
    dev = q.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1).mcsolve(t, 2025, 16)
    ref = O.Model("ising", 6, 1, 1.0, 0.2, 1.0, 1).mcsolve(t, 2025, 16)
    assert max(len(j) for j in dev["jumps"]) > 4
    for dj, rj in zip(dev["jumps"], ref["jumps"]):
        assert len(dj) == len(rj)
        assert all(a[1] == b[1] and abs(a[0] - b[0]) < 1e-9 for a, b in zip(dj, rj))


def test_ensemble_stddev_matches_sample_std(ctx):
    """qsim::ensemble_stddev (trajectories.cpp:94-104): sample std (n-1) of Re over trajectories."""
    m = q.Model("jc", 6, 1.0, 1.0, 0.1, 0.05, 0.05)
    t = np.linspace(0, 60, 61)
    r = m.mcsolve(t, 7, 64)
    ref = np.std(r["per_traj"].real, axis=0, ddof=1)
    assert np.allclose(r["stddev"], ref, rtol=1e-10, atol=1e-14)


def test_ising6_mcsolve_matches_mesolve_3sigma(ctx):
    """SPEC acceptance #12 in the pattern of test_trajectories.cpp:90-114, at 3 sigma: the 2x3
    dissipative Ising lattice of scenarios/ising_mc_2x3.json (Sz_total), 2,000 trajectories of seed
    2025, against the device mesolve and the oracle mesolve."""
    t = np.linspace(0.0, 10.0, 100)
    m = q.Model("ising", 2, 3, 1.0, 0.2, 1.0, 1)
    mc = m.mcsolve(t, 2025, 2000)
    me = m.mesolve(t, device=0)["expect"]
    om, _, _ = O.Model("ising", 2, 3, 1.0, 0.2, 1.0, 1).mesolve(t)
    assert normwise_rel(me, om) <= 1e-6
    e = 2  # Sz_total
    sd = mc["stddev"][e]
    viol = np.abs(mc["mean"][e].real - om[e].real) > 3 * sd / np.sqrt(2000) + 1e-3
    assert viol.sum() <= 1, np.nonzero(viol)


def _pairwise(mats, lo, hi):
    if hi - lo == 1:
        return mats[lo].copy()
    mid = lo + (hi - lo) // 2
    return _pairwise(mats, lo, mid) + _pairwise(mats, mid, hi)


def test_device_bracket_sums_large_ensemble(ctx):
    """The device bracket (K7) over 5,000 trajectories (13 levels) equals the host pairwise_sum of
    the per-trajectory data bit for bit, and so do sub-range sums."""
    m = O.Model("decay2", 0.25)
    t = np.linspace(0, 40, 21)
    r = _mc(ctx, m, t, 3, 0, 5000, ranges=[(0, 2500), (2500, 5000), (17, 4099)])
    per = list(r["per_traj"])
    assert np.array_equal(r["block_sum"].view(np.float64), _pairwise(per, 0, 5000).view(np.float64))
    for (lo, hi), s in zip([(0, 2500), (2500, 5000), (17, 4099)], r["range_sums"]):
        assert np.array_equal(s.view(np.float64), _pairwise(per, lo, hi).view(np.float64))


def test_cluster_dsm_layout_matches_oracle(ctx, monkeypatch):
    """Batch layout 7 (one trajectory per cluster, state in distributed shared memory): same
    trajectories as the oracle (TFIM-7 chain, seed 2025)."""
    monkeypatch.setenv("QSG_BATCH_MODE", "clusterdsm")
    m = O.Model("ising", 7, 1, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0, 10, 100)
    dev = _mc(ctx, m, t, 2025, 0, 24)
    ref = m.mcsolve(t, 2025, 24)
    _compare_trajectories(dev, ref)
