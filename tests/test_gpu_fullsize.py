"""GPU parity at the BASELINE sizes, through the product's own model builder and operator store,
against the CPU oracle.

Full deterministic solves that take the oracle minutes (configs[1] TFIM-10: 81 DP5 attempts,
~50 s on one core; configs[3] Kerr cutoffs 150/300/400) are compared with frozen oracle outputs
(tests/golden/fullsize_golden.json, scripts/make_golden_fullsize.py; the threaded oracle that
wrote them is bit-identical to the 1-thread restatement, tests/test_oracle_pinning.py).
"""
import json
import os

import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import assert_stats_close, normwise_rel

pytestmark = pytest.mark.gpu

TFIM10 = (10, 1, 1.0, 0.2, 1.0, 1)
TFIM14 = (14, 1, 1.0, 0.2, 1.0, 1)


@pytest.fixture(scope="module")
def tfim10(ctx):
    m = q.Model("ising", *TFIM10)
    L = m.export(q.SEL_L_CONST)
    op = ctx.op(L)
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    return m, op, eops, rho0


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize_golden.json")


def golden(key):
    g = json.load(open(GOLDEN))[key]
    return np.array(g["expect_re"]) + 1j * np.array(g["expect_im"]), np.array(g["stats"]), np.array(g["tlist"])


def test_tfim10_store_is_coded(tfim10):
    _, op, _, _ = tfim10
    assert q.op_storage(op)[0] in (1, 2)  # dictionary-coded (1-byte codes) or key-aligned


def test_tfim10_full_solve_matches_golden(ctx, tfim10):
    """configs[1] end to end: the device-assembled Liouvillian (qsg_liouvillian_create, the bench's
    e2e path) in the default operator store, the complete t in [0, 10] solve, against the frozen
    oracle solve (evolve.cpp:237-299, integrator.hpp:78-147)."""
    m, _, eops, rho0 = tfim10
    H = m.export(q.SEL_H_CONST)
    cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
    ref, st, t = golden("tfim10")
    op = ctx.liouvillian(H, cops)
    dev = q.mesolve(ctx, q.Generator([op]), m.dim, rho0, t, eops)
    op.close()
    assert normwise_rel(dev["expect"], ref) <= 1e-6
    assert_stats_close(dev["stats"], st)


@pytest.mark.parametrize("N", [150, 300, 400])
def test_kerr_cutoff_full_solve_matches_golden(ctx, N):
    """configs[3] cutoffs whose oracle solves take minutes: full solves against frozen outputs."""
    from tests._helpers import e_ops_csr, rho0_vec
    m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    ref, st, t = golden(f"kerr{N}")
    om = O.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    gen = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
    dev = q.mesolve(ctx, gen, m.dim, rho0_vec(om), t, e_ops_csr(om))
    assert normwise_rel(dev["expect"], ref) <= 1e-6
    assert_stats_close(dev["stats"], st)


def test_tfim10_mesolve_prefix_matches_oracle(ctx, tfim10):
    m, op, eops, rho0 = tfim10
    t = np.linspace(0.0, 0.5, 6)
    dev = q.mesolve(ctx, q.Generator([op]), m.dim, rho0, t, eops)
    om = O.Model("ising", *TFIM10)
    om.prepare_liouvillian()
    ex, st = om.mesolve_prepared(t)
    assert normwise_rel(dev["expect"], ex) <= 1e-6
    assert_stats_close(dev["stats"], st)


def test_tfim10_full_solve_properties(ctx, tfim10):
    """Full configs[1] solve: trace preservation shows up as Sz_total staying in [-10, 10] and
    the observables being real (hermitized trace formula, evolve.cpp:286-295)."""
    m, op, eops, rho0 = tfim10
    t = np.linspace(0.0, 10.0, 100)
    r = q.mesolve(ctx, q.Generator([op]), m.dim, rho0, t, eops)
    ex = r["expect"]
    assert r["stats"][2] == 2 + 6 * (r["stats"][0] + r["stats"][1])
    assert np.max(np.abs(ex.imag)) < 1e-10
    assert abs(ex[2, 0].real - 10.0) < 1e-12  # all spins up at t = 0
    assert np.all(np.abs(ex.real) <= 10.0 + 1e-9)
    assert ex[2, -1].real < ex[2, 0].real  # decay towards the steady state


@pytest.fixture(scope="module")
def tfim14_ensemble(ctx):
    """configs[2]: trajectories 0..511 of seed 2025 on the device (qsg_mcsolve) and in the oracle
    (run_ensemble restatement on every host core)."""
    m = q.Model("ising", *TFIM14)
    G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
    cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
    eops = [m.export(q.SEL_E_OP, 2)]
    t = np.linspace(0.0, 10.0, 100)
    dev = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), t, 2025, 0, 512)
    ref = O.Model("ising", *TFIM14).mcsolve(t, 2025, 512, n_threads=os.cpu_count() or 1)
    return dev, ref


def test_tfim14_trajectories_match_oracle(tfim14_ensemble):
    """Per-trajectory parity under identical seeds, every one of 512 trajectories: same jump
    channels, jump times within 1e-9 (measured <= 1.5e-13), Sz_total within 1e-9 normwise."""
    dev, ref = tfim14_ensemble
    for i in range(512):
        dj, rj = dev["jumps"][i], ref["jumps"][i]
        assert len(dj) == len(rj), i
        assert all(a[1] == b[1] and abs(a[0] - b[0]) <= 1e-9 for a, b in zip(dj, rj)), i
        assert normwise_rel(dev["per_traj"][i][0], ref["per_traj"][i][2]) <= 1e-9, i
        times = [j[0] for j in dj]
        assert all(b > a for a, b in zip(times, times[1:]))


def test_tfim14_ensemble_mean_within_3sigma(tfim14_ensemble):
    """Ensemble mean (device bracket on the GPU) against the oracle's run_ensemble mean: within
    3 sigma/sqrt(N) of the sampling error at every time, and in fact within 1e-9."""
    dev, ref = tfim14_ensemble
    n = 512
    mean = dev["block_sum"][0] / n
    sd = np.std(dev["per_traj"][:, 0, :].real, axis=0, ddof=1)
    assert dev["n_ok"] == n
    assert np.all(np.abs(mean.real - ref["mean"][2].real) <= 3 * sd / np.sqrt(n) + 1e-12)
    assert np.max(np.abs(mean - ref["mean"][2])) <= 1e-9


@pytest.mark.parametrize("N", [50, 100, 200])
def test_kerr_cutoff_sweep_matches_oracle(ctx, N):
    """configs[3]: Kerr resonator mesolve at cutoff N (Liouvillian N^2 rows), abstol 1e-8,
    tlist linspace(0,10,101), against the oracle's full solve."""
    from tests._helpers import e_ops_csr, oracle_generator, rho0_vec
    m = O.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
    t = np.linspace(0.0, 10.0, 101)
    dev = q.mesolve(ctx, oracle_generator(ctx, m, "me"), m.dim, rho0_vec(m), t, e_ops_csr(m))
    ex, st, _ = m.mesolve(t)
    assert normwise_rel(dev["expect"], ex) <= 1e-6
    assert_stats_close(dev["stats"], st)


def test_coupled_kerr_sweep_points_match_oracle(ctx):
    """configs[4] at its real size (two N=10 modes, Liouvillian 10^4 rows): the batched sweep
    engine on the grid's corners and two interior points (Delta in linspace(-2,2,16) x F in
    linspace(0.1,1,16)) against one oracle mesolve per point."""
    from tests._helpers import e_ops_csr, oracle_generator
    m = O.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
    gen = oracle_generator(ctx, m, "me")
    dl, fl = np.linspace(-2, 2, 16), np.linspace(0.1, 1.0, 16)
    pts = np.array([[dl[0], fl[0]], [dl[15], fl[0]], [dl[0], fl[15]], [dl[15], fl[15]], [dl[7], fl[9]],
                    [dl[11], fl[3]]])
    t = np.linspace(0.0, 10.0, 101)
    rho0 = np.zeros(m.dim * m.dim, complex)
    rho0[0] = 1.0
    res = q.mesolve_batch(ctx, gen, m.dim, rho0, t, e_ops_csr(m), pts)
    assert np.all(res["status"] == 0)
    for p, prm in enumerate(pts):
        ex, st, _ = m.mesolve(t, params=prm)
        assert normwise_rel(res["expect"][p], ex) <= 1e-6, p
        assert_stats_close(res["stats"][p], st)


def test_tfim10_key_aligned_solve(ctx, tfim10, monkeypatch):
    """The opt-in key-aligned store (QSG_KA_STORE / QSG_KA_SOLVE, TMA ring) on the full configs[1]
    solve: same golden, same step statistics as the default coded path."""
    m, _, eops, rho0 = tfim10
    H = m.export(q.SEL_H_CONST)
    cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
    ref, st, t = golden("tfim10")
    monkeypatch.setenv("QSG_KA_SOLVE", "1")
    op = ctx.liouvillian(H, cops)
    info = q.op_store_info(op)
    assert info["store"] == "key-aligned" and 0 < info["ka_bytes"] < info["coded_bytes"]
    dev = q.mesolve(ctx, q.Generator([op]), m.dim, rho0, t, eops)
    op.close()
    assert dev["store"] == 2
    assert normwise_rel(dev["expect"], ref) <= 1e-6
    assert_stats_close(dev["stats"], st)
