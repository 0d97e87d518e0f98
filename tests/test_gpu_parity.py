"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same inputs.

Tolerances (north_star): deterministic solver outputs within max normwise relative error 1e-6
at identical abstol/reltol/tlist; integer work (RNG) bit-exact.
"""
import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import (assert_stats_close, csr_from_oracle, e_ops_csr, normwise_rel,
                            oracle_generator, rho0_vec)

pytestmark = pytest.mark.gpu

TOL = 1e-6


def test_device_is_b200(ctx):
    assert ctx.sm_count >= 132, ctx.name


@pytest.mark.parametrize("seed,stream", [(0, 0), (2025, 0), (2025, 9999), (99, 63), (2**63 + 5, 7)])
def test_rng_bit_exact(ctx, seed, stream):
    for kind in (0, 1, 2):
        dev = q.rng_draw(ctx, seed, stream, kind, 64)
        ref = O.rng(seed, stream, kind, 64)
        assert np.array_equal(dev, ref), (kind, dev[:4], ref[:4])


@pytest.mark.parametrize("name,params,kind", [
    ("kerr", (20, 1.0, 0.01, 2.0, 1.0), "me"),
    ("ising", (3, 2, 1.0, 0.2, 1.0, 1), "me"),
    ("ising", (7, 1, 1.0, 0.2, 1.0, 1), "mc"),
    ("coupled_kerr", (4, 0.1, 0.5, 1.0), "me"),
    ("driven_cavity_td", (14, 0.4), "me"),
])
def test_generator_apply_matches_oracle(ctx, name, params, kind):
    m = O.Model(name, *params)
    gen = oracle_generator(ctx, m, kind)
    n = gen.n
    rng = np.random.default_rng(1)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    prm = m.default_params if m.n_terms else None
    if m.n_terms:
        prm = np.array([0.7, 1.3])
    t = 0.37
    dev = q.generator_apply(ctx, gen, y, t=t, params=prm)
    which = {"me": O.L_CONST, "mc": O.MC_GEN}[kind]
    ref = m.generator_apply(which, t, y, params=prm)
    assert np.max(np.abs(dev - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


def _me_parity(ctx, m, tlist, params=None, **kw):
    gen = oracle_generator(ctx, m, "me")
    res = q.mesolve(ctx, gen, m.dim, rho0_vec(m), tlist, e_ops_csr(m), params=params, **kw)
    ex, st, states = m.mesolve(tlist, params=params, **kw)
    return res, ex, st, states


def test_mesolve_kerr20_parity(ctx):
    """BASELINE config 1: Kerr N=20, Tsit5->DP5 abstol 1e-8 (runs on the CPU reference)."""
    m = O.Model("kerr", 20, 1.0, 0.01, 2.0, 1.0)
    t = np.linspace(0.0, 10.0, 101)
    res, ex, st, _ = _me_parity(ctx, m, t)
    assert normwise_rel(res["expect"], ex) <= TOL
    assert_stats_close(res["stats"], st)


def test_mesolve_damped_cavity_analytic(ctx):
    """test_evolve.cpp:124-140 restated on the device path."""
    m = O.Model("damped_cavity", 10, 1.0, 0.1, 3)
    t = np.linspace(0.0, 10.0, 101)
    res, ex, st, _ = _me_parity(ctx, m, t)
    expected = 3.0 * np.exp(-0.1 * t)
    assert np.max(np.abs(res["expect"][0].real - expected) / expected) < 1e-6
    assert normwise_rel(res["expect"], ex) <= TOL
    assert_stats_close(res["stats"], st)


@pytest.mark.parametrize("cluster_solve", ["0", "1"])
def test_mesolve_ising_states_and_saveat(ctx, monkeypatch, cluster_solve):
    """State saves and saveat events on the grid engine and on K-cluster."""
    monkeypatch.setenv("QSG_CLUSTER_SOLVE", cluster_solve)
    m = O.Model("ising", 3, 2, 1.0, 0.2, 1.0, 1)
    t = np.linspace(0.0, 4.0, 21)
    sv = np.array([0.0, 0.33, 1.0, 2.5, 4.0])
    res, ex, st, states = _me_parity(ctx, m, t, saveat=sv)
    assert normwise_rel(res["expect"], ex) <= TOL
    assert_stats_close(res["stats"], st)
    assert res["states"].shape == states.shape
    assert np.max(np.abs(res["states"] - states)) <= TOL * np.max(np.abs(states))


def test_mesolve_td_driven_cavity(ctx):
    """test_evolve.cpp:203-237: time-dependent drive via device PARAM_COS coefficient."""
    m = O.Model("driven_cavity_td", 14, 0.4)
    t = np.linspace(0.0, 6.0, 61)
    res, ex, st, _ = _me_parity(ctx, m, t, params=np.array([0.25, 1.3]))
    assert normwise_rel(res["expect"], ex) <= TOL
    assert_stats_close(res["stats"], st)


def test_mesolve_no_eops_returns_states(ctx):
    m = O.Model("kerr", 6, 1.0, 0.1, 0.5, 0.5)
    gen = oracle_generator(ctx, m, "me")
    t = np.linspace(0.0, 2.0, 5)
    res = q.mesolve(ctx, gen, m.dim, rho0_vec(m), t, [])
    ex, st, states = m.mesolve(t, store_states=True)
    assert res["states"].shape == (5, 36)
    assert np.max(np.abs(res["states"] - states)) <= 1e-6 * np.max(np.abs(states))


def test_sesolve_jc_parity(ctx):
    m = O.Model("jc", 10, 1.0, 1.0, 0.1, 0.0, 0.0)
    gen = oracle_generator(ctx, m, "se")
    t = np.linspace(0.0, 10.0 * np.pi / 0.1, 200)
    res = q.sesolve(ctx, gen, m.dim, m.psi0(), t, e_ops_csr(m))
    ex, st, _ = m.sesolve(t)
    assert normwise_rel(res["expect"], ex) <= TOL
    assert_stats_close(res["stats"], st)
    # JC vacuum Rabi oracle (test_evolve.cpp:72-83)
    assert np.max(np.abs(res["expect"][0].real - np.sin(0.1 * t) ** 2)) < 1e-4


def test_mesolve_failure_maps_to_integration_failure(ctx):
    m = O.Model("kerr", 20, 1.0, 0.01, 2.0, 1.0)
    gen = oracle_generator(ctx, m, "me")
    with pytest.raises(q.QsgError) as ei:
        q.mesolve(ctx, gen, m.dim, rho0_vec(m), np.linspace(0, 10, 11), e_ops_csr(m), max_steps=5)
    assert ei.value.code == 7 and "max step count exceeded" in str(ei.value)


def test_invalid_tlist(ctx):
    m = O.Model("kerr", 4, 1.0, 0.01, 0.5, 1.0)
    gen = oracle_generator(ctx, m, "me")
    with pytest.raises(q.QsgError) as ei:
        q.mesolve(ctx, gen, m.dim, rho0_vec(m), [0.0], e_ops_csr(m))
    assert ei.value.code == 11
    with pytest.raises(q.QsgError):
        q.mesolve(ctx, gen, m.dim, rho0_vec(m), [0.0, 2.0, 1.0], e_ops_csr(m))


@pytest.mark.parametrize("compress", ["1", "0"])
def test_operator_store_formats_agree(ctx, monkeypatch, compress):
    """Plain and dictionary-coded SELL stores give the same SpMV and the same solve."""
    monkeypatch.setenv("QSG_NO_COMPRESS", "0" if compress == "1" else "1")
    monkeypatch.setenv("QSG_COMPRESS_MIN_BYTES", "0")  # code even this L2-sized operator
    m = O.Model("ising", 3, 2, 1.0, 0.2, 1.0, 1)
    gen = oracle_generator(ctx, m, "me")
    cb, nd = q.op_storage(gen.ops[0])
    assert (cb > 0) == (compress == "1"), (cb, nd)
    rng = np.random.default_rng(5)
    y = rng.standard_normal(gen.n) + 1j * rng.standard_normal(gen.n)
    dev = q.generator_apply(ctx, gen, y)
    ref = m.generator_apply(O.L_CONST, 0.0, y)
    assert np.max(np.abs(dev - ref)) <= 1e-13 * np.max(np.abs(ref))
    t = np.linspace(0, 4, 41)
    res = q.mesolve(ctx, gen, m.dim, rho0_vec(m), t, e_ops_csr(m))
    ex, st, _ = m.mesolve(t)
    assert normwise_rel(res["expect"], ex) <= TOL


def test_context_outlives_its_operators():
    """qsg_ctx_destroy before qsg_op_destroy: the context is released by its last operator."""
    c = q.Context(0)
    m = O.Model("kerr", 6, 1.0, 0.1, 0.5, 0.5)
    a = c.op(csr_from_oracle(m, O.L_CONST))
    b = c.op(csr_from_oracle(m, O.L_CONST))
    y = np.ones(a.n, complex)
    ref = q.generator_apply(c, q.Generator([a]), y)
    c.close()  # drops the creator's reference; the two operators still pin the context
    a.close()
    b.close()  # last reference: frees the store, then the context
    assert np.all(np.isfinite(ref))


@pytest.mark.parametrize("name,prm", [("kerr", (20, 1.0, 0.01, 2.0, 1.0)), ("kerr", (50, 1.0, 0.01, 2.0, 1.0)),
                                      ("ising", (5, 1, 1.0, 0.2, 1.0, 1))])
def test_cluster_resident_solver_matches_oracle(ctx, monkeypatch, name, prm):
    """K-cluster (operator and state in one cluster's distributed shared memory) against the
    oracle: configs[0] Kerr-20, configs[3] Kerr-50, and a TFIM chain (different gather pattern)."""
    from tests._helpers import e_ops_csr, rho0_vec
    monkeypatch.setenv("QSG_CLUSTER_SOLVE", "1")
    m = O.Model(name, *prm)
    t = np.linspace(0.0, 10.0, 101)
    gen = q.Generator([ctx.op(csr_from_oracle(m, O.L_CONST))])
    dev = q.mesolve(ctx, gen, m.dim, rho0_vec(m), t, e_ops_csr(m))
    ex, st, _ = m.mesolve(t)
    assert normwise_rel(dev["expect"], ex) <= 1e-6
    assert_stats_close(dev["stats"], st)
    monkeypatch.setenv("QSG_CLUSTER_SOLVE", "0")
    ref = q.mesolve(ctx, gen, m.dim, rho0_vec(m), t, e_ops_csr(m))
    assert dev["engine"] == 2 and ref["engine"] != 2
    assert normwise_rel(dev["expect"], ref["expect"]) <= 1e-9


def test_cluster_resident_sesolve_matches_oracle(ctx, monkeypatch):
    """K-cluster in sesolve mode (<psi|E psi> observations gathered across the cluster): closed
    TFIM chain of 9 spins (512 amplitudes, 16 slices), against the oracle's sesolve."""
    monkeypatch.setenv("QSG_CLUSTER_SOLVE", "1")
    m = O.Model("ising", 9, 1, 1.0, 0.2, 0.0, 1)
    t = np.linspace(0.0, 5.0, 51)
    gen = q.Generator([ctx.op(csr_from_oracle(m, O.SE_GEN))])
    dev = q.sesolve(ctx, gen, m.dim, m.psi0(), t, e_ops_csr(m))
    assert dev["engine"] == 2
    ex, st, _ = m.sesolve(t)
    assert normwise_rel(dev["expect"], ex) <= 1e-6
    assert_stats_close(dev["stats"], st)
