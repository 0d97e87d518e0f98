"""On-device Liouvillian assembly (qsg_liouvillian_create / _export) against the oracle's
liouvillian (superop.cpp:78-91 restated in oracle/qsim_oracle.cpp): the same sparsity pattern
(explicit zeros included) and the same values, entry for entry (== on every component), for every
model of the zoo, the time-dependent term Liouvillians (evolve.cpp:39-47) and full TFIM-10
(configs[1]); then a solve on the device-built store matches the oracle.
"""
import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O
from tests._helpers import assert_stats_close, csr_from_oracle, normwise_rel

pytestmark = pytest.mark.gpu

MODELS = [
    ("kerr", (20, 1.0, 0.01, 2.0, 1.0)),
    ("kerr", (50, 1.0, 0.01, 2.0, 1.0)),
    ("ising", (3, 2, 1.0, 0.2, 1.0, 1)),
    ("ising", (7, 1, 1.0, 0.2, 1.0, 0)),
    ("jc", (10, 1.0, 1.0, 0.1, 0.05, 0.05)),
    ("damped_cavity", (10, 1.0, 0.1, 3)),
    ("coupled_kerr", (4, 0.1, 0.5, 1.0)),
    ("decay2", (0.8,)),
    ("driven_cavity_td", (14, 0.4)),
]


def _assert_same_csr(dev, rp, col, val):
    assert np.array_equal(dev.rowptr, rp)
    assert np.array_equal(dev.col, col)
    assert np.array_equal(dev.val.real, val.real) and np.array_equal(dev.val.imag, val.imag)


@pytest.mark.parametrize("name,params", MODELS)
def test_liouvillian_matches_oracle(ctx, name, params):
    m = O.Model(name, *params)
    H = csr_from_oracle(m, O.H_CONST)
    cops = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    dev = q.liouvillian_export(ctx, H, cops)
    rp, col, val, n = m.export(O.L_CONST)
    assert dev.n_rows == n
    _assert_same_csr(dev, rp, col, val)
    for k in range(m.n_terms):  # -i(spre(h_k) - spost(h_k)) of each time-dependent term
        devk = q.liouvillian_export(ctx, csr_from_oracle(m, O.H_TERM, k), [])
        _assert_same_csr(devk, *m.export(O.L_TERM, k)[:3])


def test_dissipator_only(ctx):
    m = O.Model("decay2", 0.8)
    cops = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    dev = q.liouvillian_export(ctx, None, cops)
    y = np.random.default_rng(3).standard_normal(dev.n_rows) + 0j
    op = ctx.liouvillian(None, cops)
    full = q.generator_apply(ctx, q.Generator([op]), y)
    ref = np.zeros_like(y)
    for r in range(dev.n_rows):
        for p in range(dev.rowptr[r], dev.rowptr[r + 1]):
            ref[r] += dev.val[p] * y[dev.col[p]]
    assert np.max(np.abs(full - ref)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))


def test_dims_mismatch(ctx):
    a = csr_from_oracle(O.Model("kerr", 4, 1.0, 0.01, 0.5, 1.0), O.H_CONST)
    b = csr_from_oracle(O.Model("kerr", 5, 1.0, 0.01, 0.5, 1.0), O.C_OP, 0)
    with pytest.raises(q.QsgError) as ei:
        ctx.liouvillian(a, [b])
    assert ei.value.code == 2


def test_tfim10_device_liouvillian(ctx):
    """configs[1]: the 24.6M-entry Liouvillian built on the device equals the reference's, and the
    first 0.5 time units of the solve on it match the oracle."""
    m = O.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
    H = csr_from_oracle(m, O.H_CONST)
    cops = [csr_from_oracle(m, O.C_OP, k) for k in range(m.n_cops)]
    dev = q.liouvillian_export(ctx, H, cops)
    _assert_same_csr(dev, *m.export(O.L_CONST)[:3])
    op = ctx.liouvillian(H, cops)
    assert q.op_storage(op) == (1, 201)
    eops = [csr_from_oracle(m, O.E_OP, k) for k in range(m.n_eops)]
    psi = m.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
    t = np.linspace(0.0, 0.5, 6)
    res = q.mesolve(ctx, q.Generator([op]), m.dim, rho0, t, eops)
    m.prepare_liouvillian()
    ex, st = m.mesolve_prepared(t)
    assert normwise_rel(res["expect"], ex) <= 1e-6
    assert_stats_close(res["stats"], st)


@pytest.mark.parametrize("name,params,prm", [
    ("kerr", (20, 1.0, 0.01, 2.0, 1.0), None),
    ("ising", (3, 2, 1.0, 0.2, 1.0, 1), None),
    ("jc", (10, 1.0, 1.0, 0.1, 0.05, 0.05), None),
    ("driven_cavity_td", (14, 0.4), np.array([0.25, 1.3])),
    ("coupled_kerr", (4, 0.1, 0.5, 1.0), np.array([0.5, 0.9])),
])
def test_cpp_mesolve_device_liouvillian(name, params, prm):
    """qsim::mesolve(H, rho0, tlist, c_ops, e_ops) of the C++ host API assembles L and its
    time-dependent term Liouvillians on the device; results match the oracle's mesolve."""
    t = np.linspace(0.0, 6.0, 61)
    dev = q.Model(name, *params).mesolve(t, params=prm)
    om = O.Model(name, *params)
    ex, st, _ = om.mesolve(t, params=prm)
    assert normwise_rel(dev["expect"], ex) <= 1e-6
    assert_stats_close(dev["stats"], st)
