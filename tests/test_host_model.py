"""CPU tests of the product's host model assembly (qsim C++ API via qsg_model.h) against the
oracle's restatement of the reference (factories.cpp / superop.cpp / qobj.cpp on Eigen
semantics). Operators must be bit-identical: same pattern, same complex128 values.
"""
import numpy as np
import pytest

import paper_2504_21440_b200 as q
from oracle import oracle as O

MODELS = [
    ("kerr", (20, 1.0, 0.01, 2.0, 1.0)),
    ("kerr", (7, -0.3, 0.2, 0.7, 0.4)),
    ("coupled_kerr", (4, 0.1, 0.5, 1.0)),
    ("ising", (3, 2, 1.0, 0.2, 1.0, 1)),
    ("ising", (2, 2, 0.9, 0.4, 0.2, 1)),
    ("ising", (5, 1, 1.0, 0.2, 1.0, 0)),
    ("jc", (6, 1.0, 1.0, 0.1, 0.01, 0.01)),
    ("jc_sse", (6, 1.0, 1.0, 0.1, 0.3)),
    ("jc_sme", (5, 1.0, 1.0, 0.2, 0.4, 0.2, 0.1)),
    ("damped_cavity", (10, 1.0, 0.1, 3)),
    ("decay2", (0.25,)),
    ("driven_cavity_td", (14, 0.4)),
]


def _same(a: q.CsrMatrix, b):
    rp, col, val, n = b
    assert a.n_rows == n
    assert np.array_equal(a.rowptr, rp)
    assert np.array_equal(a.col, col)
    # bitwise on both components
    assert np.array_equal(a.val.view(np.float64), val.view(np.float64)), np.max(np.abs(a.val - val))


@pytest.mark.parametrize("name,params", MODELS)
def test_model_operators_bit_identical(name, params):
    pm = q.Model(name, *params)
    om = O.Model(name, *params)
    assert (pm.dim, pm.n_terms, pm.n_cops, pm.n_eops) == (om.dim, om.n_terms, om.n_cops, om.n_eops)
    _same(pm.export(q.SEL_H_CONST), om.export(O.H_CONST))
    _same(pm.export(q.SEL_L_CONST), om.export(O.L_CONST))
    _same(pm.export(q.SEL_MC_GEN), om.export(O.MC_GEN))
    _same(pm.export(q.SEL_SE_GEN), om.export(O.SE_GEN))
    for k in range(pm.n_cops):
        _same(pm.export(q.SEL_C_OP, k), om.export(O.C_OP, k))
    for k in range(pm.n_eops):
        _same(pm.export(q.SEL_E_OP, k), om.export(O.E_OP, k))
    for k in range(pm.n_terms):
        _same(pm.export(q.SEL_H_TERM, k), om.export(O.H_TERM, k))
        _same(pm.export(q.SEL_L_TERM, k), om.export(O.L_TERM, k))
        _same(pm.export(q.SEL_MC_TERM, k), om.export(O.MC_TERM, k))
    assert np.array_equal(pm.psi0(), om.psi0())


def test_tfim10_liouvillian_size_and_identity():
    """BASELINE config 2 operator: n = 4^10 rows, 24,641,536 stored entries, bit-identical."""
    pm = q.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
    L = pm.export(q.SEL_L_CONST)
    assert L.n_rows == 4 ** 10 and L.nnz == 24_641_536
    rl = np.diff(L.rowptr)
    assert rl.min() == 21 and rl.max() == 31


def test_tfim14_mc_generator_is_15_per_row():
    """BASELINE config 3 generator -i H_eff: 16,384 rows, exactly 15 entries per row."""
    pm = q.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
    G = pm.export(q.SEL_MC_GEN)
    assert G.n_rows == 16384 and np.all(np.diff(G.rowptr) == 15)
    om = O.Model("ising", 14, 1, 1.0, 0.2, 1.0, 1)
    _same(G, om.export(O.MC_GEN))


def test_unknown_model_and_missing_params():
    with pytest.raises(q.QsgError) as e:
        q.Model("nope", 1.0)
    assert e.value.code == 12
    with pytest.raises(q.QsgError):
        q.Model("kerr", 5)


def test_ising_cap_matches_reference():
    """factories.cpp:208 caps the reference lattice at 12 sites (test_factories.cpp:177)."""
    assert O.ising_capped_error(4, 4) == 1 + 5  # TooLarge
    assert O.ising_capped_error(3, 4) == 0
