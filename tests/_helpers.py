"""Test helpers: move oracle-assembled operators into the product's CSR input format."""
import numpy as np

import paper_2504_21440_b200 as q
from oracle import oracle as O


def csr_from_oracle(model: "O.Model", which: int, k: int = 0) -> q.CsrMatrix:
    rp, col, val, n = model.export(which, k)
    return q.CsrMatrix.from_arrays(rp, col, val, n)


def oracle_generator(ctx, model, kind: str):
    """Product Generator built from the oracle's operators: 'me' Liouvillian, 'mc' -iH_eff,
    'se' -iH. Time-dependent terms get PARAM(k) coefficients (model zoo convention)."""
    const = {"me": O.L_CONST, "mc": O.MC_GEN, "se": O.SE_GEN}[kind]
    term = {"me": O.L_TERM, "mc": O.MC_TERM, "se": O.MC_TERM}[kind]
    ops = [ctx.op(csr_from_oracle(model, const))]
    coeffs = [(q.COEFF_CONST, 0, 0, 1.0, 0.0)]
    for k in range(model.n_terms):
        ops.append(ctx.op(csr_from_oracle(model, term, k)))
        coeffs.append(model_coeff(model.name, k))
    return q.Generator(ops, coeffs)


def model_coeff(name, k):
    if name == "driven_cavity_td":
        return (q.COEFF_PARAM_COS, 0, 1, 0.0, 0.0)
    return (q.COEFF_PARAM, k, 0, 0.0, 0.0)


def e_ops_csr(model):
    return [csr_from_oracle(model, O.E_OP, e) for e in range(model.n_eops)]


def rho0_vec(model):
    """Column-stacked density matrix of the model's initial state (ket -> projector)."""
    p = model.psi0()
    d = model.dim
    if model.psi0_is_ket:
        m = np.outer(p, p.conj())
        return m.reshape(-1, order="F").copy()
    return p.copy()


def normwise_rel(a, b):
    """max_k |a_k - b_k| / max_k |b_k| per observable (SURVEY §8d correctness metric)."""
    a = np.atleast_2d(a)
    b = np.atleast_2d(b)
    out = []
    for x, y in zip(a, b):
        den = np.max(np.abs(y))
        out.append(np.max(np.abs(x - y)) / (den if den > 0 else 1.0))
    return max(out)


def assert_stats_close(gpu, ref, restarts=0):
    """Step statistics of the device solve vs the oracle.

    Exact equality is not a valid criterion: accept/reject decisions with err within ulps of 1
    flip under FMA contraction alone (the oracle rebuilt with -ffp-contract=fast -march=native
    reproduces the device's Kerr-20 statistics 141/1/854 exactly, against 141/3/866 without FMA;
    DESIGN.md §6). So: the rhs_evals identity of integrator.hpp:66,103,174 must hold exactly,
    and steps / rejections must agree within a few borderline decisions.
    """
    s, r, e = (int(x) for x in gpu)
    rs, rr, re_ = (int(x) for x in ref)
    assert e == 2 + 6 * (s + r) + restarts, (gpu, ref)
    assert abs(s - rs) <= max(2, int(0.02 * rs)), (gpu, ref)
    assert abs(r - rr) <= max(3, int(0.1 * rr)), (gpu, ref)
