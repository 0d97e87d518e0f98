"""The dictionary-coded store's slice-aligned entry order (qsg_capi.cu slice_aligned_order) on
operators built to exercise it: rows whose entries sit at different distances, rows longer than the
64-entry sort limit (their slices keep the CSR order), and two-byte codes (> 256 pairs). The coded
SpMV must equal a CSR reference to rounding (the row sum runs in the aligned order), and the aligned
and CSR-ordered stores must agree with each other."""
import numpy as np
import pytest

import paper_2504_21440_b200 as q

pytestmark = pytest.mark.gpu


def _banded(n, offsets, values, long_rows=(), long_extra=()):
    """CSR with entries at row + offsets (value picked by a fixed rule from `values`), plus extra
    entries on `long_rows` so that they exceed 64 entries."""
    rp, col, val = [0], [], []
    for r in range(n):
        cs = {}
        for j, o in enumerate(offsets):
            c = r + o
            if 0 <= c < n and (r + j) % 5 != 0:  # ragged rows: not every row has every distance
                cs[c] = values[(r * 7 + j) % len(values)]
        if r in long_rows:
            for j, o in enumerate(long_extra):
                c = r + o
                if 0 <= c < n:
                    cs.setdefault(c, values[j % len(values)])
        for c in sorted(cs):
            col.append(c)
            val.append(cs[c])
        rp.append(len(col))
    return np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.complex128)


def _apply(ctx, rp, col, val, n, y, monkeypatch, align):
    monkeypatch.setenv("QSG_COMPRESS_MIN_BYTES", "0")
    monkeypatch.setenv("QSG_SELL_ALIGN", "1" if align else "0")
    op = ctx.op(q.CsrMatrix.from_arrays(rp, col, val, n))
    return q.generator_apply(ctx, q.Generator([op]), y), q.op_storage(op)


def _reference(rp, col, val, y):
    out = np.zeros_like(y)
    for r in range(len(rp) - 1):
        out[r] = np.dot(val[rp[r]:rp[r + 1]], y[col[rp[r]:rp[r + 1]]])
    return out


@pytest.mark.parametrize("case", ["one_byte", "two_byte", "long_rows"])
def test_coded_store_aligned_order(ctx, monkeypatch, case):
    rng = np.random.default_rng(7)
    n = 4096
    offsets = [0, 1, -1, 2, -2, 32, -32, 64, -64, 1024, -1024, 5, -7]
    if case == "two_byte":
        values = [complex(a, b) for a, b in rng.normal(size=(40, 2))]  # > 256 (offset, value) pairs
    else:
        values = [1.0, -0.5j, 0.25 + 0.75j, -2.0]
    long_rows = set(range(96, 128)) | {3000, 3001} if case == "long_rows" else set()
    long_extra = [o for o in range(-200, 201, 3) if o not in offsets] if case == "long_rows" else []
    rp, col, val = _banded(n, offsets, values, long_rows, long_extra)
    y = rng.normal(size=n) + 1j * rng.normal(size=n)
    ref = _reference(rp, col, val, y)
    out_a, info = _apply(ctx, rp, col, val, n, y, monkeypatch, True)
    out_c, _ = _apply(ctx, rp, col, val, n, y, monkeypatch, False)
    assert info[0] == (2 if case == "two_byte" else 1), info
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(out_a - ref)) <= 1e-13 * scale
    assert np.max(np.abs(out_c - ref)) <= 1e-13 * scale
    assert np.max(np.abs(out_a - out_c)) <= 1e-13 * scale


@pytest.mark.parametrize("model,code_bytes", [(("kerr", 20, 1.0, 0.01, 2.0, 1.0), 2), (("ising", 5, 1, 1.0, 0.2, 1.0, 1), 1)])
def test_grid_solve_on_forced_coded_store(ctx, monkeypatch, model, code_bytes):
    """The grid engine's coded stage passes for both code widths (the slice loop is instantiated
    per width): small Liouvillians forced onto the coded store (Kerr-20 has 636 (offset, value)
    pairs, so two-byte codes) against the oracle's full solve."""
    from oracle import oracle as O
    from tests._helpers import csr_from_oracle, e_ops_csr, normwise_rel, rho0_vec
    monkeypatch.setenv("QSG_COMPRESS_MIN_BYTES", "0")
    m = O.Model(*model)
    op = ctx.op(csr_from_oracle(m, O.L_CONST))
    assert q.op_storage(op)[0] == code_bytes
    t = np.linspace(0.0, 2.0, 21)
    r = q.mesolve(ctx, q.Generator([op]), m.dim, rho0_vec(m), t, e_ops_csr(m))
    assert r["engine"] in (0, 1)  # dp5_grid_kernel, cooperative or as one cluster (K-cluster: plain only)
    ref, _, _ = m.mesolve(t)
    for a, b in zip(r["expect"], ref):
        assert normwise_rel(a, b) <= 1e-6
