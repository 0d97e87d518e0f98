"""paper_2504_21440_b200 — B200-native (sm_100a) time-evolution engine for the
QuantumToolbox.jl reference hot path (sesolve / mesolve / mcsolve, Liouvillian store,
Dormand-Prince 5(4) integrator, Monte-Carlo trajectories, ensembles and sweeps).

This module is a thin ctypes binding of the in-tree C-ABI library ``lib/libqsim_b200.so``
(declared in ``include/qsg.h`` and ``include/qsg_model.h``). It exists for the test-suite,
``bench.py`` and Python users; the compute path is CUDA only. There is no CPU fallback:
importing works without a GPU, but every solver call raises ``QsgError`` when the library
or a B200 device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSG_LIB_PATH") or os.path.join(_PKG, "lib", "libqsim_b200.so")
_lib = None

P = C.c_void_p
DP = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)

STATUS_NAMES = {
    0: "OK", 1: "KindMismatch", 2: "DimsMismatch", 3: "InvalidSubsystem", 4: "InvalidDimension",
    5: "InvalidIndex", 6: "TooLarge", 7: "IntegrationFailure", 8: "EnsembleFailure",
    9: "SteadyStateFailure", 10: "DfdOverflow", 11: "InvalidGrid", 12: "InvalidScenario",
    100: "CudaError", 101: "NcclError", 102: "OutOfMemory", 103: "Unsupported",
}

COEFF_CONST, COEFF_PARAM, COEFF_PARAM_COS, COEFF_PARAM_SIN = range(4)


class QsgError(RuntimeError):
    """Raised for every non-OK status; ``code`` is the qsg_status value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(code, code)}] {msg}")
        self.code = code


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("rowptr", I32P), ("col", I32P), ("val", DP)]


class _Coeff(C.Structure):
    _fields_ = [("kind", C.c_int32), ("i", C.c_int32), ("j", C.c_int32),
                ("re", C.c_double), ("im", C.c_double)]


class _Gen(C.Structure):
    _fields_ = [("n_terms", C.c_int32), ("ops", C.POINTER(P)), ("coeffs", C.POINTER(_Coeff))]


class _Opts(C.Structure):
    _fields_ = [("method", C.c_int32), ("abstol", C.c_double), ("reltol", C.c_double),
                ("dt_fixed", C.c_double), ("store_states", C.c_int32), ("n_saveat", C.c_int64),
                ("saveat", DP), ("max_steps", C.c_int64)]


class _Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("rejected", C.c_int64), ("rhs_evals", C.c_int64)]


class _Timing(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("total_ms", C.c_double), ("attempts", C.c_int64),
                ("grid_ctas", C.c_int32), ("lanes", C.c_int32), ("store", C.c_int32), ("engine", C.c_int32)]


class _McOut(C.Structure):
    _fields_ = [("per_traj_expect", DP), ("block_sum", DP), ("n_ok", I64P), ("failed", I32P),
                ("fail_time", DP), ("traj_stats", I64P), ("jump_count", I32P),
                ("jump_time", DP), ("jump_channel", I32P), ("jump_capacity", C.c_int64),
                ("n_ranges", C.c_int32), ("range_lo", I64P), ("range_hi", I64P), ("range_sums", DP)]


class _SdeOut(C.Structure):
    _fields_ = [("per_traj_expect", DP), ("block_sum", DP), ("n_ok", C.c_int64), ("w_increments", DP),
                ("w_expectation", DP), ("w_current", DP), ("n_steps", C.c_int64), ("dt", C.c_double)]


def build(verbose: bool = False) -> None:
    """Compile lib/libqsim_b200.so (sm_100a) in-tree."""
    subprocess.run(["make", "-j", str(max(1, os.cpu_count() or 1)), "-C", _PKG] + ([] if verbose else ["-s"]),
                   check=True)


def lib():
    """Load the C-ABI library; raises QsgError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QsgError(100, f"{LIB_PATH} is missing: run paper_2504_21440_b200.build()")
        L = C.CDLL(LIB_PATH)
        L.qsg_last_error.restype = C.c_char_p
        L.qsg_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
        L.qsg_ctx_destroy.argtypes = [P]
        L.qsg_device_info.argtypes = [P, C.POINTER(C.c_int), I64P, C.c_char_p, C.c_int]
        L.qsg_op_create.argtypes = [P, C.POINTER(_Csr), C.POINTER(P)]
        L.qsg_op_destroy.argtypes = [P]
        L.qsg_op_nnz.restype = C.c_int64
        L.qsg_op_nnz.argtypes = [P]
        L.qsg_generator_apply.argtypes = [P, C.POINTER(_Gen), DP, C.c_int32, C.c_double, DP, DP]
        L.qsg_generator_apply_timed.argtypes = [P, C.POINTER(_Gen), DP, C.c_int32, C.c_double, P, P,
                                                C.c_int32, DP]
        for f in (L.qsg_mesolve, L.qsg_sesolve):
            f.argtypes = [P, C.POINTER(_Gen), C.c_int64, P, DP, C.c_int64, C.c_int32, C.POINTER(_Csr),
                          DP, C.c_int32, C.POINTER(_Opts), P, P, C.POINTER(_Stats), C.POINTER(_Timing)]
        L.qsg_mcsolve.argtypes = [P, C.POINTER(_Gen), C.c_int32, C.POINTER(_Csr), C.c_int32,
                                  C.POINTER(_Csr), C.c_int64, DP, DP, C.c_int64, DP, C.c_int32,
                                  C.c_uint64, C.c_int64, C.c_int64, C.POINTER(_Opts),
                                  C.POINTER(_McOut), C.POINTER(_Timing)]
        L.qsg_ensemble_combine.argtypes = [C.c_int32, I64P, I64P, DP, C.c_int64, C.c_int64, DP]
        L.qsg_mesolve_batch.argtypes = [P, C.POINTER(_Gen), C.c_int64, DP, DP, C.c_int64, C.c_int32,
                                        C.POINTER(_Csr), C.c_int64, DP, C.c_int32, C.POINTER(_Opts),
                                        DP, C.POINTER(_Stats), I32P, C.POINTER(_Timing)]
        L.qsg_rng_draw.argtypes = [P, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, DP,
                                   C.POINTER(C.c_uint64)]
        for f in (L.qsg_ssesolve, L.qsg_smesolve):
            f.argtypes = [P, C.POINTER(_Gen), C.c_int64, C.c_int32, C.POINTER(_Csr), C.c_int32, C.POINTER(_Csr),
                          DP, DP, C.c_int64, DP, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                          C.c_int32, C.POINTER(_SdeOut), C.POINTER(_Timing)]
        L.qsg_liouvillian_create.argtypes = [P, C.c_int64, C.POINTER(_Csr), C.c_int32, C.POINTER(_Csr),
                                             C.POINTER(P)]
        L.qsg_liouvillian_export.argtypes = [P, C.c_int64, C.POINTER(_Csr), C.c_int32, C.POINTER(_Csr),
                                             I64P, I32P, I32P, DP]
        _bind_model_api(L)
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise QsgError(rc, lib().qsg_last_error().decode())


def _dp(a):
    return None if a is None else a.ctypes.data_as(DP)


def _ptr(a):
    """Host numpy array or torch CUDA tensor -> void*."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


@dataclass
class CsrMatrix:
    """Host CSR (int32 indices, complex128 values) — the operator-store input format."""
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    n_rows: int
    n_cols: int

    @staticmethod
    def from_arrays(rowptr, col, val, n_rows, n_cols=None):
        return CsrMatrix(np.ascontiguousarray(rowptr, np.int32), np.ascontiguousarray(col, np.int32),
                         np.ascontiguousarray(val, np.complex128), int(n_rows),
                         int(n_rows if n_cols is None else n_cols))

    @property
    def nnz(self):
        return len(self.val)

    def _c(self) -> _Csr:
        return _Csr(self.n_rows, self.n_cols, self.nnz, self.rowptr.ctypes.data_as(I32P),
                    self.col.ctypes.data_as(I32P), self.val.ctypes.data_as(DP))


class Context:
    """One B200 device + stream (qsg_ctx)."""

    def __init__(self, device: int = 0):
        h = P()
        _check(lib().qsg_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        sm = C.c_int(0)
        l2 = C.c_int64(0)
        name = C.create_string_buffer(256)
        _check(lib().qsg_device_info(h, C.byref(sm), C.byref(l2), name, 256))
        self.sm_count, self.l2_bytes, self.name = sm.value, l2.value, name.value.decode()

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.qsg_ctx_destroy(self._h)
            except TypeError:  # interpreter shutdown
                pass
            self._h = None

    def __del__(self):
        self.close()

    def op(self, m: CsrMatrix) -> "Operator":
        return Operator(self, m)

    def liouvillian(self, H, c_ops=()) -> "Operator":
        """Operator store of L = -i[H, .] + sum_k D[c_k] assembled on the device
        (qsg_liouvillian_create; superop.cpp:78-91). H may be None."""
        d, hc, carr = _liou_args(H, c_ops)
        h = P()
        _check(lib().qsg_liouvillian_create(self._h, d, hc, len(c_ops), carr, C.byref(h)))
        return Operator._wrap(self, h, d * d, lib().qsg_op_nnz(h))


def _liou_args(H, c_ops):
    mats = ([H] if H is not None else []) + list(c_ops)
    if not mats:
        raise QsgError(11, "InvalidGrid: need a Hamiltonian or collapse operators")
    d = mats[0].n_rows
    hc = C.byref(H._c()) if H is not None else None
    carr = (_Csr * max(1, len(c_ops)))(*[c._c() for c in c_ops]) if len(c_ops) else None
    return d, hc, carr


def liouvillian_export(ctx: "Context", H, c_ops=()) -> CsrMatrix:
    """L assembled on the device, copied back as host CSR (qsg_liouvillian_export)."""
    d, hc, carr = _liou_args(H, c_ops)
    nnz = C.c_int64(0)
    _check(lib().qsg_liouvillian_export(ctx._h, d, hc, len(c_ops), carr, C.byref(nnz), None, None, None))
    rp = np.empty(d * d + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.complex128)
    _check(lib().qsg_liouvillian_export(ctx._h, d, hc, len(c_ops), carr, C.byref(nnz), rp.ctypes.data_as(I32P),
                                        col.ctypes.data_as(I32P), val.ctypes.data_as(DP)))
    return CsrMatrix(rp, col, val, d * d, d * d)


class Operator:
    """HBM-resident CSR operator (qsg_op)."""

    def __init__(self, ctx: Context, m: CsrMatrix):
        h = P()
        c = m._c()
        _check(lib().qsg_op_create(ctx._h, C.byref(c), C.byref(h)))
        self._h, self.ctx, self.n, self.nnz = h, ctx, m.n_rows, m.nnz

    @classmethod
    def _wrap(cls, ctx, h, n, nnz):
        o = cls.__new__(cls)
        o._h, o.ctx, o.n, o.nnz = h, ctx, int(n), int(nnz)
        return o

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.qsg_op_destroy(self._h)
            except TypeError:  # interpreter shutdown
                pass
            self._h = None

    def __del__(self):
        self.close()


class Generator:
    """G(t) = A0 + sum_k c_k(params, t) A_k (SparseGenerator, evolve.cpp:53-69)."""

    def __init__(self, ops, coeffs=None):
        self.ops = list(ops)
        self.coeffs = list(coeffs) if coeffs is not None else [(COEFF_CONST, 0, 0, 1.0, 0.0)] * len(self.ops)
        self._arr = (P * len(self.ops))(*[o._h for o in self.ops])
        self._carr = (_Coeff * len(self.ops))(*[_Coeff(*c) for c in self.coeffs])
        self._g = _Gen(len(self.ops), C.cast(self._arr, C.POINTER(P)), C.cast(self._carr, C.POINTER(_Coeff)))

    @property
    def n(self):
        return self.ops[0].n


def _opts(abstol, reltol, max_steps, store_states, saveat):
    sv = None if saveat is None else np.ascontiguousarray(saveat, np.float64)
    o = _Opts(0, abstol, reltol, 1e-3, 1 if store_states else 0, 0 if sv is None else len(sv),
              _dp(sv), max_steps)
    return o, sv


def _csr_array(ops):
    arr = (_Csr * max(1, len(ops)))(*[o._c() for o in ops])
    return arr


def _num_saves(n_t, n_e, store_states, saveat):
    if saveat is not None:
        return len(np.union1d([], saveat))
    return n_t if (store_states or n_e == 0) else 0


def _solve(fn, ctx, gen, d, y0, tlist, e_ops, params, abstol, reltol, max_steps, store_states,
           saveat, n_state):
    t = np.ascontiguousarray(tlist, np.float64)
    prm = None if params is None else np.ascontiguousarray(params, np.float64)
    o, sv = _opts(abstol, reltol, max_steps, store_states, saveat)
    eops = _csr_array(e_ops)
    ne = len(e_ops)
    expect = np.zeros(max(1, ne) * len(t), np.complex128)
    nsave = _num_saves(len(t), ne, store_states, saveat)
    states = np.zeros(nsave * n_state, np.complex128) if nsave else None
    st, tm = _Stats(), _Timing()
    y0h = y0 if hasattr(y0, "data_ptr") else np.ascontiguousarray(y0, np.complex128)
    rc = fn(ctx._h, C.byref(gen._g), d, _ptr(y0h), _dp(t), len(t), ne, eops, _dp(prm),
            0 if prm is None else len(prm), C.byref(o), _ptr(expect), _ptr(states), C.byref(st),
            C.byref(tm))
    _check(rc)
    ex = expect[: ne * len(t)].reshape(len(t), ne).T.copy()
    return {
        "expect": ex,
        "stats": (st.steps, st.rejected, st.rhs_evals),
        "states": None if states is None else states.reshape(nsave, n_state),
        "kernel_ms": tm.kernel_ms,
        "attempts": tm.attempts,
        "grid_ctas": tm.grid_ctas, "store": tm.store, "engine": tm.engine,
        "lanes": tm.lanes,
    }


def mesolve(ctx: Context, L: Generator, d: int, rho0, tlist, e_ops=(), params=None, abstol=1e-8,
            reltol=1e-6, max_steps=10_000_000, store_states=False, saveat=None):
    """qsg_mesolve: rho0 is the d x d column-stacked density matrix (length d*d)."""
    return _solve(lib().qsg_mesolve, ctx, L, d, rho0, tlist, list(e_ops), params, abstol, reltol,
                  max_steps, store_states, saveat, d * d)


def sesolve(ctx: Context, G: Generator, d: int, psi0, tlist, e_ops=(), params=None, abstol=1e-8,
            reltol=1e-6, max_steps=10_000_000, store_states=False, saveat=None):
    """qsg_sesolve with generator G = -i H."""
    return _solve(lib().qsg_sesolve, ctx, G, d, psi0, tlist, list(e_ops), params, abstol, reltol,
                  max_steps, store_states, saveat, d)


def generator_apply(ctx: Context, gen: Generator, y, t=0.0, params=None):
    y = np.ascontiguousarray(y, np.complex128)
    out = np.zeros_like(y)
    prm = None if params is None else np.ascontiguousarray(params, np.float64)
    _check(lib().qsg_generator_apply(ctx._h, C.byref(gen._g), _dp(prm), 0 if prm is None else len(prm),
                                     t, _dp(y), _dp(out)))
    return out


def generator_apply_timed(ctx: Context, gen: Generator, y_dev, out_dev, reps=20, t=0.0, params=None):
    """Mean device ms of `reps` back-to-back applies on device (torch) buffers."""
    prm = None if params is None else np.ascontiguousarray(params, np.float64)
    ms = C.c_double(0)
    _check(lib().qsg_generator_apply_timed(ctx._h, C.byref(gen._g), _dp(prm),
                                           0 if prm is None else len(prm), t,
                                           C.c_void_p(y_dev.data_ptr()), C.c_void_p(out_dev.data_ptr()),
                                           reps, C.byref(ms)))
    return ms.value


def mcsolve(ctx: Context, G: Generator, c_ops, e_ops, d: int, psi0, tlist, seed: int, traj_begin: int,
            traj_end: int, params=None, abstol=1e-8, reltol=1e-6, max_steps=10_000_000, jump_cap=256,
            per_traj=True, ranges=None):
    """qsg_mcsolve: trajectories traj_begin..traj_end-1 of the ensemble (RngStream(seed, i)).
    ranges: optional [(lo, hi), ...] positions in the block's completed-trajectory list whose
    pairwise sums are returned as "range_sums" (n_ranges x n_e x n_t)."""
    t = np.ascontiguousarray(tlist, np.float64)
    prm = None if params is None else np.ascontiguousarray(params, np.float64)
    o, _ = _opts(abstol, reltol, max_steps, False, None)
    ne, nt, nb = len(e_ops), len(t), traj_end - traj_begin
    per = np.zeros(nb * ne * nt, np.complex128) if per_traj else None
    bsum = np.zeros(max(1, ne * nt), np.complex128)
    nok = C.c_int64(0)
    failed = np.zeros(nb, np.int32)
    ftime = np.zeros(nb)
    tst = np.zeros(3 * nb, np.int64)
    jcount = np.zeros(nb, np.int32)
    jt = np.zeros(nb * jump_cap)
    jc = np.zeros(nb * jump_cap, np.int32)
    nr = 0 if not ranges else len(ranges)
    rlo = np.ascontiguousarray([r[0] for r in ranges] if nr else [0], np.int64)
    rhi = np.ascontiguousarray([r[1] for r in ranges] if nr else [0], np.int64)
    rs = np.zeros(max(1, nr * ne * nt), np.complex128)
    out = _McOut(_dp(per), _dp(bsum), C.pointer(nok), failed.ctypes.data_as(I32P), _dp(ftime),
                 tst.ctypes.data_as(I64P), jcount.ctypes.data_as(I32P), _dp(jt), jc.ctypes.data_as(I32P),
                 jump_cap, nr, rlo.ctypes.data_as(I64P), rhi.ctypes.data_as(I64P), _dp(rs))
    tm = _Timing()
    y0 = np.ascontiguousarray(psi0, np.complex128)
    _check(lib().qsg_mcsolve(ctx._h, C.byref(G._g), len(c_ops), _csr_array(c_ops), ne, _csr_array(e_ops), d,
                             _dp(y0), _dp(t), nt, _dp(prm), 0 if prm is None else len(prm), seed, traj_begin,
                             traj_end, C.byref(o), C.byref(out), C.byref(tm)))
    jumps = [list(zip(jt[i * jump_cap:i * jump_cap + min(jcount[i], jump_cap)].tolist(),
                      jc[i * jump_cap:i * jump_cap + min(jcount[i], jump_cap)].tolist())) for i in range(nb)]
    return {
        "per_traj": None if per is None else per.reshape(nb, nt, ne).transpose(0, 2, 1).copy(),
        "block_sum": bsum[: ne * nt].reshape(nt, ne).T.copy(),
        "range_sums": [rs[k * ne * nt:(k + 1) * ne * nt].reshape(nt, ne).T.copy() for k in range(nr)],
        "n_ok": nok.value,
        "failed": failed,
        "stats": tst.reshape(nb, 3),
        "njumps": jcount,
        "jumps": jumps,
        "kernel_ms": tm.kernel_ms,
        "attempts": tm.attempts,
        "grid_ctas": tm.grid_ctas,
    }


def _em_steps(t, dt_max):
    span, sp = t[-1] - t[0], t[1] - t[0]
    dtm = dt_max if dt_max > 0 else span / 1e4
    return max(1, int(np.ceil(sp / dtm * (1.0 - 1e-12)))) * (len(t) - 1)


def _sde(fn, ctx, G, sc_ops, e_ops, d, y0, tlist, seed, traj_begin, traj_end, dt_max, store_measurement, params):
    t = np.ascontiguousarray(tlist, np.float64)
    prm = None if params is None else np.ascontiguousarray(params, np.float64)
    ne, nt, nb, nch = len(e_ops), len(t), traj_end - traj_begin, len(sc_ops)
    per = np.zeros(nb * ne * nt, np.complex128)
    bsum = np.zeros(max(1, ne * nt), np.complex128)
    nst = _em_steps(t, dt_max)
    w = [np.zeros(nb * nch * nst) for _ in range(3)] if store_measurement and nch else [None] * 3
    out = _SdeOut(_dp(per), _dp(bsum), 0, _dp(w[0]), _dp(w[1]), _dp(w[2]), 0, 0.0)
    tm = _Timing()
    y = np.ascontiguousarray(y0, np.complex128)
    _check(fn(ctx._h, C.byref(G._g), d, nch, _csr_array(sc_ops), ne, _csr_array(e_ops), _dp(y), _dp(t), nt,
              _dp(prm), 0 if prm is None else len(prm), seed, traj_begin, traj_end, dt_max,
              1 if store_measurement else 0, C.byref(out), C.byref(tm)))
    bs = bsum[: ne * nt].reshape(nt, ne).T.copy()
    res = {"per_traj": per.reshape(nb, nt, ne).transpose(0, 2, 1).copy(), "block_sum": bs, "n_ok": out.n_ok,
           "mean": ensemble_combine([(0, nb)], [bs], out.n_ok) if ne else bs, "n_steps": out.n_steps,
           "dt": out.dt, "kernel_ms": tm.kernel_ms, "grid_ctas": tm.grid_ctas}
    if w[0] is not None:
        sh = lambda x: x.reshape(nb, out.n_steps, nch).transpose(0, 2, 1).copy()
        res["increments"], res["expectation"], res["current"] = (sh(x) for x in w)
    return res


def ssesolve(ctx: Context, G: Generator, sc_ops, e_ops, d: int, psi0, tlist, seed: int, traj_begin: int,
             traj_end: int, dt_max=0.0, store_measurement=False, params=None):
    """qsg_ssesolve: Euler-Maruyama SSE trajectories traj_begin..traj_end-1, G = -iH(t)."""
    return _sde(lib().qsg_ssesolve, ctx, G, sc_ops, e_ops, d, psi0, tlist, seed, traj_begin, traj_end, dt_max,
                store_measurement, params)


def smesolve(ctx: Context, L: Generator, sc_ops, e_ops, d: int, rho0, tlist, seed: int, traj_begin: int,
             traj_end: int, dt_max=0.0, store_measurement=False, params=None):
    """qsg_smesolve: L includes the dissipators of c_ops and sc_ops; rho0 column-stacked d x d."""
    return _sde(lib().qsg_smesolve, ctx, L, sc_ops, e_ops, d, rho0, tlist, seed, traj_begin, traj_end, dt_max,
                store_measurement, params)


def ensemble_combine(block_ranges, block_sums, n_ok_total):
    """qsg_ensemble_combine: deterministic pairwise combine of per-block sums (mean)."""
    b = np.ascontiguousarray([r[0] for r in block_ranges], np.int64)
    e = np.ascontiguousarray([r[1] for r in block_ranges], np.int64)
    sums = np.ascontiguousarray(np.stack([np.asarray(s).T.reshape(-1) for s in block_sums]), np.complex128)
    nv = sums.shape[1]
    mean = np.zeros(nv, np.complex128)
    _check(lib().qsg_ensemble_combine(len(b), b.ctypes.data_as(I64P), e.ctypes.data_as(I64P), _dp(sums), nv,
                                      n_ok_total, _dp(mean)))
    shape = np.asarray(block_sums[0]).shape
    return mean.reshape(shape[1], shape[0]).T.copy()


def mesolve_batch(ctx: Context, L: Generator, d: int, rho0, tlist, e_ops, params, abstol=1e-8, reltol=1e-6,
                  max_steps=10_000_000):
    """qsg_mesolve_batch: one mesolve per row of `params` (n_points x n_params)."""
    t = np.ascontiguousarray(tlist, np.float64)
    prm = np.ascontiguousarray(params, np.float64)
    npts, npar = prm.shape
    o, _ = _opts(abstol, reltol, max_steps, False, None)
    ne, nt = len(e_ops), len(t)
    ex = np.zeros(npts * ne * nt, np.complex128)
    st = (_Stats * npts)()
    status = np.zeros(npts, np.int32)
    tm = _Timing()
    y0 = np.ascontiguousarray(rho0, np.complex128)
    _check(lib().qsg_mesolve_batch(ctx._h, C.byref(L._g), d, _dp(y0), _dp(t), nt, ne, _csr_array(e_ops), npts,
                                   _dp(prm), npar, C.byref(o), _dp(ex), st, status.ctypes.data_as(I32P),
                                   C.byref(tm)))
    return {
        "expect": ex.reshape(npts, nt, ne).transpose(0, 2, 1).copy(),
        "stats": np.array([(s.steps, s.rejected, s.rhs_evals) for s in st]),
        "status": status,
        "kernel_ms": tm.kernel_ms,
        "attempts": tm.attempts,
        "grid_ctas": tm.grid_ctas,
    }


def rng_draw(ctx: Context, seed: int, stream: int, kind: int, n: int):
    if kind == 0:
        out = np.zeros(n, np.uint64)
        _check(lib().qsg_rng_draw(ctx._h, seed, stream, 0, n, None,
                                  out.ctypes.data_as(C.POINTER(C.c_uint64))))
    else:
        out = np.zeros(n, np.float64)
        _check(lib().qsg_rng_draw(ctx._h, seed, stream, kind, n, _dp(out), None))
    return out


def _bind_model_api(L):
    """qsg_model_* entry points (include/qsg_model.h)."""
    L.qsg_model_create.argtypes = [C.c_char_p, DP, C.c_int32, C.POINTER(P)]
    L.qsg_model_destroy.argtypes = [P]
    L.qsg_model_info.argtypes = [P, I64P]
    L.qsg_model_export.restype = C.c_int64
    L.qsg_model_export.argtypes = [P, C.c_int32, C.c_int32, I64P, I32P, I32P, DP]
    L.qsg_model_psi0.argtypes = [P, DP]
    L.qsg_model_default_params.argtypes = [P, DP]
    for f in (L.qsg_model_mesolve, L.qsg_model_sesolve):
        f.argtypes = [P, C.c_int32, DP, C.c_int64, DP, C.c_int32, C.POINTER(_Opts), DP, I64P, DP]
    L.qsg_model_ssesolve.argtypes = [P, C.c_int32, DP, C.c_int64, DP, C.c_int32, C.c_uint64, C.c_int32,
                                     C.c_double, C.c_int32, DP, DP, DP, DP, DP, I64P, DP, DP]
    L.qsg_model_smesolve.argtypes = [P, C.c_int32, C.c_int32, DP, C.c_int64, DP, C.c_int32, C.c_uint64,
                                     C.c_int32, C.c_double, C.c_int32, DP, DP, DP, DP, DP, I64P, DP, DP]
    L.qsg_model_mcsolve.argtypes = [P, C.c_int32, I32P, DP, C.c_int64, DP, C.c_int32, C.c_uint64, C.c_int32,
                                    C.POINTER(_Opts), DP, DP, I64P, I32P, DP, I32P, C.c_int32, I32P, DP, DP]


# export selectors of qsg_model_export (include/qsg_model.h)
SEL_H_CONST, SEL_H_TERM, SEL_C_OP, SEL_E_OP, SEL_L_CONST, SEL_L_TERM, SEL_MC_GEN, SEL_MC_TERM, SEL_SE_GEN = range(9)


class Model:
    """A BASELINE model assembled by the product's C++ host API (qsim::*, qsg_model.h)."""

    def __init__(self, name: str, *params: float):
        p = np.ascontiguousarray(params, np.float64)
        h = P()
        _check(lib().qsg_model_create(name.encode(), _dp(p), len(p), C.byref(h)))
        self._h = h
        self.name = name
        info = np.zeros(6, np.int64)
        lib().qsg_model_info(h, info.ctypes.data_as(I64P))
        self.dim, self.n_terms, self.n_cops, self.n_eops, ket, npar = (int(x) for x in info)
        self.psi0_is_ket = bool(ket)
        self.default_params = np.zeros(npar)
        if npar:
            lib().qsg_model_default_params(h, _dp(self.default_params))

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.qsg_model_destroy(self._h)
            except TypeError:
                pass
            self._h = None

    def __del__(self):
        self.close()

    def export(self, which: int, k: int = 0) -> CsrMatrix:
        nrows = C.c_int64(0)
        nnz = lib().qsg_model_export(self._h, which, k, C.byref(nrows), None, None, None)
        if nnz < 0:
            raise QsgError(11, lib().qsg_last_error().decode())
        rp = np.zeros(nrows.value + 1, np.int32)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.complex128)
        lib().qsg_model_export(self._h, which, k, C.byref(nrows), rp.ctypes.data_as(I32P),
                               col.ctypes.data_as(I32P), val.ctypes.data_as(DP))
        return CsrMatrix(rp, col, val, nrows.value, nrows.value)

    def psi0(self) -> np.ndarray:
        out = np.zeros(self.dim if self.psi0_is_ket else self.dim * self.dim, np.complex128)
        lib().qsg_model_psi0(self._h, out.ctypes.data_as(DP))
        return out

    def _solve(self, f, device, tlist, params, abstol, reltol, max_steps):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        o, _ = _opts(abstol, reltol, max_steps, False, None)
        ex = np.zeros(self.n_eops * len(t), np.complex128)
        st = np.zeros(3, np.int64)
        ms = C.c_double(0)
        _check(f(self._h, device, _dp(t), len(t), _dp(prm), len(prm), C.byref(o), _dp(ex),
                 st.ctypes.data_as(I64P), C.byref(ms)))
        return {"expect": ex.reshape(len(t), self.n_eops).T.copy(), "stats": tuple(int(x) for x in st),
                "kernel_ms": ms.value}

    def mesolve(self, tlist, params=None, device=0, abstol=1e-8, reltol=1e-6, max_steps=10_000_000):
        """qsim::mesolve(H, psi0, tlist, c_ops, e_ops, params, options) on the device."""
        return self._solve(lib().qsg_model_mesolve, device, tlist, params, abstol, reltol, max_steps)

    def sesolve(self, tlist, params=None, device=0, abstol=1e-8, reltol=1e-6, max_steps=10_000_000):
        return self._solve(lib().qsg_model_sesolve, device, tlist, params, abstol, reltol, max_steps)

    def _sde(self, sme, n_det, tlist, seed, ntraj, dt_max, store_measurement, device, params):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        ne, nt = self.n_eops, len(t)
        nch = self.n_cops - (n_det if sme else 0)
        mean = np.zeros(ne * nt, np.complex128)
        per = np.zeros(ntraj * ne * nt, np.complex128)
        nst = _em_steps(t, dt_max)
        w = [np.zeros(ntraj * nch * nst) for _ in range(3)] if store_measurement and nch else [None] * 3
        ns = C.c_int64(0)
        dt = C.c_double(0)
        ms = C.c_double(0)
        tail = (_dp(t), len(t), _dp(prm), len(prm), seed, ntraj, dt_max, 1 if store_measurement else 0, _dp(mean),
                _dp(per), *[_dp(x) for x in w], C.byref(ns), C.byref(dt), C.byref(ms))
        if sme:
            _check(lib().qsg_model_smesolve(self._h, device, n_det, *tail))
        else:
            _check(lib().qsg_model_ssesolve(self._h, device, *tail))
        out = {"mean": mean.reshape(nt, ne).T.copy(), "per_traj": per.reshape(ntraj, nt, ne).transpose(0, 2, 1).copy(),
               "device_ms": ms.value}
        if w[0] is not None:
            sh = lambda x: x.reshape(ntraj, ns.value, nch).transpose(0, 2, 1).copy()
            out["increments"], out["expectation"], out["current"] = (sh(x) for x in w)
            out["dt"] = dt.value
        return out

    def ssesolve(self, tlist, seed, ntraj, dt_max=0.0, store_measurement=False, device=0, params=None):
        """qsim::ssesolve with every model c_op as a measurement channel (trajectories.cpp:367-393)."""
        return self._sde(False, 0, tlist, seed, ntraj, dt_max, store_measurement, device, params)

    def smesolve(self, tlist, seed, ntraj, n_det=0, dt_max=0.0, store_measurement=False, device=0, params=None):
        """qsim::smesolve: model c_ops[:n_det] unmonitored, the rest measured (trajectories.cpp:474-503)."""
        return self._sde(True, n_det, tlist, seed, ntraj, dt_max, store_measurement, device, params)

    def mcsolve(self, tlist, seed, ntraj, devices=(0,), params=None, abstol=1e-8, reltol=1e-6,
                max_steps=10_000_000, jump_cap=256):
        """qsim::mcsolve (trajectories sharded over `devices` in-process)."""
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        o, _ = _opts(abstol, reltol, max_steps, False, None)
        ne, nt = self.n_eops, len(t)
        mean = np.zeros(ne * nt, np.complex128)
        per = np.zeros(ntraj * ne * nt, np.complex128)
        st = np.zeros(3, np.int64)
        nj = np.zeros(ntraj, np.int32)
        jt = np.zeros(ntraj * jump_cap)
        jc = np.zeros(ntraj * jump_cap, np.int32)
        nf = C.c_int32(0)
        ms = C.c_double(0)
        sd = np.zeros(ne * nt)
        dv = np.ascontiguousarray(devices, np.int32)
        _check(lib().qsg_model_mcsolve(self._h, len(dv), dv.ctypes.data_as(I32P), _dp(t), nt, _dp(prm), len(prm),
                                       seed, ntraj, C.byref(o), _dp(mean), _dp(per), st.ctypes.data_as(I64P),
                                       nj.ctypes.data_as(I32P), _dp(jt), jc.ctypes.data_as(I32P), jump_cap,
                                       C.byref(nf), C.byref(ms), _dp(sd)))
        jumps = [list(zip(jt[i * jump_cap:i * jump_cap + min(nj[i], jump_cap)].tolist(),
                          jc[i * jump_cap:i * jump_cap + min(nj[i], jump_cap)].tolist())) for i in range(ntraj)]
        return {"mean": mean.reshape(nt, ne).T.copy(), "per_traj": per.reshape(ntraj, nt, ne).transpose(0, 2, 1).copy(),
                "stats": tuple(int(x) for x in st), "njumps": nj, "jumps": jumps, "failed": nf.value,
                "kernel_ms": ms.value, "stddev": sd.reshape(nt, ne).T.copy()}


def op_storage(op: "Operator"):
    """(code_bytes, dictionary size) of an operator store: 0 = plain SELL-32, 1/2 = coded."""
    L = lib()
    L.qsg_op_code_bytes.restype = C.c_int32
    L.qsg_op_code_bytes.argtypes = [P]
    L.qsg_op_dict_size.restype = C.c_int32
    L.qsg_op_dict_size.argtypes = [P]
    return L.qsg_op_code_bytes(op._h), L.qsg_op_dict_size(op._h)


STORE_NAMES = {0: "plain", 1: "coded8", 2: "coded16", 3: "key-aligned"}


def op_store_info(op: "Operator") -> dict:
    """qsg_op_store_info: the stores an operator carries and the bytes one SpMV reads from each."""
    L = lib()
    L.qsg_op_store_info.argtypes = [P, I64P]
    v = (C.c_int64 * 8)()
    _check(L.qsg_op_store_info(op._h, v))
    return {"store": STORE_NAMES[int(v[0])], "plain_bytes": int(v[1]), "coded_bytes": int(v[2]),
            "ka_bytes": int(v[3]), "ka_values": int(v[4]), "ka_positions": int(v[5]), "coded_pairs": int(v[6]),
            "ka_slot_bytes": int(v[7])}
