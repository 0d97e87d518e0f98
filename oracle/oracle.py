"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle (oracle/liboracle.so).

Imported only by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs, always as the checker or the CPU baseline, never as the thing
measured or shipped. See oracle/qsim_oracle.hpp for the reference provenance.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

P = C.c_void_p
DP = C.POINTER(C.c_double)
LP = C.POINTER(C.c_long)
IP = C.POINTER(C.c_int)


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_model_new.restype = P
        L.orc_model_new.argtypes = [C.c_char_p, DP, C.c_int]
        L.orc_model_free.argtypes = [P]
        L.orc_model_dim.restype = C.c_long
        L.orc_model_dim.argtypes = [P]
        L.orc_model_count.argtypes = [P, C.c_int]
        L.orc_model_default_params.argtypes = [P, DP]
        L.orc_model_export.restype = C.c_long
        L.orc_model_export.argtypes = [P, C.c_int, C.c_int, LP, IP, IP, DP]
        L.orc_model_psi0.argtypes = [P, DP]
        for f in (L.orc_mesolve, L.orc_sesolve):
            f.argtypes = [P, DP, C.c_int, DP, C.c_int, DP, C.c_int, DP, DP, LP, DP]
        L.orc_ssesolve.argtypes = [P, DP, C.c_int, DP, C.c_int, C.c_ulonglong, C.c_int, C.c_int, C.c_double,
                                   C.c_int, DP, DP, DP, DP, DP, LP, DP]
        L.orc_smesolve.argtypes = [P, C.c_int, DP, C.c_int, DP, C.c_int, C.c_ulonglong, C.c_int, C.c_int,
                                   C.c_double, C.c_int, DP, DP, DP, DP, DP, LP, DP]
        L.orc_mcsolve.argtypes = [P, DP, C.c_int, DP, C.c_int, DP, C.c_ulonglong, C.c_int, C.c_int,
                                  DP, DP, LP, IP, DP, IP, C.c_int, IP]
        L.orc_generator_apply.argtypes = [P, C.c_int, C.c_double, DP, C.c_int, DP, DP]
        L.orc_rng.argtypes = [C.c_ulonglong, C.c_ulonglong, C.c_int, C.c_int, DP,
                              C.POINTER(C.c_ulonglong)]
        L.orc_splitmix64.restype = C.c_ulonglong
        L.orc_splitmix64.argtypes = [C.POINTER(C.c_ulonglong)]
        L.orc_ising_capped.argtypes = [C.c_int, C.c_int]
        L.orc_model_prepare_liouvillian.argtypes = [P]
        L.orc_mesolve_prepared.argtypes = [P, DP, C.c_int, DP, C.c_int, DP, DP, LP]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_threads.restype = C.c_int
        _lib = L
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(DP)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


# export selectors (oracle_capi.cpp: pick)
H_CONST, H_TERM, C_OP, E_OP, L_CONST, L_TERM, MC_GEN, MC_TERM, SE_GEN = range(9)


class Model:
    """A model assembled by the oracle's restated factories/superop code."""

    def __init__(self, name: str, *params: float):
        p = np.ascontiguousarray(params, dtype=np.float64)
        self._h = lib().orc_model_new(name.encode(), _dp(p), len(p))
        if not self._h:
            raise OracleError(-1, lib().orc_last_error().decode())
        self.name = name
        self.dim = lib().orc_model_dim(self._h)
        self.n_terms = lib().orc_model_count(self._h, 0)
        self.n_cops = lib().orc_model_count(self._h, 1)
        self.n_eops = lib().orc_model_count(self._h, 2)
        self.psi0_is_ket = bool(lib().orc_model_count(self._h, 3))
        npar = lib().orc_model_count(self._h, 4)
        self.default_params = np.zeros(npar)
        if npar:
            lib().orc_model_default_params(self._h, _dp(self.default_params))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.orc_model_free(self._h)
            except TypeError:  # interpreter shutdown
                pass
            self._h = None

    def export(self, which: int, k: int = 0):
        """Returns (rowptr int32, col int32, val complex128, nrows) CSR of the operator."""
        nrows = C.c_long(0)
        nnz = lib().orc_model_export(self._h, which, k, C.byref(nrows), None, None, None)
        if nnz < 0:
            raise OracleError(-1, lib().orc_last_error().decode())
        rowptr = np.zeros(nrows.value + 1, np.int32)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.complex128)
        lib().orc_model_export(self._h, which, k, C.byref(nrows), rowptr.ctypes.data_as(IP),
                               col.ctypes.data_as(IP), val.ctypes.data_as(DP))
        return rowptr, col, val, nrows.value

    def psi0(self) -> np.ndarray:
        n = self.dim if self.psi0_is_ket else self.dim * self.dim
        out = np.zeros(n, np.complex128)
        lib().orc_model_psi0(self._h, out.ctypes.data_as(DP))
        return out

    def _opts(self, abstol, reltol, max_steps, store_states):
        return np.array([abstol, reltol, float(max_steps), 1.0 if store_states else 0.0])

    def _solve(self, fn, tlist, params, abstol, reltol, max_steps, store_states, saveat):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        opts = self._opts(abstol, reltol, max_steps, store_states)
        sv = None if saveat is None else np.ascontiguousarray(saveat, np.float64)
        expect = np.zeros(self.n_eops * len(t), np.complex128)
        stats = np.zeros(3, np.int64)
        nsave = 0
        if store_states or self.n_eops == 0 or sv is not None:
            nsave = len(sv) if sv is not None else len(t)
        ssz = self.dim if fn == "se" else self.dim * self.dim
        states = np.zeros(nsave * ssz, np.complex128) if nsave else None
        f = lib().orc_mesolve if fn == "me" else lib().orc_sesolve
        rc = f(self._h, _dp(t), len(t), _dp(prm), len(prm), _dp(opts), 0 if sv is None else len(sv),
               _dp(sv), expect.ctypes.data_as(DP), stats.ctypes.data_as(LP),
               None if states is None else states.ctypes.data_as(DP))
        _check(rc)
        ex = expect.reshape(len(t), self.n_eops).T.copy()  # col-major n_e x n_t
        st = None if states is None else states.reshape(nsave, ssz)
        return ex, stats, st

    def mesolve(self, tlist, params=None, abstol=1e-8, reltol=1e-6, max_steps=10_000_000,
                store_states=False, saveat=None):
        return self._solve("me", tlist, params, abstol, reltol, max_steps, store_states, saveat)

    def sesolve(self, tlist, params=None, abstol=1e-8, reltol=1e-6, max_steps=10_000_000,
                store_states=False, saveat=None):
        return self._solve("se", tlist, params, abstol, reltol, max_steps, store_states, saveat)

    def prepare_liouvillian(self):
        """Build L once (the reference's liouvillian()); timed separately from the solve."""
        _check(lib().orc_model_prepare_liouvillian(self._h))

    def mesolve_prepared(self, tlist, params=None, abstol=1e-8, reltol=1e-6, max_steps=10_000_000):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        opts = self._opts(abstol, reltol, max_steps, False)
        expect = np.zeros(self.n_eops * len(t), np.complex128)
        stats = np.zeros(3, np.int64)
        _check(lib().orc_mesolve_prepared(self._h, _dp(t), len(t), _dp(prm), len(prm), _dp(opts),
                                          expect.ctypes.data_as(DP), stats.ctypes.data_as(LP)))
        return expect.reshape(len(t), self.n_eops).T.copy(), stats

    def _sde(self, sme, n_det, tlist, seed, ntraj, dt_max, store_measurement, n_threads, params):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        ne, nt = self.n_eops, len(t)
        n_ch = self.n_cops - (n_det if sme else 0)
        mean = np.zeros(ne * nt, np.complex128)
        per = np.zeros(ntraj * ne * nt, np.complex128)
        nsteps = C.c_long(0)
        dt = C.c_double(0)
        # grid size first (no measurement buffers), then the real run
        span = t[-1] - t[0]
        sp = t[1] - t[0]
        dtm = dt_max if dt_max > 0 else span / 1e4
        sub = max(1, int(np.ceil(sp / dtm * (1.0 - 1e-12))))
        n_steps = sub * (nt - 1)
        w = [np.zeros(ntraj * n_ch * n_steps) for _ in range(3)] if store_measurement else [None] * 3
        args = (_dp(t), nt, _dp(prm), len(prm), seed, ntraj, n_threads, dt_max, 1 if store_measurement else 0,
                mean.ctypes.data_as(DP), per.ctypes.data_as(DP), *[_dp(x) for x in w], C.byref(nsteps), C.byref(dt))
        rc = lib().orc_smesolve(self._h, n_det, *args) if sme else lib().orc_ssesolve(self._h, *args)
        _check(rc)
        out = {"mean": mean.reshape(nt, ne).T.copy(),
               "per_traj": per.reshape(ntraj, nt, ne).transpose(0, 2, 1).copy(),
               "n_steps": nsteps.value, "dt": dt.value}
        if store_measurement:
            sh = lambda x: x.reshape(ntraj, nsteps.value, n_ch).transpose(0, 2, 1).copy()
            out["increments"], out["expectation"], out["current"] = (sh(x) for x in w)
        return out

    def ssesolve(self, tlist, seed, ntraj, dt_max=0.0, store_measurement=False, n_threads=0, params=None):
        """trajectories.cpp:367-393 with every model c_op as a measurement channel."""
        return self._sde(False, 0, tlist, seed, ntraj, dt_max, store_measurement, n_threads, params)

    def smesolve(self, tlist, seed, ntraj, n_det=0, dt_max=0.0, store_measurement=False, n_threads=0,
                 params=None):
        """trajectories.cpp:474-503: model c_ops[:n_det] deterministic, the rest measured."""
        return self._sde(True, n_det, tlist, seed, ntraj, dt_max, store_measurement, n_threads, params)

    def mcsolve(self, tlist, seed, ntraj, n_threads=0, params=None, abstol=1e-8, reltol=1e-6,
                max_steps=10_000_000, jcap=512):
        t = np.ascontiguousarray(tlist, np.float64)
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        opts = self._opts(abstol, reltol, max_steps, False)
        ne, nt = self.n_eops, len(t)
        mean = np.zeros(ne * nt, np.complex128)
        per = np.zeros(ntraj * ne * nt, np.complex128)
        stats = np.zeros(3 * ntraj, np.int64)
        nj = np.zeros(ntraj, np.int32)
        jt = np.zeros(ntraj * jcap, np.float64)
        jc = np.zeros(ntraj * jcap, np.int32)
        failed = np.zeros(ntraj, np.int32)
        rc = lib().orc_mcsolve(self._h, _dp(t), nt, _dp(prm), len(prm), _dp(opts), seed, ntraj,
                               n_threads, mean.ctypes.data_as(DP), per.ctypes.data_as(DP),
                               stats.ctypes.data_as(LP), nj.ctypes.data_as(IP), _dp(jt),
                               jc.ctypes.data_as(IP), jcap, failed.ctypes.data_as(IP))
        _check(rc)
        jumps = []
        for i in range(ntraj):
            k = min(nj[i], jcap)
            jumps.append(list(zip(jt[i * jcap:i * jcap + k].tolist(), jc[i * jcap:i * jcap + k].tolist())))
        return {
            "mean": mean.reshape(nt, ne).T.copy(),
            "per_traj": per.reshape(ntraj, nt, ne).transpose(0, 2, 1).copy(),
            "stats": stats.reshape(ntraj, 3),
            "njumps": nj,
            "jumps": jumps,
            "failed": failed,
        }

    def generator_apply(self, which, t, y, params=None):
        prm = np.ascontiguousarray(self.default_params if params is None else params, np.float64)
        y = np.ascontiguousarray(y, np.complex128)
        out = np.zeros_like(y)
        _check(lib().orc_generator_apply(self._h, which, t, _dp(prm), len(prm),
                                         y.ctypes.data_as(DP), out.ctypes.data_as(DP)))
        return out


def set_threads(n: int) -> None:
    """Worker threads for single-solve loops; results are bit-identical to 1 thread."""
    lib().orc_set_threads(int(n))


def threads() -> int:
    return int(lib().orc_threads())


def rng(seed: int, stream: int, kind: int, n: int):
    """kind 0 next_u64, 1 uniform, 2 uniform_pos, 3 normal (rng.cpp:27-61)."""
    if kind == 0:
        out = np.zeros(n, np.uint64)
        lib().orc_rng(seed, stream, 0, n, None, out.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    else:
        out = np.zeros(n, np.float64)
        lib().orc_rng(seed, stream, kind, n, out.ctypes.data_as(DP), None)
    return out


def splitmix64_seq(state: int, n: int):
    s = C.c_ulonglong(state)
    return [lib().orc_splitmix64(C.byref(s)) for _ in range(n)]


def ising_capped_error(nx: int, ny: int) -> int:
    return lib().orc_ising_capped(nx, ny)
