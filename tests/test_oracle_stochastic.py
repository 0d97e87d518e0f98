"""Pins the oracle's stochastic solvers (ssesolve / smesolve, trajectories.cpp:251-503) with the
reference's own tests (test_trajectories.cpp:205-346), restated on the zoo's scenario-style JC
models (scenario.cpp:252-277): jc_sse has sc_ops = {sqrt(kappa) a}; jc_sme has c_ops =
{sqrt(gamma) sm, sqrt(kphi) a^dag a} and the measured sqrt(kappa) a last. CPU only.
"""
import numpy as np
import scipy.sparse as sp

from oracle import oracle as O


def _csr(m, which, k=0):
    rp, col, val, n = m.export(which, k)
    return sp.csr_matrix((val, col, rp), shape=(n, n))


def test_sse_deterministic_limit():
    """test_trajectories.cpp:205-216: no measurement rate -> sesolve within O(dt)."""
    t = np.linspace(0.0, 5.0, 26)
    sse = O.Model("jc_sse", 8, 1.0, 1.0, 0.1, 0.0).ssesolve(t, 11, 1, dt_max=1e-4)
    se, _, _ = O.Model("jc", 8, 1.0, 1.0, 0.1, 0.0, 0.0).sesolve(t)
    assert np.max(np.abs(sse["mean"][0] - se[0])) < 5e-4


def test_sse_wiener_moments_and_current_identity():
    """test_trajectories.cpp:218-244."""
    m = O.Model("jc_sse", 4, 1.0, 1.0, 0.1, 0.5)
    r = m.ssesolve(np.linspace(0.0, 1.0, 11), 21, 40, dt_max=1e-3, store_measurement=True)
    inc, dt = r["increments"], r["dt"]
    assert np.max(np.abs(r["current"] - (r["expectation"] + inc / dt))) == 0.0
    n = inc.size
    assert abs(inc.sum() / n) < 4.0 * np.sqrt(dt / n)
    assert abs((inc ** 2).sum() / n - dt) < 4.0 * dt * np.sqrt(2.0 / n)


def test_sse_single_channel_fast_path_equals_general_path():
    """test_trajectories.cpp:246-291: the fast path against the general update order, same stream."""
    m = O.Model("jc_sse", 6, 1.0, 1.0, 0.1, 0.3)
    t = np.linspace(0.0, 0.5, 6)
    fast = m.ssesolve(t, 31, 1, dt_max=1e-3)
    H, S, N = _csr(m, O.H_CONST), _csr(m, O.C_OP, 0), _csr(m, O.E_OP, 0)
    SdS, X = (S.conj().T @ S).tocsr(), (S + S.conj().T).tocsr()
    sub = max(1, int(np.ceil((t[1] - t[0]) / 1e-3 * (1.0 - 1e-12))))
    dt = (t[1] - t[0]) / sub
    normals = O.rng(31, 0, 3, 5 * sub)
    psi = m.psi0().astype(complex)
    psi /= np.linalg.norm(psi)
    ref = [np.vdot(psi, N @ psi)]
    step = 0
    for _ in range(5):
        for _ in range(sub):
            e_n = np.vdot(psi, X @ psi).real
            dw = np.sqrt(dt) * normals[step]
            step += 1
            drift = -1j * (H @ psi)
            spsi = S @ psi
            drift = drift + 0.5 * e_n * spsi
            stoch = dw * spsi - 0.5 * e_n * dw * psi
            drift = drift - 0.5 * (SdS @ psi)
            drift = drift - 0.125 * e_n * e_n * psi
            psi = psi + dt * drift + stoch
            psi = psi / np.linalg.norm(psi)
        ref.append(np.vdot(psi, N @ psi))
    assert np.max(np.abs(fast["mean"][0] - np.array(ref))) < 1e-10


def test_sme_deterministic_limit():
    """test_trajectories.cpp:293-306: every channel deterministic -> mesolve within O(dt)."""
    m = O.Model("jc_sme", 6, 1.0, 1.0, 0.1, 0.2, 0.0, 0.0)
    t = np.linspace(0.0, 4.0, 21)
    sme = m.smesolve(t, 41, 1, n_det=3, dt_max=2e-4)
    me, _, _ = m.mesolve(t)
    assert np.max(np.abs(sme["mean"][0] - me[0])) < 5e-4


def test_sse_sme_ensembles_converge_to_mesolve():
    """test_trajectories.cpp:320-344 (c1/sqrt(ntraj) + c2 dt scaling), plus the same for smesolve."""
    m = O.Model("jc_sse", 4, 1.0, 1.0, 0.1, 1.0)
    t = np.linspace(0.0, 2.0, 21)
    me, _, _ = m.mesolve(t)
    err = lambda ntraj, dt: np.max(np.abs(m.ssesolve(t, 2024, ntraj, dt_max=dt)["mean"][2] - me[2]))
    coarse, fine = err(60, 4e-3), err(240, 2e-3)
    assert fine < coarse * 1.05 and fine < 0.25
    ms = O.Model("jc_sme", 4, 1.0, 1.0, 0.1, 1.0, 0.1, 0.05)
    mes, _, _ = ms.mesolve(t)
    sme = ms.smesolve(t, 7, 40, n_det=2, dt_max=2e-3)
    assert np.max(np.abs(sme["mean"][0] - mes[0])) < 0.05
