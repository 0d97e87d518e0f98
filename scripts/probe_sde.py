"""Throughput of the device SSE/SME engines on the scenario JC models (and the oracle per trajectory)."""
import sys, time, json
import numpy as np
import paper_2504_21440_b200 as q

t = np.linspace(0.0, 10.0, 101)
ctx = q.Context(0)
for name, prm, ntraj, sme in [("jc_sse", (10, 1.0, 1.0, 0.1, 0.5), 2000, False),
                              ("jc_sme", (10, 1.0, 1.0, 0.1, 0.5, 0.1, 0.05), 200, True)]:
    m = q.Model(name, *prm)
    f = (lambda n: m.smesolve(t, 5, n, n_det=2, dt_max=1e-3)) if sme else (lambda n: m.ssesolve(t, 5, n, dt_max=1e-3))
    f(8)
    r = f(ntraj)
    print(json.dumps({"model": name, "ntraj": ntraj, "device_s": r["device_ms"] / 1e3,
                      "traj_per_s": ntraj / (r["device_ms"] / 1e3)}), flush=True)
if len(sys.argv) > 1:
    from oracle import oracle as O
    for name, prm, sme in [("jc_sse", (10, 1.0, 1.0, 0.1, 0.5), False), ("jc_sme", (10, 1.0, 1.0, 0.1, 0.5, 0.1, 0.05), True)]:
        om = O.Model(name, *prm)
        t0 = time.perf_counter()
        (om.smesolve(t, 5, 2, n_det=2, dt_max=1e-3) if sme else om.ssesolve(t, 5, 4, dt_max=1e-3))
        dt = time.perf_counter() - t0
        print(json.dumps({"oracle": name, "s_per_traj": dt / (2 if sme else 4)}), flush=True)
