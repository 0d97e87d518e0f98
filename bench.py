#!/usr/bin/env python3
"""Benchmark of the B200 time-evolution hot path (BASELINE.json configs).

Headline (N = 1, BASELINE configs[1]): mesolve of the dissipative transverse-field Ising chain,
10 spins (Liouvillian 4^10 = 1,048,576 rows, 24.6 M entries), Dormand-Prince 5(4) with the
reference defaults abstol 1e-8 / reltol 1e-6, tlist = linspace(0, 10, 100), e_ops Sx/Sy/Sz
totals. One "step" = one complete solve. `value` = device time per solve with the operator,
initial state and e_ops resident in HBM; `e2e` = the same solve through the C-ABI with host
buffers (operator store upload from pinned host CSR + rho0 in, expectations out).

For N > 1 (torchrun, one process per GPU) mesolve runs as independent replicas (a single solve
does not shard); the sharded workload — mcsolve trajectories of the 14-spin chain
combined with an NCCL all-gather of the per-rank pairwise block sums — is reported under
`secondary.mcsolve` at every N.

`--impl reference` times the CPU restatement of the reference (oracle/) on the same complete
solve, with every host thread (row-parallel SpMV and element-wise loops; bit-identical to the
single-threaded restatement, tests/test_oracle_pinning.py), rank 0 only.

`--gpus N` without a torchrun environment re-launches itself under torch.distributed.run with N
processes (one per GPU, 127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
TLIST = np.linspace(0.0, 10.0, 100)
TFIM = (10, 1, 1.0, 0.2, 1.0, 1)       # nx, ny, Jz, hx, gamma, periodic (scenarios/ising_mc_2x3.json:5)
TFIM_MC = (14, 1, 1.0, 0.2, 1.0, 1)
MC_SEED = 2025
KERR_CUTOFFS = (50, 100, 150, 200, 300, 400)

# The workload every arm of the headline line reports (identical dict in both arms).
HEADLINE_CONFIG = {
    "workload": "mesolve dissipative TFIM chain, 10 spins, periodic (BASELINE configs[1])",
    "liouvillian_rows": 1048576, "liouvillian_nnz": 24641536, "tlist": "linspace(0,10,100)",
    "abstol": 1e-08, "reltol": 1e-06, "e_ops": "Sx,Sy,Sz totals", "method": "Dormand-Prince 5(4)",
    "l2_flush": "none needed: the 7-29 MB operator store is re-read 486 times per solve, so its L2 residency "
                "is part of the workload; the 11 state vectors (185 MB) exceed the 126 MB L2",
}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def __enter__(self):
        # 50 ms period; wait for the first sample so the sampler is live before the timed region
        import selectors
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            sel = selectors.DefaultSelector()
            sel.register(self.p.stdout, selectors.EVENT_READ)
            self.first = self.p.stdout.readline() if sel.select(timeout=5.0) else ""
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]  # the pre-roll sample is excluded
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                for i, nm in enumerate(names):
                    if f[4 + i].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(gpu=True):
    """One process per GPU (NCCL); the CPU reference arm joins with gloo (no device needed)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if gpu:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def csr_bytes(m):
    return m.rowptr.nbytes + m.col.nbytes + m.val.nbytes


# ---------------------------------------------------------------------------------------------------
def run_ours(args, ws, rank, local):
    import torch
    import paper_2504_21440_b200 as q

    dev = local
    torch.cuda.set_device(dev)
    ctx = q.Context(dev)
    peak, peak_src = hbm_peak()

    # ---- model: H, c_ops and e_ops from the product's C++ API (factories.cpp:204-246), then the
    # Liouvillian assembled on the device (qsg_liouvillian_create, equal to the reference's L entry
    # for entry, tests/test_gpu_liouvillian.py) straight into the operator store
    t0 = time.perf_counter()
    model = q.Model("ising", *TFIM)
    H = model.export(q.SEL_H_CONST)
    cops = [model.export(q.SEL_C_OP, k) for k in range(model.n_cops)]
    eops = [model.export(q.SEL_E_OP, k) for k in range(model.n_eops)]
    host_ops_s = time.perf_counter() - t0
    d = model.dim
    psi = model.psi0()
    rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()

    ctx.liouvillian(H, cops).close()  # first call pays the pool growth
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = ctx.liouvillian(H, cops)
    store_build_s = time.perf_counter() - t0
    n, nnz = op.n, op.nnz
    gen = q.Generator([op])
    rho0_dev = torch.from_numpy(rho0).to(f"cuda:{dev}")

    # ---- warm-up, then K timed solves (device-timed persistent kernel, max over ranks)
    for _ in range(args.warmup):
        r = q.mesolve(ctx, gen, d, rho0_dev, TLIST, eops)
    barrier(ws)
    torch.cuda.synchronize()
    kms, attempts = [], []
    with ClockSampler(dev) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            r = q.mesolve(ctx, gen, d, rho0_dev, TLIST, eops)
            kms.append(r["kernel_ms"])
            attempts.append(r["attempts"])
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    barrier(ws)
    ms_step = allreduce_max(sum(kms) / len(kms), ws)
    value_s = ms_step / 1e3
    att = attempts[-1]
    stats = r["stats"]

    # ---- roofline of the fused DP5 kernel, per launch (= per solve). Byte model of SURVEY.md §8d
    # with the operator-store term of the format actually read.
    store_info = q.op_store_info(op)
    cb, ndict = q.op_storage(op)
    mat_bytes = store_bytes(cb, ndict, n, nnz)  # the SpMV / start passes read the coded or plain store
    stage_bytes = solve_store_bytes(store_info, r["store"])  # the stage passes read this one
    b_att = 6 * stage_bytes + 47 * 16 * n
    b_init = 2 * mat_bytes + 6 * 16 * n
    alg_bytes = b_att * att + b_init
    achieved = alg_bytes / (ms_step / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "dp5_grid_kernel_dram_bytes.json")
    if os.path.exists(tp):
        try:
            key = {0: "plain", 1: "coded", 2: "key_aligned"}[int(r["store"])]
            traffic = json.load(open(tp)).get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the C-ABI with host buffers (pinned), copies inside the timed region:
    # the reference's mesolve(H, rho0, tlist, c_ops, e_ops) inputs -> device Liouvillian assembly +
    # operator store (qsg_liouvillian_create) -> qsg_mesolve(host rho0 -> host expect)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
    pcsr = lambda m: q.CsrMatrix(pin(m.rowptr), pin(m.col), pin(m.val), m.n_rows, m.n_cols)
    Hh, cops_h = pcsr(H), [pcsr(c) for c in cops]
    rho0_h = pin(rho0)
    e2e_steps = max(1, min(args.steps, 10))
    for _ in range(3):  # untimed warm-up: the stream-ordered pool reaches its steady-state blocks
        op_w = ctx.liouvillian(Hh, cops_h)
        q.mesolve(ctx, q.Generator([op_w]), d, rho0_h, TLIST, eops)
        op_w.close()
    barrier(ws)
    t0 = time.perf_counter()
    e2e_each = []
    for _ in range(e2e_steps):
        ts = time.perf_counter()
        op2 = ctx.liouvillian(Hh, cops_h)
        r2 = q.mesolve(ctx, q.Generator([op2]), d, rho0_h, TLIST, eops)
        _ = r2["expect"].sum()
        op2.close()
        e2e_each.append(time.perf_counter() - ts)
    e2e_s = allreduce_max((time.perf_counter() - t0) / e2e_steps, ws)
    h2d = csr_bytes(H) + sum(csr_bytes(c) for c in cops) + rho0.nbytes + sum(csr_bytes(e) for e in eops)
    d2h = r2["expect"].nbytes

    # the same, starting from the reference-built Liouvillian CSR (host build timed separately)
    e2e_L = None
    if not args.quick:
        t0 = time.perf_counter()
        L = model.export(q.SEL_L_CONST)
        host_l_build_s = time.perf_counter() - t0
        Lh = pcsr(L)
        op_w = ctx.op(Lh)
        q.mesolve(ctx, q.Generator([op_w]), d, rho0_h, TLIST, eops)
        op_w.close()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            op3 = ctx.op(Lh)
            r3 = q.mesolve(ctx, q.Generator([op3]), d, rho0_h, TLIST, eops)
            _ = r3["expect"].sum()
            op3.close()
        e2e_L = {"value": allreduce_max((time.perf_counter() - t0) / e2e_steps, ws), "unit": "s",
                 "h2d_bytes_per_step": int(csr_bytes(L) + rho0.nbytes + sum(csr_bytes(e) for e in eops)),
                 "path": "qsg_op_create(pinned host Liouvillian CSR) + qsg_mesolve",
                 "host_liouvillian_build_s": host_l_build_s}
        del Lh, L

    # ---- secondary: SpMV of the operator store (SpMV HBM GB/s metric), and the same solve on the
    # plain (int32 column + complex128 value) store for comparison
    y = torch.randn(n, dtype=torch.complex128, device=f"cuda:{dev}")
    out = torch.empty_like(y)
    spmv_ms = q.generator_apply_timed(ctx, gen, y, out, reps=20)
    spmv_bytes = mat_bytes + 32 * n
    secondary = {"spmv_tfim10": {"store": "coded" if cb else "plain", "ms": spmv_ms,
                                 "GBps": spmv_bytes / spmv_ms / 1e6, "frac": spmv_bytes / spmv_ms / 1e6 / peak,
                                 "bytes_model": "store bytes + 32*n"}}
    os.environ["QSG_NO_COMPRESS"] = "1"
    op_p = ctx.liouvillian(H, cops)
    del os.environ["QSG_NO_COMPRESS"]
    gen_p = q.Generator([op_p])
    q.mesolve(ctx, gen_p, d, rho0_dev, TLIST, eops)
    kp = [q.mesolve(ctx, gen_p, d, rho0_dev, TLIST, eops) for _ in range(max(1, min(args.steps, 3)))]
    ms_p = sum(x["kernel_ms"] for x in kp) / len(kp)
    mat_p = store_bytes(0, 0, n, nnz)
    alg_p = (6 * mat_p + 47 * 16 * n) * kp[-1]["attempts"] + 2 * mat_p + 6 * 16 * n
    spmv_p = q.generator_apply_timed(ctx, gen_p, y, out, reps=20)
    secondary["plain_store"] = {
        "solve_ms": ms_p, "GBps": alg_p / ms_p / 1e6, "frac": alg_p / ms_p / 1e6 / peak,
        "spmv_ms": spmv_p, "spmv_GBps": (mat_p + 32 * n) / spmv_p / 1e6,
        "bytes_model": "per attempt 6*(20*nnz+4*n+8*n/32) + 47*16*n"}
    op_p.close()
    secondary["operator_store"] = {"code_bytes": cb, "dict_pairs": ndict, "bytes_per_spmv": mat_bytes,
                                   "plain_bytes_per_spmv": mat_p}
    if e2e_L is not None:
        secondary["e2e_from_liouvillian_csr"] = e2e_L
    cpu_legs = rank == 0 and ws == 1 and not args.no_cpu
    if not args.quick:
        secondary["kerr_sweep_spmv"] = kerr_sweep_spmv(ctx, q, torch, dev, peak)
        secondary["kerr_cutoff_mesolve"] = kerr_cutoff_mesolve(ctx, q, peak, cpu=cpu_legs)
        secondary["mcsolve"] = mcsolve_sharded(args, ctx, q, torch, ws, rank, peak, cpu=cpu_legs)
        secondary["param_sweep"] = param_sweep_sharded(args, ctx, q, torch, ws, rank, cpu=cpu_legs)
        secondary["stochastic"] = stochastic_secondary(args, q, rank)
        secondary["sesolve_tfim20"] = sesolve_tfim20(ctx, q, peak)
    del out, y

    line = {
        "metric": "mesolve_time_to_solution",
        "value": value_s,
        "unit": "s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic: reference TFIM construction (factories.cpp:204-246), all-up initial state",
        "config": dict(HEADLINE_CONFIG, parallelism=f"replicas x{ws}" if ws > 1 else "single solve, one cooperative grid"),
        "run": {"dp5_attempts": att, "stats_steps_rejected_rhs": list(stats), "host_operator_build_s": host_ops_s,
                "device_liouvillian_and_store_build_s": store_build_s, "grid_ctas": r["grid_ctas"],
                "timed_wall_s": wall, "operator_store": store_info},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "dp5_grid_kernel (persistent fused DP5 solve, 1 launch per solve)",
                     "bytes_model": "per attempt 6*store + 47*16*n (SURVEY.md 8d vector passes) + start 2 SpMV; "
                                    "store = bytes of the operator store the stage passes stream "
                                    "(qsg_op_store_info: key-aligned blocks, or code_bytes*nnz + 4*n + "
                                    "16*n/32 + 20*pairs coded, or 20*nnz + 4*n + 8*n/32 plain)",
                     "store_streamed": {0: "plain", 1: "coded", 2: "key-aligned"}[int(r["store"])],
                     "store_bytes_per_spmv": stage_bytes},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "per_step_s": e2e_each,
                "path": "qsg_liouvillian_create(pinned host H, c_ops) + qsg_mesolve(host rho0 -> host expect)"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "secondary": secondary,
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(stats)
    ctx.close()
    return line


def solve_store_bytes(info, store):
    """Bytes one stage SpMV of the grid solver reads from the store it streamed (timing.store:
    0 plain, 1 coded, 2 key-aligned)."""
    return {0: info["plain_bytes"], 1: info["coded_bytes"], 2: info["ka_bytes"]}[int(store)]


def store_bytes(code_bytes, dict_pairs, n, nnz):
    """Bytes one SpMV reads from the operator store (SELL-32): entries + row lengths + slice
    offsets (+ the (offset, value) dictionary of a coded store)."""
    nsl = (n + 31) // 32
    if code_bytes:
        return code_bytes * nnz + 4 * n + 16 * nsl + 20 * dict_pairs
    return 20 * nnz + 4 * n + 8 * nsl


def kerr_sweep_spmv(ctx, q, torch, dev, peak):
    """BASELINE configs[3]: Liouvillian SpMV of the Kerr resonator for N = 50..400 (L2-resident
    for the smaller cutoffs, so bytes/time can exceed the HBM copy rate)."""
    out = {}
    for N in KERR_CUTOFFS:
        m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
        Lk = m.export(q.SEL_L_CONST)
        g = q.Generator([ctx.op(Lk)])
        y = torch.randn(Lk.n_rows, dtype=torch.complex128, device=f"cuda:{dev}")
        o = torch.empty_like(y)
        ms = q.generator_apply_timed(ctx, g, y, o, reps=50)
        cbk, ndk = q.op_storage(g.ops[0])
        b = store_bytes(cbk, ndk, Lk.n_rows, Lk.nnz) + 32 * Lk.n_rows
        out[f"N{N}"] = {"rows": Lk.n_rows, "nnz": Lk.nnz, "us": ms * 1e3, "GBps": b / ms / 1e6}
    return out


def kerr_cutoff_mesolve(ctx, q, peak, cpu=False):
    """BASELINE configs[3]: Kerr resonator mesolve over cutoffs N (Liouvillian up to 160k rows),
    abstol 1e-8, tlist linspace(0,10,101); device time per solve and byte-model GB/s. cpu: the
    oracle (1 thread, as the reference's mesolve) on the first 0.2 time units of the same solve
    at every N, reported per DP5 attempt beside the device's per-attempt time."""
    out = {}
    tl = np.linspace(0.0, 10.0, 101)
    kerr_traffic = {}
    tp = os.path.join(ROOT, "profiles", "r02_kerr_cutoff_traffic.json")
    if os.path.exists(tp):
        kerr_traffic = json.load(open(tp)).get("cutoffs", {})
    for N in KERR_CUTOFFS:
        m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
        Lk = m.export(q.SEL_L_CONST)
        g = q.Generator([ctx.op(Lk)])
        eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
        psi = m.psi0()
        rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
        q.mesolve(ctx, g, m.dim, rho0, tl, eops)  # warm-up
        r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
        n, nnz = Lk.n_rows, Lk.nnz
        cbk, ndk = q.op_storage(g.ops[0])
        b = (6 * store_bytes(cbk, ndk, n, nnz) + 47 * 16 * n) * r["attempts"]
        out[f"N{N}"] = {"rows": n, "nnz": nnz, "solve_ms": r["kernel_ms"], "attempts": r["attempts"],
                        "us_per_attempt": r["kernel_ms"] * 1e3 / r["attempts"], "GBps_model": b / r["kernel_ms"] / 1e6,
                        "grid_ctas": r["grid_ctas"], "note": "L2-resident operator: GB/s can exceed the HBM rate"}
        tr = kerr_traffic.get(f"N{N}")
        if tr:  # committed ncu capture of the same solve (profiles/r02_kerr_cutoff_traffic.json)
            out[f"N{N}"]["ncu"] = {"dram_bytes": tr["dram_bytes"], "lts_bytes": tr["lts_bytes"],
                                   "lts_GBps": tr["lts_GBps"], "gpu_time_ms": tr["gpu_time_ms"]}
        if cpu:
            from oracle import oracle as O
            O.set_threads(1)
            om = O.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
            om.prepare_liouvillian()
            t0 = time.perf_counter()
            _, st = om.mesolve_prepared(np.linspace(0.0, 0.2, 3))
            dt = time.perf_counter() - t0
            per = dt / int(st[0] + st[1])
            out[f"N{N}"]["cpu_baseline"] = {
                "us_per_attempt": per * 1e6, "cores": 1, "kind": "port",
                "sample": f"oracle mesolve t in [0,0.2] ({int(st[0] + st[1])} attempts, {dt:.2f} s)",
                "device_speedup_per_attempt": per * 1e3 / (r["kernel_ms"] / r["attempts"])}
    return out


def sesolve_tfim20(ctx, q, peak):
    """§8a8 sesolve on the same persistent grid engine: closed TFIM chain of 20 spins (ket of
    1,048,576 amplitudes, G = -iH with 22.0 M entries), all-up start, tlist linspace(0,10,100),
    Sx/Sy/Sz totals. Device time per solve and the SURVEY §8d byte model of the fused attempt."""
    t0 = time.perf_counter()
    m = q.Model("ising", 20, 1, 1.0, 0.2, 0.0, 1)
    G = m.export(q.SEL_SE_GEN)
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    host_s = time.perf_counter() - t0
    op = ctx.op(G)
    g = q.Generator([op])
    psi = m.psi0()
    tl = np.linspace(0.0, 10.0, 100)
    q.sesolve(ctx, g, m.dim, psi, tl, eops)
    r = q.sesolve(ctx, g, m.dim, psi, tl, eops)
    n, nnz = G.n_rows, G.nnz
    cb, nd = q.op_storage(op)
    b = (6 * store_bytes(cb, nd, n, nnz) + 47 * 16 * n) * r["attempts"]
    out = {"workload": "sesolve closed TFIM chain, 20 spins, periodic (ket dim 2^20)", "rows": n, "nnz": nnz,
           "solve_ms": r["kernel_ms"], "attempts": r["attempts"], "store": "coded" if cb else "plain",
           "dict_pairs": nd, "GBps_model": b / r["kernel_ms"] / 1e6, "frac": b / r["kernel_ms"] / 1e6 / peak,
           "host_operator_build_s": host_s, "stats_steps_rejected_rhs": list(r["stats"])}
    op.close()
    return out


def param_sweep_sharded(args, ctx, q, torch, ws, rank, cpu=False):
    """BASELINE configs[4]: 256 (Delta, F) points of two coupled Kerr modes (N=10 each,
    U=0.1, J=0.5, gamma=1), Delta in linspace(-2,2,16) x F in linspace(0.1,1,16), one mesolve per
    point, points sharded in contiguous blocks over ranks (no numeric reduction)."""
    from paper_2504_21440_b200.dist import shard_range

    m = q.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
    ops = [ctx.op(m.export(q.SEL_L_CONST))] + [ctx.op(m.export(q.SEL_L_TERM, k)) for k in range(m.n_terms)]
    g = q.Generator(ops, [(q.COEFF_CONST, 0, 0, 1.0, 0.0), (q.COEFF_PARAM, 0, 0, 0.0, 0.0),
                          (q.COEFF_PARAM, 1, 0, 0.0, 0.0)])
    eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
    pts = np.array([[d, f] for d in np.linspace(-2, 2, 16) for f in np.linspace(0.1, 1.0, 16)])
    b, e = shard_range(len(pts), rank, ws)
    rho0 = np.zeros(m.dim * m.dim, complex)
    rho0[0] = 1.0
    tl = np.linspace(0.0, 10.0, 101)
    q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, pts[b:b + 1])  # warm-up
    barrier(ws)
    r = q.mesolve_batch(ctx, g, m.dim, rho0, tl, eops, pts[b:e])
    t_ms = allreduce_max(r["kernel_ms"], ws)
    res = {"workload": "256-point coupled-Kerr (N=10x10, Liouvillian 10^4 rows) mesolve sweep",
           "points": len(pts), "points_this_rank": e - b, "device_s": t_ms / 1e3,
           "points_per_s": len(pts) / (t_ms / 1e3), "attempts_rank0": r["attempts"],
           "failed": int((r["status"] != 0).sum())}
    if cpu:
        res["cpu_baseline"] = sweep_cpu(pts, tl)
    return res


def sweep_cpu(pts, tl):
    """Oracle sweep points (each a single-threaded mesolve, as the reference's): 4 points on one
    thread, and one point per host thread run concurrently (independent points)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    O.set_threads(1)
    m = O.Model("coupled_kerr", 10, 0.1, 0.5, 1.0)
    m.prepare_liouvillian()
    t0 = time.perf_counter()
    for p in pts[:4]:
        m.mesolve_prepared(tl, params=p)
    one = 4 / (time.perf_counter() - t0)
    th = host_threads()
    models = [O.Model("coupled_kerr", 10, 0.1, 0.5, 1.0) for _ in range(th)]
    for mm in models:
        mm.prepare_liouvillian()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(th) as ex:
        list(ex.map(lambda k: models[k].mesolve_prepared(tl, params=pts[k]), range(th)))
    many = th / (time.perf_counter() - t0)
    return {"points_per_s_1_thread": one, "points_per_s_all_threads": many, "cores": th, "kind": "port",
            "sample": f"oracle mesolve of grid points: 4 sequential on 1 thread; {th} concurrent on {th} threads"}


def stochastic_secondary(args, q, rank):
    """ssesolve / smesolve (Euler-Maruyama, trajectories.cpp:251-503) on the
    reference scenario's JC assembly (scenario.cpp:252-277), N=10, tlist linspace(0,10,101),
    dt_max 1e-3 (10^4 steps per trajectory). Device time of the trajectory kernel; the oracle
    (CPU restatement, 1 thread) timed on a few trajectories beside it, rank 0 only."""
    t = np.linspace(0.0, 10.0, 101)
    out = {}
    cases = [("ssesolve", "jc_sse", (10, 1.0, 1.0, 0.1, 0.5), args.sde_traj, False),
             ("smesolve", "jc_sme", (10, 1.0, 1.0, 0.1, 0.5, 0.1, 0.05), max(1, args.sde_traj // 10), True)]
    for key, name, prm, ntraj, sme in cases:
        m = q.Model(name, *prm)
        run = (lambda n: m.smesolve(t, 5, n, n_det=2, dt_max=1e-3)) if sme else \
              (lambda n: m.ssesolve(t, 5, n, dt_max=1e-3))
        run(8)
        r = run(ntraj)
        out[key] = {"workload": f"{name}{prm} x {ntraj} trajectories, 10^4 Euler-Maruyama steps each",
                    "device_s": r["device_ms"] / 1e3, "traj_per_s": ntraj / (r["device_ms"] / 1e3)}
        if rank == 0:
            from oracle import oracle as O
            om = O.Model(name, *prm)
            k = 2 if sme else 8
            t0 = time.perf_counter()
            (om.smesolve(t, 5, k, n_det=2, dt_max=1e-3, n_threads=1) if sme
             else om.ssesolve(t, 5, k, dt_max=1e-3, n_threads=1))
            out[key]["cpu_oracle_traj_per_s_1_thread"] = k / (time.perf_counter() - t0)
    return out


def mcsolve_sharded(args, ctx, q, torch, ws, rank, peak, cpu=False):
    """BASELINE configs[2] workload (TFIM-14 mcsolve, 10k trajectories by default), sharded in
    contiguous blocks (trajectory i = RngStream(2025, i) on every N), block sums combined in the
    reference's pairwise bracket after an NCCL all-gather. Roofline: SURVEY §8d's 47*16*n bytes
    per trajectory-attempt over all ranks' attempts / the max-over-ranks device time."""
    from paper_2504_21440_b200.dist import ProductComm, combine_leaves, ensemble_shards, gather_leaf_sums

    ntraj = args.mc_traj
    m = q.Model("ising", *TFIM_MC)
    G = q.Generator([ctx.op(m.export(q.SEL_MC_GEN))])
    cops = [m.export(q.SEL_C_OP, k) for k in range(m.n_cops)]
    eops = [m.export(q.SEL_E_OP, 2)]
    shards = ensemble_shards(ntraj, ws)
    b, e, leaves = shards[rank]
    rel = [(lo - b, hi - b) for lo, hi in leaves]  # leaf positions in this rank's completed list
    q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), TLIST, MC_SEED, b, min(e, b + 64), per_traj=False)  # warm-up
    comm, comm_note = None, None
    if ws > 1:
        try:
            comm = ProductComm(ctx, rank, ws)
        except Exception as ex:  # keep the line: torch.distributed (NCCL) all-gather instead
            comm_note = f"product NCCL communicator unavailable ({ex}); torch.distributed all_gather used"
    barrier(ws)
    r = q.mcsolve(ctx, G, cops, eops, m.dim, m.psi0(), TLIST, MC_SEED, b, e, per_traj=False, ranges=rel)
    t_ms = allreduce_max(r["kernel_ms"], ws)
    att_all = allreduce_sum(r["attempts"], ws)
    if ws > 1:
        nl = max(len(s[2]) for s in shards)
        sums, counts = gather_leaf_sums(r["range_sums"], r["n_ok"], nl, ws, comm=comm,
                                        device=torch.device("cuda", ctx.device))
        if comm is not None:
            comm.close()
    else:
        sums, counts = [r["range_sums"]], [r["n_ok"]]
    n_ok = sum(counts)
    mean = combine_leaves(ntraj, ws, sums, counts) if n_ok == ntraj else None
    n = m.dim
    ach = att_all * 47 * 16 * n / (t_ms / 1e3) / 1e9
    res = {"workload": "mcsolve TFIM-14 (16384-dim), Sz_total, tlist linspace(0,10,100), seed 2025",
           "ntraj": ntraj, "n_ok": n_ok, "device_s": t_ms / 1e3, "traj_per_s": ntraj / (t_ms / 1e3),
           "attempts_all_ranks": att_all, "mean_Sz_t10": None if mean is None else float(mean[0, -1].real),
           "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                        "bytes_model": "47*16*n per trajectory-attempt (SURVEY.md 8d), operator L2-resident"},
           "shards": "whole pairwise-bracket subtrees per rank (dist.ensemble_shards), sums on the device",
           "collective": (comm_note or "product NCCL all-gather (qsg_comm_allgather) of per-rank bracket-subtree sums")
                         if ws > 1 else None}
    if cpu:
        from oracle import oracle as O
        th = host_threads()
        om = O.Model("ising", *TFIM_MC)
        k = 2 * th
        t0 = time.perf_counter()
        om.mcsolve(TLIST, MC_SEED, k, n_threads=th)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"traj_per_s": k / dt, "cores": th, "kind": "port",
                               "sample": f"oracle run_ensemble, trajectories 0..{k - 1} of seed 2025 on {th} threads "
                                         f"({dt:.1f} s)"}
    return res


def oracle_tfim10(threads, spins=10):
    """The oracle's TFIM-10 model with the Liouvillian prebuilt (the reference builds it inside
    mesolve, evolve.cpp:243-252; the GPU line times the device assembly separately too).
    spins != 10 only through the --ref-sample-spins test hook."""
    from oracle import oracle as O
    O.set_threads(threads)
    m = O.Model("ising", spins, *TFIM[1:])
    t0 = time.perf_counter()
    m.prepare_liouvillian()
    return O, m, time.perf_counter() - t0


def cpu_baseline(gpu_stats):
    """One complete configs[1] solve by the oracle (CPU restatement of evolve.cpp/integrator.hpp)
    on every host thread; its step statistics must match the device solve's."""
    th = host_threads()
    O, m, build = oracle_tfim10(th)
    t0 = time.perf_counter()
    _, st = m.mesolve_prepared(TLIST)
    dt = time.perf_counter() - t0
    O.set_threads(1)
    return {"value": dt, "unit": "s", "cores": th, "kind": "port",
            "sample": f"one complete TFIM-10 solve (t in [0,10], {int(st[0] + st[1])} DP5 attempts, stats "
                      f"{list(map(int, st))} vs device {list(map(int, gpu_stats))}), oracle with {th} threads "
                      f"(row-parallel SpMV, bit-identical to 1 thread); Liouvillian build {build:.1f} s excluded"}


def run_reference(args, ws, rank):
    """--impl reference: the CPU restatement of the reference running the same complete solves on
    this host (rank 0 only; the other ranks exit without work)."""
    if rank != 0:
        return None
    th = host_threads()
    O, m, build = oracle_tfim10(th, args.ref_sample_spins)
    for _ in range(args.warmup):
        m.mesolve_prepared(TLIST)
    vals = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, st = m.mesolve_prepared(TLIST)
        vals.append(time.perf_counter() - t0)
    v = sum(vals) / len(vals)
    sample = (f"complete TFIM-10 solve per step (t in [0,10], {int(st[0] + st[1])} DP5 attempts, stats "
              f"{list(map(int, st))}); oracle = CPU restatement of evolve.cpp/integrator.hpp/superop.cpp with "
              f"{th} threads (row-parallel SpMV + element-wise loops, bit-identical to the single-threaded "
              f"reference order); Liouvillian build {build:.1f} s excluded, as on the GPU line")
    return {"metric": "mesolve_time_to_solution", "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128",
            "data": "synthetic: reference TFIM construction (factories.cpp:204-246), all-up initial state",
            "config": dict(HEADLINE_CONFIG, parallelism=f"replicas x{ws}" if ws > 1 else "single solve, one cooperative grid"),
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "s", "cores": th, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "run": {"per_step_s": vals}}


def maybe_relaunch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run with N ranks."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mc-traj", type=int, default=10000)
    ap.add_argument("--sde-traj", type=int, default=2000)
    ap.add_argument("--quick", action="store_true", help="headline only (no secondary workloads)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--ref-sample-spins", type=int, default=10,
                    help=argparse.SUPPRESS)  # test hook: a smaller chain for the CPU launch test
    args = ap.parse_args()
    maybe_relaunch(args)
    ws, rank, local = dist_init(gpu=args.impl != "reference")
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
    else:
        line = run_ours(args, ws, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
