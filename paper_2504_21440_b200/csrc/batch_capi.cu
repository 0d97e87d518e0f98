// C-ABI of the batched engine: qsg_mcsolve (trajectories.cpp:106-249 + run_ensemble :26-92)
// and qsg_mesolve_batch (one mesolve per parameter point, PAPER.md:647-652 pattern).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "batch_engine.h"
#include "ensemble.h"
#include "qsg_internal.h"

using namespace qsg;

namespace {

struct TmpOps {
  std::vector<qsg_op*> ops;
  ~TmpOps() {
    for (auto* o : ops) qsg_op_destroy(o);
  }
};

// The batch engine reads the plain store unless QSG_BATCH_CODES=1: its operators are re-read by
// every CTA from L2, and on TFIM-14 the code -> dictionary hop made the gathers slower
// (705 vs 763 traj/s, profiles/r01_summary.md).
bool batch_codes() {
  const char* e = std::getenv("QSG_BATCH_CODES");
  return e && e[0] == '1';
}

qsg_status make_sell(qsg_ctx* ctx, const qsg_csr& a, TmpOps& keep, DevSell& out) {
  qsg_op* op = nullptr;
  if (qsg_status s = qsg_op_create(ctx, &a, &op)) return s;
  keep.ops.push_back(op);
  out = sell_view(op, batch_codes());
  return QSG_OK;
}

// Device-side ensemble sums requested from run_batch (mcsolve): n_ranges == 0 = one sum over
// every completed trajectory of the block.
struct SumReq {
  bool on = false;
  long long nv = 0;
  int n_ranges = 0;
  const long long* lo = nullptr;
  const long long* hi = nullptr;
};

struct RunOut {
  std::vector<double2> expect;
  std::vector<double2> sums;  // SumReq results, n_ranges (or 1) x nv
  long long n_ok = 0;
  std::vector<int> status, jcount, jch;
  std::vector<double> ftime, jtime;
  std::vector<long long> stats;
  double kernel_ms = 0;
  long long attempts = 0;
  int grid = 0;
  bool grid_mode = false;
  int layout = 0;
};

// Runs systems [sys_begin, sys_begin + n_sys) through the batch kernel and downloads outputs.
qsg_status run_batch(qsg_ctx* ctx, BatchProblem P, long long n_sys, int jump_cap, RunOut& o,
                     bool want_expect = true, const SumReq& req = SumReq{}) {
  cudaStream_t s = ctx->stream;
  cudaError_t ce;
  P.n_systems = n_sys;
  P.jump_cap = jump_cap;
  // Layouts (batch_engine.cu): 4 = one trajectory per CTA (default), 1 = one 32-slot batch spread
  // over the whole GPU, 0/2/3 = 8/4/2 slots per CTA, 5/6 = 1/2 slots per thread-block cluster.
  // Measured on TFIM-14 (profiles/r01_summary.md, scripts/probe_mcmodes.py): one trajectory per
  // CTA wins from ~300 trajectories up among the CTA layouts (740 traj/s at 10,000 vs 621/500/428
  // for 2/4/8 slots and 274 for the grid batch): its private state is smallest, so more of it
  // stays in L1/L2. The grid batch wins only while per-CTA runs would leave most SMs idle.
  // QSG_BATCH_MODE=grid|local|local4|local2|local1|cluster1|cluster2 overrides;
  // QSG_CLUSTER sets the cluster size (default 16).
  const long long slots1 = static_cast<long long>(batch_max_blocks_per_sm(4)) * ctx->sm_count;
  int layout = 4;
  if (P.n >= 4096 && n_sys * 3 < slots1) layout = 1;
  if (const char* m = std::getenv("QSG_BATCH_MODE")) {
    const std::string v(m);
    layout = v == "grid"        ? 1
             : v == "local"     ? 0
             : v == "local4"    ? 2
             : v == "local2"    ? 3
             : v == "cluster1"  ? 5
             : v == "cluster2"  ? 6
             : v == "clusterdsm" ? 7
                                : 4;
  }
  // layout 7 (one trajectory per cluster, its state in the cluster's shared memory): the rows per
  // CTA are a power of two so a gather's owner CTA is a shift; up to 16 CTAs of ~200 KB each
  int dsm_shift = 0, dsm_cs = 0;
  {
    int sh = 5;
    while ((1LL << sh) * 16 < P.n) ++sh;
    const int cs7 = static_cast<int>((P.n + (1LL << sh) - 1) >> sh);
    if (batch_dsm_smem(sh) <= 200u * 1024u && cs7 >= 1 && cs7 <= 16) {
      dsm_shift = sh;
      dsm_cs = cs7;
    }
  }
  if (layout == 7 && dsm_cs == 0) layout = 4;
  int cs = 16;
  // mesolve parameter sweeps (configs[4]): one point per cluster of cs CTAs, cs the smallest size
  // whose co-resident points' state fits 1.5x L2 while every CTA slot still has work (16 when
  // there are too few points to fill the GPU otherwise, e.g. a sharded sweep). Coupled Kerr
  // 10x10, 256 points (scripts/probe_sweep.py): 158 ms one point per CTA; clusters of 2/4/8/16
  // CTAs 117/102/118/178 ms (4 CTAs: 74 points x 2.2 MB in flight). mcsolve keeps one trajectory
  // per CTA: its jump and norm bookkeeping made the cluster layouts no faster (section above).
  if (layout == 4 && P.mode == 1 && P.n >= 4096 && !std::getenv("QSG_BATCH_MODE")) {
    const double state = static_cast<double>(batch_work_stride(P.n, 5)) * sizeof(double2);
    for (int c = 2; c <= 16; c *= 2) {
      const int cap = batch_max_clusters(5, c);
      if (cap <= 0) break;
      if (n_sys * c < slots1 && c < 16) continue;  // few points: wider clusters keep the SMs busy
      if (std::min<long long>(cap, n_sys) * state <= 1.5 * static_cast<double>(ctx->l2_bytes)) {
        layout = 5;
        cs = c;
        break;
      }
    }
  }
  if (const char* c = std::getenv("QSG_CLUSTER")) cs = std::max(1, std::min(16, std::atoi(c)));
  if (layout == 7) cs = dsm_cs;
  if (layout == 7) {
    cs = dsm_cs;
    P.dsm_shift = dsm_shift;
  }
  const bool grid_mode = layout == 1;
  const bool cluster_mode = layout == 5 || layout == 6 || layout == 7;
  const int per_sm = batch_max_blocks_per_sm(layout);
  if (per_sm <= 0) return cuda_fail(cudaGetLastError(), "batch occupancy");
  const long long want = (n_sys + batch_slots(layout) - 1) / batch_slots(layout);  // batches
  int grid;
  if (grid_mode) {
    grid = std::min(per_sm * ctx->sm_count, (P.n + 31) / 32);
  } else if (cluster_mode) {
    const int cap = batch_max_clusters(layout, layout == 7 ? cs | (dsm_shift << 8) : cs);
    if (cap <= 0) return cuda_fail(cudaGetLastError(), "cluster occupancy");
    grid = static_cast<int>(std::min<long long>(cap, want)) * cs;
  } else {
    grid = static_cast<int>(std::min<long long>(static_cast<long long>(per_sm) * ctx->sm_count, want));
  }
  if (const char* eg = std::getenv("QSG_BATCH_GRID")) grid = std::max(1, std::min(grid, std::atoi(eg)));
  const size_t stride = batch_work_stride(P.n, layout);
  const int n_batches = grid_mode ? 1 : cluster_mode ? grid / cs : grid;
  if (!grid_mode) {  // per-batch workspaces: fit them in 60% of free memory (the queue refills)
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      const long long fit = static_cast<long long>(fr / 10 * 6 / (stride * sizeof(double2)));
      if (fit < 1) {
        set_error("OutOfMemory: batch workspace does not fit on the device");
        return QSG_OUT_OF_MEMORY;
      }
      if (fit < n_batches) grid = static_cast<int>(fit) * (cluster_mode ? cs : 1);
    }
  }
  o.grid = grid;
  o.grid_mode = grid_mode;
  o.layout = layout;
  DevBuf work, q, ex, st, ft, stt, jc, jt, jch, att, gp, gf, gb;
  const size_t nvals = static_cast<size_t>(std::max(1, P.n_e)) * P.n_t;
  if ((ce = work.alloc(stride * (grid_mode ? 1 : cluster_mode ? grid / cs : grid) * sizeof(double2), s)) ||
      (ce = q.alloc(8, s)) ||
      (ce = ex.alloc(nvals * n_sys * sizeof(double2), s)) || (ce = st.alloc(sizeof(int) * n_sys, s)) ||
      (ce = ft.alloc(sizeof(double) * n_sys, s)) || (ce = stt.alloc(sizeof(long long) * 3 * n_sys, s)) ||
      (ce = jc.alloc(sizeof(int) * n_sys, s)) ||
      (ce = jt.alloc(sizeof(double) * std::max<long long>(1, n_sys * jump_cap), s)) ||
      (ce = jch.alloc(sizeof(int) * std::max<long long>(1, n_sys * jump_cap), s)) || (ce = att.alloc(8, s)) ||
      (ce = gp.alloc(sizeof(double) * 32 * 15 * grid, s)) || (ce = gf.alloc(sizeof(double) * 32 * 15, s)) ||
      (ce = gb.alloc(2 * sizeof(unsigned), s)))
    return cuda_fail(ce, "batch workspace");
  cudaMemsetAsync(q.p, 0, 8, s);
  cudaMemsetAsync(att.p, 0, 8, s);
  cudaMemsetAsync(gb.p, 0, 2 * sizeof(unsigned), s);
  cudaMemsetAsync(ex.p, 0, nvals * n_sys * sizeof(double2), s);
  cudaMemsetAsync(jc.p, 0, sizeof(int) * n_sys, s);
  P.work = work.as<double2>();
  P.work_stride = static_cast<long long>(stride);
  P.queue = q.as<unsigned long long>();
  P.expect = ex.as<double2>();
  P.status = st.as<int>();
  P.fail_t = ft.as<double>();
  P.stats = stt.as<long long>();
  P.jump_count = jc.as<int>();
  P.jump_time = jt.as<double>();
  P.jump_channel = jch.as<int>();
  P.attempts_total = att.as<long long>();
  P.gpart = gp.as<double>();
  P.gfin = gf.as<double>();
  P.bar = gb.as<unsigned>();
  {  // every operator plain (no key-aligned or coded rows): the plain-only instantiation
    bool lean = true;
    for (int k = 0; k < P.gen.n_terms; ++k) lean = lean && P.gen.A[k].code_bytes == 0 && P.gen.A[k].ka_nval == 0;
    for (int k = 0; k < P.n_c; ++k) lean = lean && P.c_ops[k].code_bytes == 0 && P.c_ops[k].ka_nval == 0;
    for (int k = 0; k < P.n_e; ++k) lean = lean && P.e_ops[k].code_bytes == 0 && P.e_ops[k].ka_nval == 0;
    const char* le = std::getenv("QSG_BATCH_LEAN");
    P.lean = lean && !(le && le[0] == '0');
  }
  cudaEventRecord(ctx->ev[2], s);
  if ((ce = launch_batch(P, layout, grid, cs, s))) return cuda_fail(ce, "batch launch");
  cudaEventRecord(ctx->ev[3], s);
  if (req.on && req.nv > 0) {  // ensemble bracket sums on the device (K7)
    if ((ce = device_bracket_sums(ex.as<double2>(), st.as<int>(), n_sys, static_cast<long long>(nvals), req.n_ranges,
                                  req.lo, req.hi, s, o.n_ok, o.sums)))
      return cuda_fail(ce, "ensemble sums");
  }
  o.expect.resize(want_expect ? nvals * n_sys : 0);
  o.status.resize(n_sys);
  o.ftime.resize(n_sys);
  o.stats.resize(3 * n_sys);
  o.jcount.resize(n_sys);
  o.jtime.resize(std::max<long long>(1, n_sys * jump_cap));
  o.jch.resize(std::max<long long>(1, n_sys * jump_cap));
  if ((want_expect &&
       (ce = cudaMemcpyAsync(o.expect.data(), ex.p, nvals * n_sys * sizeof(double2), cudaMemcpyDeviceToHost, s))) ||
      (ce = cudaMemcpyAsync(o.status.data(), st.p, sizeof(int) * n_sys, cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(o.ftime.data(), ft.p, sizeof(double) * n_sys, cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(o.stats.data(), stt.p, sizeof(long long) * 3 * n_sys, cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(o.jcount.data(), jc.p, sizeof(int) * n_sys, cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(o.jtime.data(), jt.p, sizeof(double) * o.jtime.size(), cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(o.jch.data(), jch.p, sizeof(int) * o.jch.size(), cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaMemcpyAsync(&o.attempts, att.p, 8, cudaMemcpyDeviceToHost, s)) || (ce = cudaStreamSynchronize(s)))
    return cuda_fail(ce, "batch solve");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
  o.kernel_ms = ms;
  return QSG_OK;
}

qsg_status common_setup(qsg_ctx* ctx, const qsg_generator* G, long long n, const double* tlist, long long n_t,
                        const qsg_solve_opts* opts, BatchProblem& P) {
  if (!ctx) {
    set_error("InvalidGrid: null context");
    return QSG_INVALID_GRID;
  }
  cudaSetDevice(ctx->device);
  if (qsg_status s = check_tlist(tlist, n_t)) return s;
  if (qsg_status s = check_generator(G, n)) return s;
  if (opts && opts->method != 0) {
    set_error("InvalidGrid: only the adaptive Dormand-Prince 5(4) method runs on the device");
    return QSG_UNSUPPORTED;
  }
  P.n = static_cast<int>(n);
  P.gen = make_devgen(G, batch_codes());
  // time-independent generator (constant or params[i] coefficients): stage 2 can use k1 = G y
  // (batch_kernel.cuh P1); QSG_K1G=0 keeps the two-vector gather
  {
    bool aut = true;
    for (int k = 1; k < G->n_terms; ++k)
      aut = aut && G->coeffs && (G->coeffs[k].kind == QSG_COEFF_CONST || G->coeffs[k].kind == QSG_COEFF_PARAM);
    const char* kg = std::getenv("QSG_K1G");
    P.autonomous = aut && !(kg && kg[0] == '0');
  }
  // generator terms that carry a key-aligned store are read through it (ka_row_slot) unless
  // QSG_BATCH_KA=0
  if (const char* e = std::getenv("QSG_BATCH_KA"))
    if (e[0] == '0')
      for (int k = 0; k < P.gen.n_terms; ++k) P.gen.A[k].ka_nval = 0;
  P.atol = opts ? opts->abstol : 1e-8;
  P.rtol = opts ? opts->reltol : 1e-6;
  if (!(P.atol > 0 && P.rtol > 0)) {
    set_error("InvalidGrid: tolerances must be positive");
    return QSG_INVALID_GRID;
  }
  P.max_steps = opts ? opts->max_steps : 10000000LL;
  P.n_t = static_cast<int>(n_t);
  P.t0 = tlist[0];
  P.tf = tlist[n_t - 1];
  return QSG_OK;
}

}  // namespace

extern "C" qsg_status qsg_mcsolve(qsg_ctx* ctx, const qsg_generator* G, int32_t n_c, const qsg_csr* c_ops,
                                  int32_t n_e, const qsg_csr* e_ops, int64_t d, const double* psi0,
                                  const double* tlist, int64_t n_t, const double* params, int32_t n_params,
                                  uint64_t seed, int64_t traj_begin, int64_t traj_end, const qsg_solve_opts* opts,
                                  qsg_mc_out* out, qsg_timing* timing) {
  QSG_RANGE("qsg_mcsolve");
  BatchProblem P{};
  if (qsg_status s = common_setup(ctx, G, d, tlist, n_t, opts, P)) return s;
  if (traj_end <= traj_begin) {
    set_error("InvalidGrid: ntraj must be >= 1");
    return QSG_INVALID_GRID;
  }
  if (n_c > kBatchMaxCops || n_e > kBatchMaxEops) {
    set_error("TooLarge: mcsolve supports at most 24 collapse and 8 expectation operators");
    return QSG_TOO_LARGE;
  }
  cudaStream_t s = ctx->stream;
  cudaError_t ce;
  P.mode = 0;
  P.d = static_cast<int>(d);
  P.eps_t = 1e-12 * std::max(1.0, std::fabs(P.tf));  // trajectories.cpp:130
  P.seed = seed;
  P.sys_begin = traj_begin;
  TmpOps keep;
  for (int k = 0; k < n_c; ++k) {
    if (c_ops[k].n_rows != d || c_ops[k].n_cols != d) {
      set_error("DimsMismatch: collapse operator dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
    if (qsg_status st = make_sell(ctx, c_ops[k], keep, P.c_ops[k])) return st;
  }
  for (int e = 0; e < n_e; ++e) {
    if (e_ops[e].n_rows != d || e_ops[e].n_cols != d) {
      set_error("DimsMismatch: e_op dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
    if (qsg_status st = make_sell(ctx, e_ops[e], keep, P.e_ops[e])) return st;
  }
  P.n_c = n_c;
  P.n_e = n_e;
  DevBuf dy0, dt, dp;
  if ((ce = upload(dy0, psi0, sizeof(double2) * d, s)) || (ce = upload(dt, tlist, sizeof(double) * n_t, s)) ||
      (n_params > 0 && (ce = upload(dp, params, sizeof(double) * n_params, s))))
    return cuda_fail(ce, "mcsolve inputs");
  P.y0 = dy0.as<double2>();
  P.tlist = dt.as<double>();
  P.params = n_params > 0 ? dp.as<double>() : nullptr;
  P.n_params = n_params;
  const long long nsys = traj_end - traj_begin;
  const int cap = static_cast<int>(std::max<int64_t>(1, out ? out->jump_capacity : 1));
  const size_t nv = static_cast<size_t>(n_e) * n_t;
  RunOut o;
  SumReq req;
  std::vector<long long> rlo, rhi;
  req.on = nv > 0;
  req.nv = static_cast<long long>(nv);
  if (out && out->n_ranges > 0) {  // the caller's sub-ranges, then the whole list for block_sum
    rlo.assign(out->range_lo, out->range_lo + out->n_ranges);
    rhi.assign(out->range_hi, out->range_hi + out->n_ranges);
    rlo.push_back(0);
    rhi.push_back(-1);
    req.n_ranges = out->n_ranges + 1;
    req.lo = rlo.data();
    req.hi = rhi.data();
  }
  const bool want_expect = out && out->per_traj_expect;
  if (qsg_status st = run_batch(ctx, P, nsys, std::max(cap, 64), o, want_expect, req)) return st;
  const int run_cap = std::max(cap, 64);
  long long n_ok = 0;
  for (long long i = 0; i < nsys; ++i) {
    const bool ok = o.status[i] == kDone;
    if (out) {
      if (out->failed) out->failed[i] = ok ? 0 : o.status[i];
      if (out->fail_time) out->fail_time[i] = o.ftime[i];
      if (out->traj_stats)
        for (int k = 0; k < 3; ++k) out->traj_stats[3 * i + k] = o.stats[3 * i + k];
      if (out->jump_count) out->jump_count[i] = o.jcount[i];
      // the device records min(jcount, run_cap) >= min(jcount, cap) jumps; jump_count keeps the full
      // count, so a caller whose buffer was too small sees jump_count > jump_capacity and re-calls
      const double* jt = o.jtime.data() + i * run_cap;
      const int* jc = o.jch.data() + i * run_cap;
      const int nstore = std::min(cap, o.jcount[i]);
      for (int j = 0; j < nstore; ++j) {
        if (out->jump_time) out->jump_time[i * cap + j] = jt[j];
        if (out->jump_channel) out->jump_channel[i * cap + j] = jc[j];
      }
      if (want_expect && nv > 0)
        std::copy(reinterpret_cast<const double*>(o.expect.data() + i * nv),
                  reinterpret_cast<const double*>(o.expect.data() + (i + 1) * nv), out->per_traj_expect + 2 * i * nv);
    }
    n_ok += ok ? 1 : 0;
  }
  if (out && out->n_ok) *out->n_ok = n_ok;
  if (out && nv > 0) {  // sums from the device bracket (zeros when nothing completed)
    const double* sums = reinterpret_cast<const double*>(o.sums.data());
    const int nr = out->n_ranges > 0 ? out->n_ranges : 0;
    if (nr > 0 && out->range_sums) std::copy(sums, sums + 2 * nv * nr, out->range_sums);
    if (out->block_sum) std::copy(sums + 2 * nv * nr, sums + 2 * nv * (nr + 1), out->block_sum);
  }
  if (timing) {
    timing->kernel_ms = o.kernel_ms;
    timing->attempts = o.attempts;
    timing->grid_ctas = o.grid;
    timing->lanes = batch_slots(o.layout);
  }
  return QSG_OK;
}

extern "C" qsg_status qsg_mesolve_batch(qsg_ctx* ctx, const qsg_generator* L, int64_t d, const double* rho0,
                                        const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                                        int64_t n_points, const double* params, int32_t n_params,
                                        const qsg_solve_opts* opts, double* expect, qsg_stats* stats,
                                        int32_t* status, qsg_timing* timing) {
  QSG_RANGE("qsg_mesolve_batch");
  BatchProblem P{};
  if (qsg_status s = common_setup(ctx, L, d * d, tlist, n_t, opts, P)) return s;
  if (n_points < 1) {
    set_error("InvalidGrid: need at least one parameter point");
    return QSG_INVALID_GRID;
  }
  if (n_e > kBatchMaxEops) {
    set_error("TooLarge: at most 8 e_ops per sweep");
    return QSG_TOO_LARGE;
  }
  cudaStream_t s = ctx->stream;
  cudaError_t ce;
  P.mode = 1;
  P.d = static_cast<int>(d);
  P.eps_t = 1e-12 * std::max({1.0, std::fabs(P.tf), std::fabs(P.t0)});  // evolve.cpp:128
  std::vector<int> eo_off(1, 0), eo_i, eo_j;
  std::vector<double> eo_v;
  for (int e = 0; e < n_e; ++e) {
    const qsg_csr& A = e_ops[e];
    if (A.n_rows != d || A.n_cols != d) {
      set_error("DimsMismatch: e_ops dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
    for (long long r = 0; r < A.n_rows; ++r)
      for (int p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
        eo_i.push_back(static_cast<int>(r));
        eo_j.push_back(A.col[p]);
        eo_v.push_back(A.val[2 * p]);
        eo_v.push_back(A.val[2 * p + 1]);
      }
    eo_off.push_back(static_cast<int>(eo_i.size()));
  }
  DevBuf dy0, dt, dp, a, b, c, v;
  if ((ce = upload(dy0, rho0, sizeof(double2) * d * d, s)) || (ce = upload(dt, tlist, sizeof(double) * n_t, s)) ||
      (ce = upload(dp, params, sizeof(double) * std::max<long long>(1, n_points * n_params), s)) ||
      (ce = upload(a, eo_off.data(), sizeof(int) * eo_off.size(), s)) ||
      (ce = upload(b, eo_i.data(), sizeof(int) * eo_i.size(), s)) ||
      (ce = upload(c, eo_j.data(), sizeof(int) * eo_j.size(), s)) ||
      (ce = upload(v, eo_v.data(), sizeof(double) * eo_v.size(), s)))
    return cuda_fail(ce, "sweep inputs");
  P.y0 = dy0.as<double2>();
  P.tlist = dt.as<double>();
  P.params = n_params > 0 ? dp.as<double>() : nullptr;
  P.n_params = n_params;
  P.n_e = n_e;
  P.eo_off = a.as<int>();
  P.eo_i = b.as<int>();
  P.eo_j = c.as<int>();
  P.eo_v = v.as<double2>();
  P.sys_begin = 0;
  RunOut o;
  if (qsg_status st = run_batch(ctx, P, n_points, 1, o)) return st;
  const size_t nv = static_cast<size_t>(n_e) * n_t;
  qsg_status rc = QSG_OK;
  for (long long i = 0; i < n_points; ++i) {
    if (expect)
      std::copy(reinterpret_cast<const double*>(o.expect.data() + i * nv),
                reinterpret_cast<const double*>(o.expect.data() + (i + 1) * nv), expect + 2 * i * nv);
    if (stats) stats[i] = qsg_stats{o.stats[3 * i], o.stats[3 * i + 1], o.stats[3 * i + 2]};
    if (status) status[i] = o.status[i] == kDone ? 0 : QSG_INTEGRATION_FAILURE;
    if (o.status[i] != kDone && rc == QSG_OK) rc = status_from_device(o.status[i], o.ftime[i]);
  }
  if (timing) {
    timing->kernel_ms = o.kernel_ms;
    timing->attempts = o.attempts;
    timing->grid_ctas = o.grid;
    timing->lanes = batch_slots(o.layout);
  }
  return status ? QSG_OK : rc;
}
