// Stochastic Schroedinger / master equations with Euler-Maruyama (ssesolve / smesolve,
// trajectories.cpp:251-503), batched one trajectory per CTA. A persistent grid pulls trajectories
// from a queue; trajectory i draws its Wiener increments from RngStream(seed, i) (Box-Muller with
// the cached second normal, rng.cpp:49-61), so results do not depend on the CTA that ran it.
//
// Per Euler-Maruyama step (fixed dt, make_em_grid trajectories.cpp:261-275):
//   SSE  pass A: e_c = Re <psi| X_c psi> for every channel (X = S + S^dag); thread 0 draws dW_c.
//        pass B: drift = -iH(t) psi and the channel terms, combined per element in the
//                reference's order (single-channel fast path :313-326, general path :327-347);
//                |psi_new|^2 partials.   pass C: psi = psi_new / |psi_new|.
//   SME  pass A: rho_new = rho + dt L(t) rho; srho_c = S_c rho; e_c = Re tr(srho_c + srho_c^dag).
//        pass B: rho_new += dW_c (srho_c + srho_c^dag - e_c rho)   (:448-456)
//        pass C: rho = (rho_new + rho_new^dag) / 2 with its trace;  pass D: rho /= Re tr(rho).
// Observations at every tlist point (psi.dot(E psi) :304-309; sum E(r,c) rho(c,r) :429-437).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "qsg_internal.h"
#include "../../include/qsim/qobj.hpp"

namespace qsg {
namespace {

constexpr int kSdeThreads = 256;
constexpr int kSdeMaxCh = 8;
constexpr int kSdeMaxE = 8;

struct SdeProblem {
  int mode;  // 0 SSE (vector length d), 1 SME (vector length d*d)
  int n, d;
  DevGen gen;
  const double* params;
  int n_ch;
  DevSell S[kSdeMaxCh], SdS[kSdeMaxCh], X[kSdeMaxCh];  // SSE: S, S^dag S, S + S^dag; SME: S (plain)
  int n_e;
  DevSell E[kSdeMaxE];  // SSE observations
  const int* eo_off;    // SME observations: entries (i, j, v) of every E
  const int* eo_i;
  const int* eo_j;
  const double2* eo_v;
  const double2* y0;
  const double* tlist;
  int n_t, sub;
  long long n_steps;
  double dt, sqrt_dt, t0;
  unsigned long long seed;
  long long sys_begin, n_sys;
  double2* work;
  long long work_stride;
  unsigned long long* queue;
  double2* expect;  // n_sys x (n_e x n_t)
  double* winc;     // n_sys x (n_ch x n_steps) or null
  double* wexp;
  double* wcur;
};

struct Rng {
  unsigned long long s[4];
  double cached;
  int has_cached;
};
__device__ __forceinline__ unsigned long long rotl(unsigned long long x, int k) { return (x << k) | (x >> (64 - k)); }
__device__ void rng_seed(Rng& r, unsigned long long seed, unsigned long long stream) {  // rng.cpp:14-25
  unsigned long long z = seed ^ ((stream + 1) * 0x9E3779B97F4A7C15ULL);
  for (int i = 0; i < 4; ++i) {
    unsigned long long x = (z += 0x9E3779B97F4A7C15ULL);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    r.s[i] = x ^ (x >> 31);
  }
  if ((r.s[0] | r.s[1] | r.s[2] | r.s[3]) == 0) r.s[0] = 1;
  r.has_cached = 0;
  r.cached = 0.0;
}
__device__ unsigned long long rng_u64(Rng& r) {  // rng.cpp:27-37
  const unsigned long long result = rotl(r.s[0] + r.s[3], 23) + r.s[0];
  const unsigned long long t = r.s[1] << 17;
  r.s[2] ^= r.s[0];
  r.s[3] ^= r.s[1];
  r.s[1] ^= r.s[2];
  r.s[0] ^= r.s[3];
  r.s[2] ^= t;
  r.s[3] = rotl(r.s[3], 45);
  return result;
}
__device__ double rng_uniform(Rng& r) { return static_cast<double>(rng_u64(r) >> 11) * 0x1.0p-53; }
__device__ double rng_normal(Rng& r) {  // rng.cpp:49-61
  if (r.has_cached) {
    r.has_cached = 0;
    return r.cached;
  }
  double u1 = rng_uniform(r);
  while (u1 == 0.0) u1 = rng_uniform(r);
  const double u2 = rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double phi = 2.0 * 3.141592653589793 * u2;
  r.cached = rr * sin(phi);
  r.has_cached = 1;
  return rr * cos(phi);
}

// row `row` of a plain SELL operator applied to a gathered vector (any row, not lane-aligned)
template <class XF>
__device__ __forceinline__ double2 sell_row_at(const DevSell& A, int row, XF&& xf) {
  const int sl = row >> 5, ln = row & 31;
  const int len = __ldg(A.rowlen + row);
  const long long base = __ldg(A.slice_off + sl) * 32 + ln;
  double2 acc = make_double2(0.0, 0.0);
  for (int j = 0; j < len; ++j) cfma(__ldg(A.val + base + 32LL * j), xf(__ldg(A.col + base + 32LL * j)), acc);
  return acc;
}

// T threads per trajectory: one warp for small systems (many trajectories per SM, cheap barriers),
// 256 for large ones.
template <int MODE, int T>
__global__ void __launch_bounds__(T) sde_kernel(const __grid_constant__ SdeProblem P) {
  __shared__ double s_red[T / 32];
  __shared__ double s_e[kSdeMaxCh], s_dw[kSdeMaxCh];
  __shared__ long long s_sys;
  __shared__ double s_scale;
  const int W = T / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n, d = P.d, nsl = (n + 31) >> 5;
  double2* psi = P.work + static_cast<long long>(blockIdx.x) * P.work_stride;
  double2* pn = psi + n;      // SSE psi_new / SME rho_new
  double2* sr = psi + 2 * n;  // SME S_c rho, n_ch arrays
  Rng rng;                    // thread 0 only
  auto rows = [&](auto&& f) {
    for (int b = warp; b < nsl; b += W) f(b, (b << 5) + lane);
  };
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long q = atomicAdd(P.queue, 1ull);
      s_sys = q < static_cast<unsigned long long>(P.n_sys) ? static_cast<long long>(q) : -1;
    }
    __syncthreads();
    const long long sys = s_sys;
    if (sys < 0) return;
    if (threadIdx.x == 0) rng_seed(rng, P.seed, static_cast<unsigned long long>(P.sys_begin + sys));
    for (int r = threadIdx.x; r < n; r += blockDim.x) psi[r] = P.y0[r];
    __syncthreads();
    auto observe = [&](int k) {
      for (int e = 0; e < P.n_e; ++e) {
        double ar = 0.0, ai = 0.0;
        if (MODE == 0) {  // psi.dot(E psi) = sum conj(psi_r) (E psi)_r
          rows([&](int b, int r) {
            const double2 v = sell_row(P.E[e], b, lane, [&](int c) { return psi[c]; });
            if (r < n) {
              const double2 p = psi[r];
              ar += p.x * v.x + p.y * v.y;
              ai += p.x * v.y - p.y * v.x;
            }
          });
        } else {  // sum_{(i,j) in E} E(i,j) rho(j,i)
          for (int q = P.eo_off[e] + threadIdx.x; q < P.eo_off[e + 1]; q += blockDim.x) {
            const double2 v = cmul(P.eo_v[q], psi[P.eo_j[q] + d * P.eo_i[q]]);
            ar += v.x;
            ai += v.y;
          }
        }
        ar = block_sum(ar, s_red);
        ai = block_sum(ai, s_red);
        if (threadIdx.x == 0)
          P.expect[(sys * P.n_e + 0) * P.n_t + static_cast<long long>(k) * P.n_e + e] = make_double2(ar, ai);
      }
    };
    observe(0);
    long long step = 0;
    for (int k = 1; k < P.n_t; ++k) {
      for (int s = 0; s < P.sub; ++s, ++step) {
        const double t = P.t0 + P.dt * static_cast<double>(step);
        // ---- pass A: channel expectations
        for (int c = 0; c < P.n_ch; ++c) {
          double a = 0.0;
          if (MODE == 0) {
            rows([&](int b, int r) {
              const double2 v = sell_row(P.X[c], b, lane, [&](int cc) { return psi[cc]; });
              if (r < n) a += psi[r].x * v.x + psi[r].y * v.y;
            });
          } else {
            for (int i = threadIdx.x; i < d; i += blockDim.x) {  // diagonal of S rho: (S rho)(i,i)
              const double2 v = sell_row_at(P.S[c], i, [&](int kk) { return psi[kk + d * i]; });
              a += v.x + v.x;
            }
          }
          a = block_sum(a, s_red);
          if (threadIdx.x == 0) s_e[c] = a;
        }
        if (MODE == 1) {  // rho_new = rho + dt L rho; srho_c = S_c rho
          rows([&](int b, int r) {
            const double2 g = gen_row(P.gen, P.params, b, t, [&](int c) { return psi[c]; });
            if (r < n) {
              const double2 p = psi[r];
              pn[r] = make_double2(p.x + P.dt * g.x, p.y + P.dt * g.y);
              const int i = r % d, j = r / d;
              for (int c = 0; c < P.n_ch; ++c)
                sr[static_cast<long long>(c) * n + r] = sell_row_at(P.S[c], i, [&](int kk) { return psi[kk + d * j]; });
            }
          });
        }
        if (threadIdx.x == 0)
          for (int c = 0; c < P.n_ch; ++c) {
            s_dw[c] = P.sqrt_dt * rng_normal(rng);
            if (P.winc) {
              const long long idx = (sys * P.n_ch + 0) * P.n_steps + step * P.n_ch + c;
              P.winc[idx] = s_dw[c];
              P.wexp[idx] = s_e[c];
              P.wcur[idx] = s_e[c] + s_dw[c] / P.dt;
            }
          }
        __syncthreads();
        if (MODE == 0) {
          // ---- pass B: drift and update, then |psi_new|^2
          double nrm = 0.0;
          const double dt = P.dt;
          rows([&](int b, int r) {
            double2 drift = gen_row(P.gen, P.params, b, t, [&](int c) { return psi[c]; });
            if (P.n_ch == 1) {
              const double2 st = sell_row(P.S[0], b, lane, [&](int c) { return psi[c]; });
              const double2 tm = sell_row(P.SdS[0], b, lane, [&](int c) { return psi[c]; });
              if (r < n) {
                const double e_n = s_e[0], dw0 = s_dw[0];
                const double c1 = dt * 0.5 * e_n + dw0, c2 = dt * 0.5;
                const double c3 = dt * 0.125 * e_n * e_n + 0.5 * e_n * dw0;
                const double2 p = psi[r];
                double2 v;
                v.x = ((dt * drift.x + c1 * st.x) - c2 * tm.x) - c3 * p.x;
                v.y = ((dt * drift.y + c1 * st.y) - c2 * tm.y) - c3 * p.y;
                const double2 q = make_double2(p.x + v.x, p.y + v.y);
                pn[r] = q;
                nrm += q.x * q.x + q.y * q.y;
              }
            } else {
              double2 stoch = make_double2(0.0, 0.0);
              const double2 p = r < n ? psi[r] : make_double2(0.0, 0.0);
              for (int c = 0; c < P.n_ch; ++c) {
                const double e_n = s_e[c], dw = s_dw[c];
                const double2 tm = sell_row(P.S[c], b, lane, [&](int cc) { return psi[cc]; });
                const double a = 0.5 * e_n, bb = 0.5 * e_n * dw;
                drift = make_double2(drift.x + a * tm.x, drift.y + a * tm.y);
                stoch = make_double2(stoch.x + dw * tm.x, stoch.y + dw * tm.y);
                stoch = make_double2(stoch.x - bb * p.x, stoch.y - bb * p.y);
                const double2 t2 = sell_row(P.SdS[c], b, lane, [&](int cc) { return psi[cc]; });
                const double qq = 0.125 * e_n * e_n;
                drift = make_double2(drift.x - 0.5 * t2.x, drift.y - 0.5 * t2.y);
                drift = make_double2(drift.x - qq * p.x, drift.y - qq * p.y);
              }
              if (r < n) {
                const double2 q = make_double2(p.x + (dt * drift.x + stoch.x), p.y + (dt * drift.y + stoch.y));
                pn[r] = q;
                nrm += q.x * q.x + q.y * q.y;
              }
            }
          });
          nrm = block_sum(nrm, s_red);
          if (threadIdx.x == 0) s_scale = sqrt(nrm);
          __syncthreads();
          const double sc = s_scale;
          for (int r = threadIdx.x; r < n; r += blockDim.x) {  // pass C: psi /= psi.norm()
            const double2 q = pn[r];
            psi[r] = make_double2(q.x / sc, q.y / sc);
          }
          __syncthreads();
        } else {
          // ---- pass B: rho_new += dW_c (S rho + (S rho)^dag - e_c rho), channel by channel
          for (int r = threadIdx.x; r < n; r += blockDim.x) {
            const int i = r % d, j = r / d, rt = j + d * i;
            double2 q = pn[r];
            const double2 p = psi[r];
            for (int c = 0; c < P.n_ch; ++c) {
              const double2 a = sr[static_cast<long long>(c) * n + r], bt = sr[static_cast<long long>(c) * n + rt];
              double2 hop = make_double2(a.x + bt.x, a.y - bt.y);
              hop = make_double2(hop.x - s_e[c] * p.x, hop.y - s_e[c] * p.y);
              q = make_double2(q.x + s_dw[c] * hop.x, q.y + s_dw[c] * hop.y);
            }
            pn[r] = q;
          }
          __syncthreads();
          // ---- pass C: rho = 0.5 (rho_new + rho_new^dag), trace
          double tr = 0.0;
          for (int r = threadIdx.x; r < n; r += blockDim.x) {
            const int i = r % d, j = r / d;
            const double2 a = pn[r], bt = pn[j + d * i];
            const double2 h = make_double2(0.5 * (a.x + bt.x), 0.5 * (a.y - bt.y));
            psi[r] = h;
            if (i == j) tr += h.x;
          }
          tr = block_sum(tr, s_red);
          if (threadIdx.x == 0) s_scale = tr;
          __syncthreads();
          const double sc = s_scale;
          for (int r = threadIdx.x; r < n; r += blockDim.x) {  // pass D: rho /= Re tr(rho)
            const double2 h = psi[r];
            psi[r] = make_double2(h.x / sc, h.y / sc);
          }
          __syncthreads();
        }
      }
      observe(k);
    }
    __syncthreads();
  }
}

using qsim::Complex;
using qsim::SparseMatrix;

SparseMatrix host_sparse(const qsg_csr& a) {
  SparseMatrix m;
  m.rows = a.n_rows;
  m.cols = a.n_cols;
  m.rowptr.assign(a.rowptr, a.rowptr + a.n_rows + 1);
  m.col.assign(a.col, a.col + a.nnz);
  const Complex* v = reinterpret_cast<const Complex*>(a.val);
  m.val.assign(v, v + a.nnz);
  return m;
}
qsg_csr view_of(const SparseMatrix& m) {
  return qsg_csr{m.rows, m.cols, static_cast<int64_t>(m.val.size()), m.rowptr.data(), m.col.data(),
                 reinterpret_cast<const double*>(m.val.data())};
}

struct OwnedOps {
  std::vector<qsg_op*> ops;
  ~OwnedOps() {
    for (auto* o : ops) qsg_op_destroy(o);
  }
};

// pairwise_sum over [lo, hi) of trajectory matrices (trajectories.cpp:17-22)
void pairwise(const std::vector<const double2*>& m, size_t lo, size_t hi, size_t nv, double2* out) {
  if (hi - lo == 1) {
    std::memcpy(out, m[lo], nv * sizeof(double2));
    return;
  }
  const size_t mid = lo + (hi - lo) / 2;
  std::vector<double2> r(nv);
  pairwise(m, lo, mid, nv, out);
  pairwise(m, mid, hi, nv, r.data());
  for (size_t i = 0; i < nv; ++i) out[i] = make_double2(out[i].x + r[i].x, out[i].y + r[i].y);
}

qsg_status run_sde(qsg_ctx* ctx, int mode, const qsg_generator* G, int64_t d, int32_t n_sc, const qsg_csr* sc_ops,
                   int32_t n_e, const qsg_csr* e_ops, const double* y0_in, const double* tlist, int64_t n_t,
                   const double* params, int32_t n_params, uint64_t seed, int64_t traj_begin, int64_t traj_end,
                   double dt_max, int32_t store_meas, qsg_sde_out* out, qsg_timing* timing) {
  if (!ctx || !G || !out || !tlist) {
    set_error("InvalidGrid: null argument");
    return QSG_INVALID_GRID;
  }
  if (qsg_status s = check_tlist(tlist, n_t)) return s;
  const double spacing = tlist[1] - tlist[0];
  for (int64_t i = 2; i < n_t; ++i)  // trajectories.cpp:264-266
    if (std::abs((tlist[i] - tlist[i - 1]) - spacing) > 1e-9 * spacing) {
      set_error("InvalidGrid: stochastic solvers need a uniform tlist");
      return QSG_INVALID_GRID;
    }
  if (n_sc < 0 || n_sc > kSdeMaxCh || n_e < 0 || n_e > kSdeMaxE) {
    set_error("TooLarge: stochastic solvers support at most 8 measurement channels and 8 e_ops");
    return QSG_TOO_LARGE;
  }
  const long long n_sys = traj_end - traj_begin;
  if (n_sys < 1) {
    set_error("InvalidGrid: ntraj must be >= 1");
    return QSG_INVALID_GRID;
  }
  const long long n = mode == 0 ? d : d * d;
  if (qsg_status s = check_generator(G, n)) return s;
  for (int c = 0; c < n_sc; ++c)
    if (sc_ops[c].n_rows != d || sc_ops[c].n_cols != d) {
      set_error("DimsMismatch: sc_op dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
  for (int e = 0; e < n_e; ++e)
    if (e_ops[e].n_rows != d || e_ops[e].n_cols != d) {
      set_error("DimsMismatch: e_op dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
  // make_em_grid (trajectories.cpp:261-275)
  const double span = tlist[n_t - 1] - tlist[0];
  const double dtm = dt_max <= 0.0 ? span / 1e4 : dt_max;
  const long sub = std::max(1L, static_cast<long>(std::ceil(spacing / dtm * (1.0 - 1e-12))));
  const double dt = spacing / static_cast<double>(sub);
  const long long n_steps = static_cast<long long>(sub) * (n_t - 1);
  out->n_steps = n_steps;
  out->dt = dt;

  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  cudaError_t ce;
  SdeProblem P{};
  P.mode = mode;
  P.n = static_cast<int>(n);
  P.d = static_cast<int>(d);
  P.gen = make_devgen(G);
  P.n_ch = n_sc;
  P.n_e = n_e;
  OwnedOps keep;
  std::vector<SparseMatrix> mats;
  mats.reserve(static_cast<size_t>(3 * n_sc + n_e));
  auto mk = [&](const SparseMatrix& m, DevSell& dst, bool codes) -> qsg_status {
    mats.push_back(m);
    const qsg_csr v = view_of(mats.back());
    qsg_op* op = nullptr;
    if (qsg_status st = qsg_op_create(ctx, &v, &op)) return st;
    keep.ops.push_back(op);
    dst = sell_view(op, codes);
    return QSG_OK;
  };
  for (int c = 0; c < n_sc; ++c) {
    const SparseMatrix sm = host_sparse(sc_ops[c]);
    if (qsg_status st = mk(sm, P.S[c], mode == 0)) return st;
    if (mode == 0) {  // S^dag S and S + S^dag in the reference's arithmetic (trajectories.cpp:382-384)
      const SparseMatrix sd = qsim::sparse_transpose(sm, true);
      if (qsg_status st = mk(qsim::sparse_mul(sd, sm), P.SdS[c], true)) return st;
      if (qsg_status st = mk(qsim::sparse_add(sm, sd), P.X[c], true)) return st;
    }
  }
  DevBuf d_eoff, d_ei, d_ej, d_ev;
  if (mode == 0) {
    for (int e = 0; e < n_e; ++e)
      if (qsg_status st = mk(host_sparse(e_ops[e]), P.E[e], true)) return st;
  } else {
    std::vector<int> off(1, 0), ei, ej;
    std::vector<double2> ev;
    for (int e = 0; e < n_e; ++e) {
      const qsg_csr& A = e_ops[e];
      for (long long r = 0; r < A.n_rows; ++r)
        for (int p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
          ei.push_back(static_cast<int>(r));
          ej.push_back(A.col[p]);
          ev.push_back(make_double2(A.val[2 * p], A.val[2 * p + 1]));
        }
      off.push_back(static_cast<int>(ei.size()));
    }
    if ((ce = upload(d_eoff, off.data(), sizeof(int) * off.size(), s)) ||
        (ce = upload(d_ei, ei.data(), sizeof(int) * std::max<size_t>(1, ei.size()), s)) ||
        (ce = upload(d_ej, ej.data(), sizeof(int) * std::max<size_t>(1, ej.size()), s)) ||
        (ce = upload(d_ev, ev.data(), sizeof(double2) * std::max<size_t>(1, ev.size()), s)))
      return cuda_fail(ce, "e_ops");
    P.eo_off = d_eoff.as<int>();
    P.eo_i = d_ei.as<int>();
    P.eo_j = d_ej.as<int>();
    P.eo_v = d_ev.as<double2>();
  }
  // initial state: SSE normalises psi0 (trajectories.cpp:388-389); SME takes rho0 as given
  std::vector<double2> y0(static_cast<size_t>(n));
  if (is_device_ptr(y0_in)) cudaMemcpy(y0.data(), y0_in, sizeof(double2) * n, cudaMemcpyDefault);
  else std::memcpy(y0.data(), y0_in, sizeof(double2) * n);
  if (mode == 0) {
    double sq = 0.0;
    for (const auto& v : y0) sq += v.x * v.x + v.y * v.y;
    const double nrm = std::sqrt(sq);
    for (auto& v : y0) v = make_double2(v.x / nrm, v.y / nrm);
  }
  DevBuf d_y0, d_t, d_p, d_q, d_ex, d_wi, d_we, d_wc, d_work;
  if ((ce = upload(d_y0, y0.data(), sizeof(double2) * n, s)) ||
      (ce = upload(d_t, tlist, sizeof(double) * n_t, s)) || (ce = d_q.alloc(8, s)))
    return cuda_fail(ce, "inputs");
  if (n_params > 0) {
    if ((ce = upload(d_p, params, sizeof(double) * n_params, s))) return cuda_fail(ce, "params");
    P.params = d_p.as<double>();
  }
  cudaMemsetAsync(d_q.p, 0, 8, s);
  const size_t nvals = static_cast<size_t>(std::max(1, static_cast<int>(n_e))) * n_t;
  if ((ce = d_ex.alloc(sizeof(double2) * nvals * n_sys, s))) return cuda_fail(ce, "expect");
  cudaMemsetAsync(d_ex.p, 0, sizeof(double2) * nvals * n_sys, s);
  const size_t nw = static_cast<size_t>(n_sys) * n_sc * n_steps;
  if (store_meas && n_sc > 0) {
    if ((ce = d_wi.alloc(sizeof(double) * nw, s)) || (ce = d_we.alloc(sizeof(double) * nw, s)) ||
        (ce = d_wc.alloc(sizeof(double) * nw, s)))
      return cuda_fail(ce, "Wiener records");
    P.winc = d_wi.as<double>();
    P.wexp = d_we.as<double>();
    P.wcur = d_wc.as<double>();
  }
  // threads per trajectory, measured on JC N=10 (scripts/probe_sde.py): SSE (n = 20) one warp
  // 35.2k traj/s vs 9.8k at 256 threads; SME (n = 400) 512 threads 3.43k vs 2.83k at 256, 0.70k at 32
  int threads = n <= 256 ? 32 : 512;
  if (const char* e = std::getenv("QSG_SDE_THREADS")) {
    const int v = std::atoi(e);
    threads = v == 32 || v == 128 || v == 512 ? v : kSdeThreads;
  }
  const void* kfn = mode == 0 ? (threads == 32    ? reinterpret_cast<const void*>(sde_kernel<0, 32>)
                                 : threads == 128 ? reinterpret_cast<const void*>(sde_kernel<0, 128>)
                                 : threads == 512 ? reinterpret_cast<const void*>(sde_kernel<0, 512>)
                                                  : reinterpret_cast<const void*>(sde_kernel<0, kSdeThreads>))
                              : (threads == 32    ? reinterpret_cast<const void*>(sde_kernel<1, 32>)
                                 : threads == 128 ? reinterpret_cast<const void*>(sde_kernel<1, 128>)
                                 : threads == 512 ? reinterpret_cast<const void*>(sde_kernel<1, 512>)
                                                  : reinterpret_cast<const void*>(sde_kernel<1, kSdeThreads>));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, 0);
  if (per_sm <= 0) return cuda_fail(cudaGetLastError(), "occupancy");
  const long long stride = (mode == 0 ? 2 : 2 + n_sc) * n;
  int grid = static_cast<int>(std::min<long long>(static_cast<long long>(per_sm) * ctx->sm_count, n_sys));
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
    const long long fit = static_cast<long long>(fr / 10 * 6 / (stride * sizeof(double2)));
    if (fit < 1) {
      set_error("OutOfMemory: trajectory workspace does not fit on the device");
      return QSG_OUT_OF_MEMORY;
    }
    grid = static_cast<int>(std::min<long long>(grid, fit));
  }
  if ((ce = d_work.alloc(sizeof(double2) * stride * grid, s))) return cuda_fail(ce, "workspace");
  P.y0 = d_y0.as<double2>();
  P.tlist = d_t.as<double>();
  P.n_t = static_cast<int>(n_t);
  P.sub = static_cast<int>(sub);
  P.n_steps = n_steps;
  P.dt = dt;
  P.sqrt_dt = std::sqrt(dt);
  P.t0 = tlist[0];
  P.seed = seed;
  P.sys_begin = traj_begin;
  P.n_sys = n_sys;
  P.work = d_work.as<double2>();
  P.work_stride = stride;
  P.queue = d_q.as<unsigned long long>();
  P.expect = d_ex.as<double2>();
  cudaEventRecord(ctx->ev[2], s);
  if (mode == 0 && threads == 32) sde_kernel<0, 32><<<grid, 32, 0, s>>>(P);
  else if (mode == 0 && threads == 128) sde_kernel<0, 128><<<grid, 128, 0, s>>>(P);
  else if (mode == 0 && threads == 512) sde_kernel<0, 512><<<grid, 512, 0, s>>>(P);
  else if (mode == 0) sde_kernel<0, kSdeThreads><<<grid, kSdeThreads, 0, s>>>(P);
  else if (threads == 32) sde_kernel<1, 32><<<grid, 32, 0, s>>>(P);
  else if (threads == 128) sde_kernel<1, 128><<<grid, 128, 0, s>>>(P);
  else if (threads == 512) sde_kernel<1, 512><<<grid, 512, 0, s>>>(P);
  else sde_kernel<1, kSdeThreads><<<grid, kSdeThreads, 0, s>>>(P);
  if ((ce = cudaGetLastError())) return cuda_fail(ce, "stochastic launch");
  cudaEventRecord(ctx->ev[3], s);
  std::vector<double2> ex(nvals * n_sys);
  if ((ce = cudaMemcpyAsync(ex.data(), d_ex.p, sizeof(double2) * ex.size(), cudaMemcpyDeviceToHost, s)) ||
      (ce = cudaStreamSynchronize(s)))
    return cuda_fail(ce, "stochastic solve");
  if (store_meas && n_sc > 0) {
    if (out->w_increments) cudaMemcpyAsync(out->w_increments, d_wi.p, sizeof(double) * nw, cudaMemcpyDefault, s);
    if (out->w_expectation) cudaMemcpyAsync(out->w_expectation, d_we.p, sizeof(double) * nw, cudaMemcpyDefault, s);
    if (out->w_current) cudaMemcpyAsync(out->w_current, d_wc.p, sizeof(double) * nw, cudaMemcpyDefault, s);
    if ((ce = cudaStreamSynchronize(s))) return cuda_fail(ce, "Wiener records");
  }
  if (timing) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
    timing->kernel_ms = ms;
    timing->attempts = n_steps * n_sys;
    timing->grid_ctas = grid;
    timing->lanes = 1;
  }
  // the device slab keeps max(1, n_e) rows per trajectory; the caller's buffers hold n_e * n_t
  // values per trajectory (nothing at all when there are no e_ops)
  const size_t nv = static_cast<size_t>(n_e) * n_t;
  if (nv > 0) {
    if (out->per_traj_expect) {
      double2* dst = reinterpret_cast<double2*>(out->per_traj_expect);
      for (long long i = 0; i < n_sys; ++i) std::memcpy(dst + nv * i, ex.data() + nvals * i, sizeof(double2) * nv);
    }
    std::vector<const double2*> blocks;
    for (long long i = 0; i < n_sys; ++i) blocks.push_back(ex.data() + nvals * i);
    if (out->block_sum) pairwise(blocks, 0, blocks.size(), nv, reinterpret_cast<double2*>(out->block_sum));
  }
  out->n_ok = n_sys;
  return QSG_OK;
}

}  // namespace
}  // namespace qsg

using namespace qsg;

extern "C" {

qsg_status qsg_ssesolve(qsg_ctx* ctx, const qsg_generator* G, int64_t d, int32_t n_sc, const qsg_csr* sc_ops,
                        int32_t n_e, const qsg_csr* e_ops, const double* psi0, const double* tlist, int64_t n_t,
                        const double* params, int32_t n_params, uint64_t seed, int64_t traj_begin,
                        int64_t traj_end, double dt_max, int32_t store_measurement, qsg_sde_out* out,
                        qsg_timing* timing) {
  QSG_RANGE("qsg_ssesolve");
  return run_sde(ctx, 0, G, d, n_sc, sc_ops, n_e, e_ops, psi0, tlist, n_t, params, n_params, seed, traj_begin,
                 traj_end, dt_max, store_measurement, out, timing);
}

qsg_status qsg_smesolve(qsg_ctx* ctx, const qsg_generator* L, int64_t d, int32_t n_sc, const qsg_csr* sc_ops,
                        int32_t n_e, const qsg_csr* e_ops, const double* rho0, const double* tlist, int64_t n_t,
                        const double* params, int32_t n_params, uint64_t seed, int64_t traj_begin,
                        int64_t traj_end, double dt_max, int32_t store_measurement, qsg_sde_out* out,
                        qsg_timing* timing) {
  QSG_RANGE("qsg_smesolve");
  return run_sde(ctx, 1, L, d, n_sc, sc_ops, n_e, e_ops, rho0, tlist, n_t, params, n_params, seed, traj_begin,
                 traj_end, dt_max, store_measurement, out, timing);
}

}  // extern "C"
