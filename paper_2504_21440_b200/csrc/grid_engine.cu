// Persistent cooperative Dormand-Prince 5(4) solver for ONE large system (mesolve / sesolve).
//
// One launch integrates the whole tlist: every CTA of a cooperative grid owns a contiguous
// range of 32-row SELL slices; the six RHS evaluations of an attempt (integrator.hpp:91-102) are
// fused SpMV passes whose epilogue forms the next stage input, the stage-7 pass also produces
// the embedded-error partials (integrator.hpp:105-116), and the accept/reject PI controller
// (integrator.hpp:119-145) runs redundantly — and identically — in every CTA after a
// deterministic grid reduction. Observations (evolve.cpp:160-165, 284-297) evaluate the Hairer
// dense output (integrator.hpp:127-131,150-154) lazily, only at the indices the e_ops touch,
// fused into the next attempt's first pass. No host round trip per step.
//
// Register budget: the integrator state lives in shared memory and is advanced by thread 0 of
// each CTA between barriers; the SpMV passes only hold the buffer pointers they touch, which
// keeps the kernel at <= 64 registers and 2 CTAs x 16 warps per SM for latency hiding.
//
// Passes per attempt: 6 (stage 2 gathers y + h*a21*k1 on the fly), one grid barrier each.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <type_traits>

#include "engine.cuh"
#include "grid_engine.h"

namespace qsg {

namespace {

#ifndef QSG_GRID_THREADS
#define QSG_GRID_THREADS 512
#endif
constexpr int kThreads = QSG_GRID_THREADS;
#ifndef QSG_GRID_MINB
#define QSG_GRID_MINB 2
#endif

struct Pending {
  double theta;  // NaN: observe buffer Y directly
  int grid_idx;  // -1: save-only
  int save_idx;  // -1: no state save
};

// logical buffer ids
enum { Y = 0, YO = 1, K1 = 2, K2 = 3, K3 = 4, K4 = 5, K5 = 6, K6 = 7, K7 = 8, SA = 9, SB = 10 };

// Integrator state of the solve — identical in every CTA, written by thread 0 only.
struct Ctl {
  double2* p[11];  // logical -> physical buffer (FSAL / y rotation, integrator.hpp:133-138)
  const double* ev_t;  // event times / grid index / save index (P.ev_*, or a shared-memory copy)
  const int* ev_grid;
  const int* ev_save;
  double t, t_old, h, h_last, facold, hh, h0, d1;
  double fail_t;
  long long steps, rejected, rhs_evals, attempts_total;
  int status, clamped, attempts, next, np, obs_par, flush, done;
  Pending pend[kMaxPending];
};

__device__ __forceinline__ double2 dense_at(double2* const* p, int c, double theta, double h) {
  // integrator.hpp:127-131 (rc1..rc5) and :150-154 (evaluation), per element. After an accepted
  // step the FSAL swap (:138) put the step's k1 under the K7 label and its k7 under K1.
  if (isnan(theta)) return p[Y][c];
  const double2 yo = p[YO][c];
  const double2 y1 = p[Y][c];
  const double2 k1 = p[K7][c];
  const double2 k7 = p[K1][c];
  const double2 k3 = p[K3][c], k4 = p[K4][c], k5 = p[K5][c], k6 = p[K6][c];
  using namespace dp;
  const double th1 = 1.0 - theta;
  const double2 rc2 = csub(y1, yo);
  const double2 rc3 = csub(cscale(h, k1), rc2);
  const double2 rc4 = csub(csub(rc2, cscale(h, k7)), rc3);
  double2 rc5;
  rc5.x = h * (d1 * k1.x + d3 * k3.x + d4 * k4.x + d5 * k5.x + d6 * k6.x + d7 * k7.x);
  rc5.y = h * (d1 * k1.y + d3 * k3.y + d4 * k4.y + d5 * k5.y + d6 * k6.y + d7 * k7.y);
  double2 o;
  o.x = yo.x + theta * (rc2.x + th1 * (rc3.x + theta * (rc4.x + th1 * rc5.x)));
  o.y = yo.y + theta * (rc2.y + th1 * (rc3.y + theta * (rc4.y + th1 * rc5.y)));
  return o;
}

// Observation pass for the pending events: expectation partials into reduction slots and state
// saves. ME: expect_e = sum_{(i,j) in A_e} A(i,j) * rho_h(j,i), rho_h = (rho + rho^dag)/2
// (evolve.cpp:286-295); SE: <psi|E psi> (evolve.cpp:341-345).
template <int MODE>
__device__ __noinline__ void observe_pass(const GridProblem& P, const Ctl& c, double* slots, double* smem,
                                          int rank, int G) {
  double2* const* p = c.p;
  const int np = c.np;
  const double h_last = c.h_last;
  const int gtid = rank * blockDim.x + threadIdx.x;
  const int gstride = G * blockDim.x;
  for (int e = 0; e < P.n_e; ++e) {
    for (int q = 0; q < np; ++q) {
      double2 acc = make_double2(0.0, 0.0);
      const double th = c.pend[q].theta;
      if (c.pend[q].grid_idx >= 0) {
        if (MODE == 0) {
          const int beg = P.eo_off[e], end = P.eo_off[e + 1];
          for (int k = beg + gtid; k < end; k += gstride) {
            const int i = P.eo_i[k], j = P.eo_j[k];
            const double2 rji = dense_at(p, i * P.d + j, th, h_last);  // rho(j,i) = y[i*d + j]
            const double2 rij = dense_at(p, j * P.d + i, th, h_last);  // rho(i,j) = y[j*d + i]
            const double2 rh = cscale(0.5, cadd(rji, cconj(rij)));
            acc = cadd(acc, cmul(P.eo_v[k], rh));
          }
        } else if (P.n_se_ops == P.n_e) {  // e_op operator stores (observe_se)
          for (int r = gtid; r < P.n; r += gstride) {
            const double2 ev =
                sell_row(P.se_ops[e], r >> 5, r & 31, [&](int col) { return dense_at(p, col, th, h_last); });
            acc = cadd(acc, cmul(cconj(dense_at(p, r, th, h_last)), ev));
          }
        } else {
          const int* rp = P.se_rowptr + static_cast<long long>(e) * (P.n + 1);
          const long long off = P.se_off[e];
          for (int r = gtid; r < P.n; r += gstride) {
            double2 ev = make_double2(0.0, 0.0);
            for (int k = rp[r]; k < rp[r + 1]; ++k)
              ev = cadd(ev, cmul(P.se_val[off + k], dense_at(p, P.se_col[off + k], th, h_last)));
            acc = cadd(acc, cmul(cconj(dense_at(p, r, th, h_last)), ev));
          }
        }
      }
      const double sx = block_sum(acc.x, smem);
      const double sy = block_sum(acc.y, smem);
      if (threadIdx.x == 0) {
        const int s = 2 * (q * P.n_e + e);
        slots[static_cast<long long>(s) * G + rank] = sx;
        slots[static_cast<long long>(s + 1) * G + rank] = sy;
      }
    }
  }
  for (int q = 0; q < np; ++q) {  // state saves: every CTA writes its share
    if (c.pend[q].save_idx < 0) continue;
    const double th = c.pend[q].theta;
    double2* out = P.states + static_cast<long long>(c.pend[q].save_idx) * P.n;
    for (int r = gtid; r < P.n; r += gstride) {
      if (MODE == 0) {
        const int i = r % P.d, j = r / P.d;
        const double2 a = dense_at(p, r, th, h_last);          // rho(i,j)
        const double2 b = dense_at(p, i * P.d + j, th, h_last);  // rho(j,i)
        out[r] = cscale(0.5, cadd(a, cconj(b)));
      } else {
        out[r] = dense_at(p, r, th, h_last);
      }
    }
  }
}

// CTA 0 folds the observation slots (written before the last barrier) into expect[].
__device__ __noinline__ void observe_commit(const GridProblem& P, const Ctl& c, const double* slots, int G) {
  if (blockIdx.x != 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nv = 2 * c.np * P.n_e;
  for (int s = warp; s < nv; s += nw) {
    double v = 0.0;
    for (int g = lane; g < G; g += 32) v += slots[static_cast<long long>(s) * G + g];
    v = warp_sum(v);
    if (lane == 0) {
      const int q = (s / 2) / P.n_e, e = (s / 2) % P.n_e;
      if (c.pend[q].grid_idx >= 0) {
        double* dst = reinterpret_cast<double*>(P.expect + static_cast<long long>(c.pend[q].grid_idx) * P.n_e + e);
        dst[s & 1] = v;
      }
    }
  }
}

// every CTA reads slot s (partials of all G CTAs) in the same order -> identical value in *out
__device__ __forceinline__ void grid_value(const double* red, int s, int G, double* out) {
  if ((threadIdx.x >> 5) == 0) {
    const int lane = threadIdx.x & 31;
    double v = 0.0;
    for (int g = lane; g < G; g += 32) v += red[static_cast<long long>(s) * G + g];
    v = warp_sum(v);
    if (lane == 0) *out = v;
  }
}

// Grid-wide barrier of the solve: the monotone-counter grid barrier of a cooperative launch, or,
// when the whole grid is one thread-block cluster (small systems), the hardware cluster barrier
// (release/acquire at cluster scope; the acquire also invalidates L1, so gathers see the other
// CTAs' stores).
__device__ __forceinline__ void sync_all(const GridProblem& P, int G) {
  if (P.cluster) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    grid_barrier(P.bar, G);
  }
}

// sesolve observations <psi|E psi> (evolve.cpp:341-345) with psi(theta) materialised once per
// event in SB (free from the end of stage 2, or of stage 6 for a flush, until stage 3 writes it):
// each e_op entry then gathers one amplitude instead of evaluating the 8-vector dense output, and
// the e_ops share one evaluation. TFIM-20 (3 e_ops of 20 entries per row, 100 events): the
// observations were 41% of the solve. Same values and summation order as observe_pass. Every CTA
// calls it (grid barriers inside); sb_busy: SB is still being gathered (materialised stage-2 input).
__device__ __noinline__ void observe_se(const GridProblem& P, const Ctl& c, double* slots, double* smem, int rank,
                                        int G, bool sb_busy) {
  double2* const* p = c.p;
  const int np = c.np;
  const double h_last = c.h_last;
  const int gtid = rank * blockDim.x + threadIdx.x;
  const int gstride = G * blockDim.x;
  double2* psi = p[SB];
  for (int q = 0; q < np; ++q) {
    if (q > 0 || sb_busy) sync_all(P, G);  // nobody still gathers SB
    const double th = c.pend[q].theta;
    for (int r = gtid; r < P.n; r += gstride) psi[r] = dense_at(p, r, th, h_last);
    sync_all(P, G);
    for (int e = 0; e < P.n_e; ++e) {
      double2 acc = make_double2(0.0, 0.0);
      if (c.pend[q].grid_idx >= 0) {
        if (P.n_se_ops == P.n_e) {
          // the e_op's operator store: a warp's rows are one SELL slice (gtid = lane mod 32)
          const DevSell& E = P.se_ops[e];
          for (int r = gtid; r < P.n; r += gstride) {
            const double2 ev = sell_row(E, r >> 5, r & 31, [&](int col) { return psi[col]; });
            acc = cadd(acc, cmul(cconj(psi[r]), ev));
          }
        } else {
          const int* rp = P.se_rowptr + static_cast<long long>(e) * (P.n + 1);
          const long long off = P.se_off[e];
          for (int r = gtid; r < P.n; r += gstride) {
            double2 ev = make_double2(0.0, 0.0);
            for (int k = rp[r]; k < rp[r + 1]; ++k) ev = cadd(ev, cmul(P.se_val[off + k], psi[P.se_col[off + k]]));
            acc = cadd(acc, cmul(cconj(psi[r]), ev));
          }
        }
      }
      const double sx = block_sum(acc.x, smem);
      const double sy = block_sum(acc.y, smem);
      if (threadIdx.x == 0) {
        const int s = 2 * (q * P.n_e + e);
        slots[static_cast<long long>(s) * G + rank] = sx;
        slots[static_cast<long long>(s + 1) * G + rank] = sy;
      }
    }
    if (c.pend[q].save_idx >= 0) {  // state save: every CTA writes its share
      double2* out = P.states + static_cast<long long>(c.pend[q].save_idx) * P.n;
      for (int r = gtid; r < P.n; r += gstride) out[r] = psi[r];
    }
  }
}

__device__ __forceinline__ void push_pending(const GridProblem& P, Ctl& c, double theta) {
  c.pend[c.np] = Pending{theta, c.ev_grid[c.next], c.ev_save[c.next]};
  ++c.np;
  ++c.next;
}

// One fused stage pass: k_S = G(ts) x over this CTA's slices, then the stage epilogue
// (integrator.hpp:91-102 for S = 2..6; error partial of :106-116 for S = 7).
// PF (every term on the dictionary-coded store): a single-term generator runs the software-
// pipelined loop below (next slice's codes and operands prefetched into L2, dictionary in shared
// memory, operands loaded after the SpMV); multi-term generators load the operands before the
// SpMV so their HBM latency overlaps the gathers. The plain store loads them after the SpMV,
// where holding them would spill.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Key-aligned store stream of one warp (ST == 2). The warp's slices b0, b0+W, ... (cnt of them) are
// re-read in the same order by every stage pass, so their blocks form one endless stream that a
// 2-slot ring in shared memory prefetches through the TMA engine (cp.async.bulk + mbarrier): the
// block of stream position u lands in slot u & 1, on that slot's (u >> 1)-th barrier phase. Two
// blocks are always in flight, across pass and grid-barrier boundaries too (the store is
// read-only); the kernel drains them before it exits. Lane j caches the block bounds of sequence
// index cbase + j, so issuing a copy costs two shuffles, not a dependent global load.
struct KaRing {
  uint4* base;               // slot 0; slot 1 at base + slot_words
  unsigned long long* bar;   // this warp's two mbarriers
  const uint4* blk;          // store blocks (global)
  const unsigned* off;       // block offsets (global, 16-byte units)
  int slot_words, b0, W, cnt, cbase;
  int knext;                 // sequence index of the next block to issue (wraps at cnt)
  unsigned used, issued;     // stream positions (identical in every lane)
  unsigned off_lo, off_hi;   // lane j: bounds of sequence index cbase + j

  __device__ __forceinline__ void refill(int k) {
    cbase = k & ~31;
    const int j = cbase + (threadIdx.x & 31);
    if (j < cnt) {
      const int b = b0 + j * W;
      off_lo = __ldg(off + b);
      off_hi = __ldg(off + b + 1);
    }
  }
  __device__ __forceinline__ void issue() {
    const int k = knext;
    knext = k + 1 == cnt ? 0 : k + 1;
    if (k < cbase || k >= cbase + 32) refill(k);
    const unsigned lo = __shfl_sync(0xffffffffu, off_lo, k - cbase);
    const unsigned hi = __shfl_sync(0xffffffffu, off_hi, k - cbase);
    if ((threadIdx.x & 31) == 0) {
      const unsigned sl = issued & 1u;
      bulk_g2s(base + sl * slot_words, blk + lo, 16u * (hi - lo), bar + sl);
    }
    ++issued;
  }
  __device__ __forceinline__ const uint4* wait() {
    const unsigned sl = used & 1u;
    mbar_wait(bar + sl, (used >> 1) & 1u);
    return base + sl * slot_words;
  }
  // every lane is done reading the current slot: hand it to the async proxy for position used + 2
  __device__ __forceinline__ void release() {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) fence_proxy_async();
    ++used;
    issue();
  }
};

// One slice of the key-aligned store from its staged block (engine.cuh layout). Every shared-memory
// word is read at a warp-uniform address (one wavefront per 32-bit word, two per value): per
// position only its key word (and a partial mask), per value group one value. Positions of a group
// share their value, so the group's gathers are summed first and multiplied once:
//   acc += v_g * (sum_{p in g} x[row ^ key_p]),
// groups in ascending value id, then the non-uniform positions (per-lane value ids) in key order.
#ifndef KA_UNROLL
#define KA_UNROLL 4
#endif
template <class XF>
__device__ __forceinline__ double2 ka_row(const uint4* __restrict__ blk4, const double2* __restrict__ vals, int row,
                                          XF&& xf) {
  const unsigned* __restrict__ w = reinterpret_cast<const unsigned*>(blk4);
  __builtin_assume(__isShared(w));
  __builtin_assume(__isShared(vals));
  const int lane = threadIdx.x & 31;
  const unsigned bit = 1u << lane;
  asm volatile("" : "+r"(row));  // keep row in a register: ptxas otherwise rematerialises it per gather
  const uint4 h = blk4[0];
  const int G = static_cast<int>(h.x), NN = static_cast<int>(h.y), Pu = static_cast<int>(h.z);
  double2 acc = make_double2(0.0, 0.0);
  const unsigned* kw_p = w + kKaHdrWords + G;  // key words, group order
  const unsigned* mk_p = kw_p + Pu;            // partial masks, same order
  for (int g = 0; g < G; ++g) {
    const unsigned gw = w[kKaHdrWords + g];
    const int cnt = static_cast<int>(gw >> 16);
    double2 sum = make_double2(0.0, 0.0);
    for (int c = 0; c < cnt; c += KA_UNROLL) {
      unsigned kw[KA_UNROLL];
#pragma unroll
      for (int u = 0; u < KA_UNROLL; ++u) kw[u] = c + u < cnt ? kw_p[u] : 0x80000000u;  // past the end: empty mask
      double2 x[KA_UNROLL];
      int q = 0;
#pragma unroll
      for (int u = 0; u < KA_UNROLL; ++u) {
        const bool part = static_cast<int>(kw[u]) < 0;
        const unsigned m = part ? (c + u < cnt ? mk_p[q] : 0u) : 0xffffffffu;
        q += (part && c + u < cnt) ? 1 : 0;
        const int col = (row ^ static_cast<int>(kw[u])) & 0x7fffffff;
        x[u] = (m & bit) ? xf(col) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < KA_UNROLL; ++u) sum = cadd(sum, x[u]);
      kw_p += KA_UNROLL;
      mk_p += q;
    }
    kw_p += cnt - ((cnt + KA_UNROLL - 1) / KA_UNROLL) * KA_UNROLL;  // undo the overshoot of the last chunk
    cfma(vals[gw & 0xffffu], sum, acc);
  }
  const unsigned* ep = mk_p;
  for (int e = 0; e < NN; ++e, ep += kKaNonUniWords) {
    const unsigned key = ep[0], msk = ep[1];
    if (msk & bit) {
      const unsigned short vid = reinterpret_cast<const unsigned short*>(ep + 2)[lane];
      cfma(vals[vid], xf(row ^ static_cast<int>(key)), acc);
    }
  }
  return acc;
}

// X2 (stage 2 only): 0 = the SpMV gathers y + h a21 k1 on the fly (two vectors); 1 = that input was
// materialised in SB by x2_pass (one extra streaming pass and barrier); 2 = autonomous single-term
// generator: since k1 = G y exactly (start, FSAL k1 <- k7 = G ysti7, unchanged after a rejection),
// k2 = G(y + h a21 k1) = k1 + (h a21) G k1, so the SpMV gathers k1 alone and the epilogue adds k1 —
// no x2 pass, no extra barrier, one gathered vector.
// ST: 0 generic rows, 1 coded store (software-pipelined), 2 key-aligned store through the ring.
template <int S, int ST, int X2 = 0>
__device__ __forceinline__ double stage_pass(const GridProblem& P, const Ctl& c, int s0, int s1,
                                             const double2* sval = nullptr, const int* soff = nullptr,
                                             KaRing* ring = nullptr) {
  constexpr bool PF = ST >= 1;
  using namespace dp;
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  const double hh = c.hh;
  const double ts = S == 2 ? c.t + c2 * hh : S == 3 ? c.t + c3 * hh : S == 4 ? c.t + c4 * hh
                  : S == 5 ? c.t + c5 * hh : c.t + hh;
  // every buffer pointer is read from the shared control block once per pass and kept in a
  // restrict-qualified global pointer: stores through them cannot alias the control block, so the
  // loop neither re-reads it nor issues generic loads
  auto gptr = [](double2* p) {
    __builtin_assume(__isGlobal(p));
    return p;
  };
  const double2* __restrict__ y = gptr(c.p[Y]);
  const double2* __restrict__ k1 = gptr(c.p[K1]);
  const double2* __restrict__ x = S == 2 ? (X2 == 1 ? gptr(c.p[SB]) : X2 == 2 ? gptr(c.p[K1]) : nullptr)
                                         : gptr((S == 3 || S == 5 || S == 7) ? c.p[SA] : c.p[SB]);
  const double2* __restrict__ pk2 = gptr(c.p[K2]);
  const double2* __restrict__ pk3 = gptr(c.p[K3]);
  const double2* __restrict__ pk4 = gptr(c.p[K4]);
  const double2* __restrict__ pk5 = gptr(c.p[K5]);
  const double2* __restrict__ pk6 = gptr(c.p[K6]);
  double2* __restrict__ kout = gptr(c.p[S == 2 ? K2 : S == 3 ? K3 : S == 4 ? K4 : S == 5 ? K5 : S == 6 ? K6 : K7]);
  double2* __restrict__ xout = gptr(c.p[(S == 3 || S == 5) ? SB : SA]);
  double esq = 0.0;
  const double2 z = make_double2(0.0, 0.0);
  struct Ops {
    double2 yy, q1, q2, q3, q4, q5, q6, y1;
  };
  // streamed once per pass: do not allocate in L1, which then keeps more of the x-gather lines
  auto ldo = [](const double2* p) { return ld_na_c2(p); };
  (void)ring;
  auto load_operands = [&](int row, bool ok, Ops& o) {
    o.yy = ok ? ldo(y + row) : z;
    o.q1 = ok ? ldo(k1 + row) : z;
    o.q2 = (S >= 3 && S <= 5 && ok) ? ldo(pk2 + row) : z;
    o.q3 = (S >= 4 && ok) ? ldo(pk3 + row) : z;
    o.q4 = (S >= 5 && ok) ? ldo(pk4 + row) : z;
    o.q5 = (S >= 6 && ok) ? ldo(pk5 + row) : z;
    o.q6 = (S == 7 && ok) ? ldo(pk6 + row) : z;
    o.y1 = (S == 7 && ok) ? ldo(x + row) : z;
  };
  auto xin = [&](int col) {
    if constexpr (S == 2 && X2 == 0) {
      const double2 a = y[col], q = k1[col];
      return make_double2(a.x + hh * (a21 * q.x), a.y + hh * (a21 * q.y));
    } else {
      return x[col];
    }
  };
  auto epilogue = [&](int row, double2 k, const Ops& o) {
    const double2 yy = o.yy, q1 = o.q1, q2 = o.q2, q3 = o.q3, q4 = o.q4, q5 = o.q5, q6 = o.q6, y1 = o.y1;
    if (S == 2 && X2 == 2) {  // k2 = k1 + (h a21) G k1
      const double ca = hh * a21;
      k = make_double2(q1.x + ca * k.x, q1.y + ca * k.y);
    }
    if (S == 2) {
      kout[row] = k;
      xout[row] = make_double2(yy.x + hh * (a31 * q1.x + a32 * k.x), yy.y + hh * (a31 * q1.y + a32 * k.y));
    } else if (S == 3) {
      kout[row] = k;
      xout[row] = make_double2(yy.x + hh * (a41 * q1.x + a42 * q2.x + a43 * k.x),
                                  yy.y + hh * (a41 * q1.y + a42 * q2.y + a43 * k.y));
    } else if (S == 4) {
      kout[row] = k;
      xout[row] = make_double2(yy.x + hh * (a51 * q1.x + a52 * q2.x + a53 * q3.x + a54 * k.x),
                                  yy.y + hh * (a51 * q1.y + a52 * q2.y + a53 * q3.y + a54 * k.y));
    } else if (S == 5) {
      kout[row] = k;
      xout[row] = make_double2(yy.x + hh * (a61 * q1.x + a62 * q2.x + a63 * q3.x + a64 * q4.x + a65 * k.x),
                                  yy.y + hh * (a61 * q1.y + a62 * q2.y + a63 * q3.y + a64 * q4.y + a65 * k.y));
    } else if (S == 6) {
      kout[row] = k;
      xout[row] = make_double2(yy.x + hh * (a71 * q1.x + a73 * q3.x + a74 * q4.x + a75 * q5.x + a76 * k.x),
                                  yy.y + hh * (a71 * q1.y + a73 * q3.y + a74 * q4.y + a75 * q5.y + a76 * k.y));
    } else {
      kout[row] = k;
      double2 e;
      e.x = hh * (e1 * q1.x + e3 * q3.x + e4 * q4.x + e5 * q5.x + e6 * q6.x + e7 * k.x);
      e.y = hh * (e1 * q1.y + e3 * q3.y + e4 * q4.y + e5 * q5.y + e6 * q6.y + e7 * k.y);
      const double sc = P.atol + P.rtol * fmax(cabs_(yy), cabs_(y1));
      const double qq = cabs_(e) / sc;
      esq += qq * qq;
    }
  };
  if constexpr (ST == 2) {
    // key-aligned store: blocks arrive through the warp's ring; sval is the value table
    KaRing& R = *ring;
    for (int k = 0; k < R.cnt; ++k) {
      const int b = R.b0 + k * R.W;
      const int row = (b << 5) + lane;
      const bool ok = row < n;
      const uint4* blk = R.wait();
      const double2 kk = ka_row(blk, sval, row, xin);
      R.release();
      const int bn = b + R.W;
      if (bn < s1) {
        const int rn = (bn << 5) + lane;
        if (rn < n) {
          prefetch_l2(y + rn);
          prefetch_l2(k1 + rn);
          if (S >= 3 && S <= 5) prefetch_l2(pk2 + rn);
          if (S >= 4) prefetch_l2(pk3 + rn);
          if (S >= 5) prefetch_l2(pk4 + rn);
          if (S >= 6) prefetch_l2(pk5 + rn);
          if (S == 7) {
            prefetch_l2(pk6 + rn);
            prefetch_l2(x + rn);
          }
        }
      }
      Ops o;
      load_operands(row, ok, o);
      if (ok) epilogue(row, kk, o);
    }
    return esq;
  }
  if constexpr (PF) {
    if (P.gen.n_terms == 1) {
      // Software-pipelined coded SpMV: the next slice's row metadata is loaded at the top of the
      // iteration, and its codes and epilogue operands are prefetched into L2 once that metadata
      // is in, so each slice waits on one L2 round trip (the x gathers) instead of three
      // (metadata, HBM codes, gathers).
      const DevSell& A = P.gen.A[0];
      const CodedView cv = coded_view(A);
      const int* __restrict__ rowlen = A.rowlen;
      const long long* __restrict__ code_off = A.code_off;
      auto meta = [&](int b, int& len, long long& base) {
        len = __ldg(rowlen + b * 32 + lane);
        base = __ldg(code_off + b) + 8LL * lane;  // interleaved groups of 8 codes
      };
      // the slice loop instantiated per code width (one copy runs): no per-entry width test
      auto slices = [&](auto cb) {
        constexpr int CB = decltype(cb)::value;
        int b = s0 + warp, len = 0;
        long long base = 0;
        if (b < s1) meta(b, len, base);
        for (; b < s1; b += W) {
          const int bn = b + W;
          int len_n = 0;
          long long base_n = 0;
          if (bn < s1) meta(bn, len_n, base_n);
          const int row = (b << 5) + lane;
          const bool ok = row < n;
          Ops o;
          const double2 k = sval ? sell_row_coded_smem<CB>(cv, sval, soff, row, len, base, xin)
                                 : sell_row_coded_v(cv, row, len, base, xin);
          if (bn < s1) {
            // the next slice's code block (32 rows x width codes, contiguous): one sector run per lane
            const long long cb_n = base_n - 8LL * lane;
            const char* blk = cv.cbytes == 1 ? reinterpret_cast<const char*>(cv.code8 + cb_n)
                                             : reinterpret_cast<const char*>(cv.code16 + cb_n);
            prefetch_l2(blk + lane * 32 * cv.cbytes);  // 1 KB x code bytes window (array padded by 1 K codes)
            const int rn = (bn << 5) + lane;
            if (rn < n) {
              prefetch_l2(y + rn);
              prefetch_l2(k1 + rn);
              if (S >= 3 && S <= 5) prefetch_l2(pk2 + rn);
              if (S >= 4) prefetch_l2(pk3 + rn);
              if (S >= 5) prefetch_l2(pk4 + rn);
              if (S >= 6) prefetch_l2(pk5 + rn);
              if (S == 7) {
                prefetch_l2(pk6 + rn);
                prefetch_l2(x + rn);
              }
            }
          }
          // operands after the SpMV: they were prefetched into L2 one slice ahead, and holding them in
          // registers across the SpMV only spills (measured 30.8 ms vs 33.8 ms per TFIM-10 solve)
          load_operands(row, ok, o);
          if (ok) epilogue(row, k, o);
          len = len_n;
          base = base_n;
        }
      };
      if (cv.cbytes == 1) slices(std::integral_constant<int, 1>{});
      else slices(std::integral_constant<int, 2>{});
      return esq;
    }
  }
  for (int b = s0 + warp; b < s1; b += W) {
    const int row = (b << 5) + lane;
    const bool ok = row < n;
    Ops o;
    if (PF) load_operands(row, ok, o);
    const double2 k = gen_row(P.gen, P.params, b, ts, xin);
    if (!ok) continue;
    if (!PF) load_operands(row, ok, o);
    epilogue(row, k, o);
  }
  return esq;
}

// SB = y + h a21 k1 over this CTA's rows: the stage-2 input, same expression as the on-the-fly
// gather (integrator.hpp:91), so the result is bit-identical
__device__ __noinline__ void x2_pass(const GridProblem& P, const Ctl& c, int s0, int s1) {
  const double2* __restrict__ y = c.p[Y];
  const double2* __restrict__ k1 = c.p[K1];
  double2* __restrict__ sb = c.p[SB];
  const double hh = c.hh;
  const int r0 = s0 * 32, r1 = min(P.n, s1 * 32);
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double2 a = ld_na_c2(y + r), q = ld_na_c2(k1 + r);
    sb[r] = make_double2(a.x + hh * (dp::a21 * q.x), a.y + hh * (dp::a21 * q.y));
  }
}

// start (integrator.hpp:61-69): k1 = G(t0) y and the d0/d1 norms of initial_step (:160-167)
__device__ __noinline__ void start_pass(const GridProblem& P, const Ctl& c, int s0, int s1, double* d0,
                                        double* d1) {
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* y = c.p[Y];
  double a0 = 0.0, a1 = 0.0;
  for (int b = s0 + warp; b < s1; b += W) {
    const int row = (b << 5) + lane;
    const double2 k = gen_row(P.gen, P.params, b, c.t, [&](int col) { return y[col]; });
    if (row < P.n) {
      c.p[K1][row] = k;
      const double2 yy = y[row];
      const double sc = P.atol + P.rtol * cabs_(yy);
      a0 += cnorm(make_double2(yy.x / sc, yy.y / sc));
      a1 += cnorm(make_double2(k.x / sc, k.y / sc));
    }
  }
  *d0 = a0;
  *d1 = a1;
}

// initial_step trial evaluation (integrator.hpp:172-180): d2 partial of G(t0+h0)(y + h0 k1) - k1
__device__ __noinline__ double start_pass2(const GridProblem& P, const Ctl& c, int s0, int s1) {
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* y = c.p[Y];
  const double2* k1 = c.p[K1];
  const double h0 = c.h0;
  double a = 0.0;
  for (int b = s0 + warp; b < s1; b += W) {
    const int row = (b << 5) + lane;
    const double2 k = gen_row(P.gen, P.params, b, c.t + h0, [&](int col) {
      const double2 u = y[col], v = k1[col];
      return make_double2(u.x + h0 * v.x, u.y + h0 * v.y);
    });
    if (row < P.n) {
      const double2 yy = y[row], kk1 = k1[row];
      const double sc = P.atol + P.rtol * cabs_(yy);
      const double2 df = csub(k, kk1);
      a += cnorm(make_double2(df.x / sc, df.y / sc));
    }
  }
  return a;
}

// thread 0: the Dopri5::step prologue for the next attempt (integrator.hpp:80-89) and the
// max_steps guard of the solve loop (evolve.cpp:157-159).
__device__ void begin_attempt(const GridProblem& P, Ctl& c) {
  if (c.attempts == 0 && c.steps >= P.max_steps) {
    c.status = kFailMaxSteps;
    c.fail_t = c.t;
    return;
  }
  c.hh = fmin(c.h, P.tf - c.t);
  c.clamped = c.hh < c.h;
  if (!(c.hh > 0.0)) {
    c.status = kFailPastEnd;
    c.fail_t = c.t;
  } else if (c.hh <= fabs(c.t) * 1e-15 + 1e-300) {
    c.status = kFailUnderflow;
    c.fail_t = c.t;
  } else if (++c.attempts > 1000) {
    c.status = kFailRejected;
    c.fail_t = c.t;
  }
}

// thread 0: accept / reject (integrator.hpp:116-145) and event bookkeeping (evolve.cpp:160-165)
// err of the attempt from the summed squares (integrator.hpp:116-117)
__device__ __forceinline__ double attempt_err(const GridProblem& P, double err_sq) {
  const double err = sqrt(err_sq / static_cast<double>(P.n));
  return isfinite(err) ? err : 10.0;
}

// The controller's two powers pow(err, expo1) and pow(facold, beta) (integrator.hpp:120-121,144),
// evaluated by lanes 0 and 1 of the calling warp at once; every lane gets both.
__device__ __forceinline__ double2 controller_pows(double err, double facold) {
  const int lane = threadIdx.x & 31;
  const double v = pow(lane == 0 ? err : facold, lane == 0 ? dp::expo1 : dp::beta);
  return make_double2(__shfl_sync(0xffffffffu, v, 0), __shfl_sync(0xffffffffu, v, 1));
}

// pw: {pow(err, expo1), pow(facold, beta)} precomputed (controller_pows), or nullptr
__device__ void finish_attempt(const GridProblem& P, Ctl& c, double err_sq, int kcap, const double2* pw = nullptr) {
  using namespace dp;
  const double err = attempt_err(P, err_sq);
  c.rhs_evals += 6;
  ++c.attempts_total;
  if (err <= 1.0) {
    const double fac11 = pw ? pw->x : pow(err, expo1);
    double fac = fac11 / (pw ? pw->y : pow(c.facold, beta));
    fac = fmax(facc2, fmin(facc1, fac / safe));
    const double h_new = c.hh / fac;
    c.facold = fmax(err, 1e-4);
    c.t_old = c.t;
    c.t += c.hh;
    c.h_last = c.hh;
    double2* oy = c.p[Y];  // y_old <- y, y <- ysti7, FSAL k1 <-> k7
    c.p[Y] = c.p[SA];
    c.p[SA] = c.p[YO];
    c.p[YO] = oy;
    double2* k1p = c.p[K1];
    c.p[K1] = c.p[K7];
    c.p[K7] = k1p;
    ++c.steps;
    c.h = c.clamped ? fmax(c.h, h_new) : h_new;
    c.attempts = 0;
    while (c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t && c.np < kcap)
      push_pending(P, c, (fmin(c.ev_t[c.next], c.t) - c.t_old) / c.h_last);
    const bool more = c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t;
    const bool last = c.t >= P.tf - P.eps_t;
    c.flush = more || (last && c.np > 0);
    c.done = last || c.next >= P.n_ev;
  } else {
    ++c.rejected;
    c.h = c.hh / fmin(facc1, (pw ? pw->x : pow(err, expo1)) / safe);
    c.flush = 0;
    c.done = 0;
  }
}

template <int MODE, int ST>
__global__ void __launch_bounds__(kThreads, QSG_GRID_MINB) dp5_grid_kernel(const __grid_constant__ GridProblem P) {
  constexpr bool PF = ST >= 1;
  __shared__ double s_red[kThreads / 32];
  __shared__ double s_val[2];
  __shared__ Ctl c;
  extern __shared__ __align__(16) unsigned char s_dyn[];

  const int G = gridDim.x, rank = blockIdx.x;
  const int nsl = (P.n + 31) >> 5;
  const int spc = (nsl + G - 1) / G;
  const int s0 = rank * spc, s1 = min(nsl, s0 + spc);
  double* red = P.red;
  const int kcap = max(1, min(kMaxPending, kObsSlots / (2 * max(1, P.n_e))));
  auto slots = [&](int par) { return red + static_cast<long long>(kSlotObs0 + par * kObsSlots) * G; };
  // observation flush: pass, barrier, CTA-0 commit (double-buffered slots)
  auto flush_obs = [&]() {
    if (MODE == 1) observe_se(P, c, slots(c.obs_par), s_red, rank, G, false);
    else observe_pass<MODE>(P, c, slots(c.obs_par), s_red, rank, G);
    sync_all(P, G);
    observe_commit(P, c, slots(c.obs_par), G);
    __syncthreads();
    if (threadIdx.x == 0) {
      c.obs_par ^= 1;
      c.np = 0;
    }
    __syncthreads();
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 11; ++i) c.p[i] = P.buf[i];
    c.ev_t = P.ev_t;
    c.ev_grid = P.ev_grid;
    c.ev_save = P.ev_save;
    c.t = c.t_old = P.t0;
    c.h = c.h_last = 0.0;
    c.facold = 1e-4;
    c.steps = c.rejected = c.rhs_evals = c.attempts_total = 0;
    c.status = kRunning;
    c.attempts = c.next = c.np = c.obs_par = c.flush = c.done = 0;
    c.fail_t = 0.0;
    // events at t0 observe y0 directly (evolve.cpp:134-137)
    while (c.next < P.n_ev && c.ev_t[c.next] <= P.t0 + P.eps_t && c.np < kcap)
      push_pending(P, c, __longlong_as_double(0x7ff8000000000000ll));
  }
  __syncthreads();

  // dictionary of a single-term coded generator staged in shared memory (P.smem_dict entries)
  const double2* sval = nullptr;
  const int* soff = nullptr;
  KaRing ring{};
  if constexpr (ST == 2) {
    // value table, then one 2-slot ring and two mbarriers per warp (layout of dict_smem_bytes)
    const DevSell& A = P.gen.A[0];
    double2* vt = reinterpret_cast<double2*>(s_dyn);
    for (int i = threadIdx.x; i < A.ka_nval; i += blockDim.x) vt[i] = A.ka_val[i];
    const int W = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const int sw = A.ka_slot / 16;
    uint4* rings = reinterpret_cast<uint4*>(vt + A.ka_nval);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(rings + 2 * sw * W);
    ring.base = rings + 2 * sw * warp;
    ring.bar = bars + 2 * warp;
    ring.blk = A.ka_blk;
    ring.off = A.ka_off;
    ring.slot_words = sw;
    ring.b0 = s0 + warp;
    ring.W = W;
    ring.cnt = ring.b0 < s1 ? (s1 - ring.b0 + W - 1) / W : 0;
    ring.cbase = -64;
    ring.knext = 0;
    ring.used = ring.issued = 0;
    if ((threadIdx.x & 31) == 0) {
      mbar_init(ring.bar, 1);
      mbar_init(ring.bar + 1, 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (ring.cnt > 0) {
      ring.issue();
      ring.issue();
    }
    sval = vt;
  }
  if (ST == 1 && P.smem_dict > 0) {
    const DevSell& A = P.gen.A[0];
    double2* dv = reinterpret_cast<double2*>(s_dyn);
    int* dof = reinterpret_cast<int*>(dv + P.smem_dict);
    for (int i = threadIdx.x; i < P.smem_dict; i += blockDim.x) {
      dv[i] = A.dict_val[i];
      dof[i] = A.dict_off[i];
    }
    __syncthreads();
    sval = dv;
    soff = dof;
  }

  // ---------------- start + initial_step ----------------
  {
    double d0, d1;
    start_pass(P, c, s0, s1, &d0, &d1);
    d0 = block_sum(d0, s_red);
    d1 = block_sum(d1, s_red);
    if (threadIdx.x == 0) {
      red[static_cast<long long>(kSlotD0) * G + rank] = d0;
      red[static_cast<long long>(kSlotD1) * G + rank] = d1;
    }
    if (c.np) observe_pass<MODE>(P, c, slots(c.obs_par), s_red, rank, G);
    sync_all(P, G);
    if (c.np) observe_commit(P, c, slots(c.obs_par), G);
    grid_value(red, kSlotD0, G, &s_val[0]);
    __syncthreads();
    if (threadIdx.x == 0) s_val[1] = s_val[0];
    __syncthreads();
    grid_value(red, kSlotD1, G, &s_val[0]);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (c.np) {
        c.obs_par ^= 1;
        c.np = 0;
      }
      c.rhs_evals += 1;
      const double dd0 = sqrt(s_val[1] / static_cast<double>(P.n));
      const double dd1 = sqrt(s_val[0] / static_cast<double>(P.n));
      double h0 = (dd0 < 1e-5 || dd1 < 1e-5) ? 1e-6 : 0.01 * dd0 / dd1;  // integrator.hpp:168-170
      h0 = fmin(h0, P.tf - c.t);
      if (!(h0 > 0)) h0 = 1e-6;
      c.h0 = h0;
      c.d1 = dd1;
    }
    __syncthreads();
    double d2 = start_pass2(P, c, s0, s1);
    d2 = block_sum(d2, s_red);
    if (threadIdx.x == 0) red[static_cast<long long>(kSlotD2) * G + rank] = d2;
    sync_all(P, G);
    grid_value(red, kSlotD2, G, &s_val[0]);
    __syncthreads();
    if (threadIdx.x == 0) {
      c.rhs_evals += 1;
      const double dd2 = sqrt(s_val[0] / static_cast<double>(P.n)) / c.h0;  // :180-186
      double h1;
      if (fmax(c.d1, dd2) <= 1e-15) h1 = fmax(1e-6, c.h0 * 1e-3);
      else h1 = pow(0.01 / fmax(c.d1, dd2), 0.2);
      c.h = fmin(fmin(100.0 * c.h0, h1), P.tf - c.t);
    }
    __syncthreads();
  }

  // ---------------- solve loop (evolve.cpp:156-167) ----------------
  for (;;) {
    if (threadIdx.x == 0) {
      if (c.next >= P.n_ev) c.done = 1;
      else begin_attempt(P, c);
    }
    __syncthreads();
    if (c.done || c.status != kRunning) break;
    // stage 2 (+ observations of the previous accepted step)
    if (P.k1g) {
      stage_pass<2, ST, 2>(P, c, s0, s1, sval, soff, &ring);
    } else if (PF && P.x2) {
      x2_pass(P, c, s0, s1);
      sync_all(P, G);
      stage_pass<2, ST, 1>(P, c, s0, s1, sval, soff, &ring);
    } else {
      stage_pass<2, ST == 2 ? 1 : ST>(P, c, s0, s1, sval, soff, &ring);
    }
    if (c.np) {
      if (MODE == 1) observe_se(P, c, slots(c.obs_par), s_red, rank, G, PF && P.x2 && !P.k1g);
      else observe_pass<MODE>(P, c, slots(c.obs_par), s_red, rank, G);
    }
    sync_all(P, G);
    if (c.np) {
      observe_commit(P, c, slots(c.obs_par), G);
      __syncthreads();
      if (threadIdx.x == 0) {
        c.obs_par ^= 1;
        c.np = 0;
      }
    }
    stage_pass<3, ST>(P, c, s0, s1, sval, soff, &ring);
    sync_all(P, G);
    stage_pass<4, ST>(P, c, s0, s1, sval, soff, &ring);
    sync_all(P, G);
    stage_pass<5, ST>(P, c, s0, s1, sval, soff, &ring);
    sync_all(P, G);
    stage_pass<6, ST>(P, c, s0, s1, sval, soff, &ring);
    sync_all(P, G);
    double esq = stage_pass<7, ST>(P, c, s0, s1, sval, soff, &ring);
    esq = block_sum(esq, s_red);
    if (threadIdx.x == 0) red[static_cast<long long>(kSlotErr) * G + rank] = esq;
    sync_all(P, G);
    grid_value(red, kSlotErr, G, &s_val[0]);
    __syncthreads();
    if (threadIdx.x < 32) {
      const double2 pw = controller_pows(attempt_err(P, s_val[0]), c.facold);
      if (threadIdx.x == 0) finish_attempt(P, c, s_val[0], kcap, &pw);
    }
    __syncthreads();
    while (c.flush) {  // pending list full, or the solve ends with events pending
      flush_obs();
      if (threadIdx.x == 0) {
        while (c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t && c.np < kcap)
          push_pending(P, c, (fmin(c.ev_t[c.next], c.t) - c.t_old) / c.h_last);
        const bool more = c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t;
        c.flush = more || (c.t >= P.tf - P.eps_t && c.np > 0);
      }
      __syncthreads();
    }
    if (c.done) break;
  }

  // ---------------- pending and trailing events observe the final state (evolve.cpp:169) ----
  if (c.status == kRunning) {
    if (c.np) flush_obs();
    while (c.next < P.n_ev) {
      if (threadIdx.x == 0)
        while (c.next < P.n_ev && c.np < kcap) push_pending(P, c, __longlong_as_double(0x7ff8000000000000ll));
      __syncthreads();
      flush_obs();
    }
  }
  if constexpr (ST == 2) {  // the two blocks still in flight land before the CTA exits
    if (ring.cnt > 0) {
      ring.wait();
      ++ring.used;
      ring.wait();
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    GridCtl* o = P.ctl;
    o->t = c.t;
    o->h = c.h;
    o->status = c.status == kRunning ? kDone : c.status;
    o->fail_t = c.fail_t;
    o->steps = c.steps;
    o->rejected = c.rejected;
    o->rhs_evals = c.rhs_evals;
    o->attempts = c.attempts_total;
    o->final_buf = 0;
  }
}

// =================================================================================================
// K-cluster: the whole solve resident in the distributed shared memory of ONE thread-block cluster
// (small systems, configs[0]/[3]). CTA r owns rows [r*R, (r+1)*R) (R a multiple of 32): its slices
// of the operator (column pre-split into (owner CTA, local row), values) and its rows of the 11
// state vectors live in its shared memory for the whole solve. The SpMV gathers x[col] from the
// owner's shared memory (ld.shared::cluster), the epilogue touches only local rows, and the passes
// are separated by hardware cluster barriers. Nothing is read from L2 after the prologue, so no
// barrier's L1 invalidation matters. Control, events and the PI controller are the grid engine's
// (Ctl, begin_attempt, finish_attempt), replicated identically in every CTA; reductions are CTA
// partials read by every CTA from every CTA's shared memory in rank order (deterministic).
// 12 warps per CTA: Kerr N = 20/35/50/70/100 9.70/9.26/9.33/9.94/14.54 us per attempt, against
// 9.88/9.35/9.44/10.07/15.44 with 16 warps (256 threads: faster to N = 50, 13.2/17.2 at N = 70/100;
// profiles/r02_cl_kv.log)
#ifndef QSG_CL_THREADS
#define QSG_CL_THREADS 384
#endif
constexpr int kClThreads = QSG_CL_THREADS;
constexpr int kEvSmem = 1024;  // events staged in shared memory when the solve has at most this many

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Cluster barrier. Every value one CTA reads from another lives in shared memory, so the release
// side only has to order this CTA's shared-memory writes: a shared::cta-restricted release fence
// (MEMBAR.CTA + FENCE.VIEW.ASYNC.S) ahead of a relaxed arrive, instead of the MEMBAR.ALL.GPU that
// `arrive.release` emits (-0.8 us per Kerr attempt, profiles/r02_cl_release.log); the wait keeps
// its cluster-scope acquire.
__device__ __forceinline__ void cl_sync() {
  asm volatile(
      "fence.release.sync_restrict::shared::cta.cluster;\n\t"
      "barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_map(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 cl_ld2(unsigned a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double cl_ld(unsigned a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}

// element c (global index) of logical buffer b, from its owner CTA
// owner = c / R by a multiply-high with rmagic = ceil(2^32 / R): exact for c * R < 2^32, which the
// plan guarantees (n <= 16 R, R < 2^14)
__device__ __forceinline__ double2 cl_elem(double2* const* p, int b, int c, int R, unsigned rmagic) {
  const unsigned owner = __umulhi(static_cast<unsigned>(c), rmagic);
  const unsigned loc = static_cast<unsigned>(c - static_cast<int>(owner) * R);
  return cl_ld2(cl_map(smem_u32(p[b] + loc), owner));
}
// dense output (integrator.hpp:127-131,150-154) at global index c, read from its owner CTA
__device__ __forceinline__ double2 cl_dense(double2* const* p, int c, double theta, double h, int R, unsigned rm) {
  if (isnan(theta)) return cl_elem(p, Y, c, R, rm);
  const double2 yo = cl_elem(p, YO, c, R, rm), y1 = cl_elem(p, Y, c, R, rm), k1 = cl_elem(p, K7, c, R, rm),
                k7 = cl_elem(p, K1, c, R, rm), k3 = cl_elem(p, K3, c, R, rm), k4 = cl_elem(p, K4, c, R, rm),
                k5 = cl_elem(p, K5, c, R, rm), k6 = cl_elem(p, K6, c, R, rm);
  using namespace dp;
  const double th1 = 1.0 - theta;
  const double2 rc2 = csub(y1, yo);
  const double2 rc3 = csub(cscale(h, k1), rc2);
  const double2 rc4 = csub(csub(rc2, cscale(h, k7)), rc3);
  double2 rc5;
  rc5.x = h * (d1 * k1.x + d3 * k3.x + d4 * k4.x + d5 * k5.x + d6 * k6.x + d7 * k7.x);
  rc5.y = h * (d1 * k1.y + d3 * k3.y + d4 * k4.y + d5 * k5.y + d6 * k6.y + d7 * k7.y);
  double2 o;
  o.x = yo.x + theta * (rc2.x + th1 * (rc3.x + theta * (rc4.x + th1 * rc5.x)));
  o.y = yo.y + theta * (rc2.y + th1 * (rc3.y + theta * (rc4.y + th1 * rc5.y)));
  return o;
}

// Cluster-wide deterministic sum of one value per CTA: every CTA writes its partial into slot k of
// its own reduction array; after the caller's cluster barrier a whole warp reads slot k of the C
// CTAs (lane r from CTA r, all loads in flight at once) and folds them in a fixed xor tree, the
// same order in every CTA. Returns the total in every lane.
__device__ __forceinline__ double cl_warp_sum(double* red, int k, int C) {
  const int lane = threadIdx.x & 31;
  double v = lane < C ? cl_ld(cl_map(smem_u32(red + k), static_cast<unsigned>(lane))) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One SpMV row of the CTA's resident operator slice sl (lane = row in slice), gathering logical
// buffer xb (S2: y + h a21 k1 on the fly) from every CTA's shared memory.
template <bool S2>
__device__ __forceinline__ double2 cl_row_at(const int* rowlen, const int* soff, const unsigned* tgt,
                                             const double2* val, int sl, int lane, unsigned xa, unsigned ya,
                                             unsigned ka, double hh) {
  const int len = rowlen[sl * 32 + lane];
  const int base = soff[sl] * 32 + lane;
  double2 acc = make_double2(0.0, 0.0);
  constexpr int U = 8;  // one round of DSMEM gathers for rows of up to 8 entries (Kerr: 6)
  for (int j = 0; j < len; j += U) {
    unsigned tg[U];
    double2 v[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      tg[u] = j + u < len ? tgt[base + 32 * (j + u)] : 0u;
      v[u] = j + u < len ? val[base + 32 * (j + u)] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < len) {
        const unsigned own = tg[u] >> 24, off = (tg[u] & 0xffffffu) * 16u;
        if constexpr (S2) {
          const double2 a = cl_ld2(cl_map(ya + off, own)), q = cl_ld2(cl_map(ka + off, own));
          x[u] = make_double2(a.x + hh * (dp::a21 * q.x), a.y + hh * (dp::a21 * q.y));
        } else {
          x[u] = cl_ld2(cl_map(xa + off, own));
        }
      } else {
        x[u] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < len) cfma(v[u], x[u], acc);
  }
  return acc;
}
template <bool S2>
__device__ __forceinline__ double2 cl_row(const int* rowlen, const int* soff, const unsigned* tgt, const double2* val,
                                          int sl, int lane, double2* const* p, int xb, double hh) {
  return cl_row_at<S2>(rowlen, soff, tgt, val, sl, lane, smem_u32(p[xb]), smem_u32(p[Y]), smem_u32(p[K1]), hh);
}

#ifdef QSG_CL_TIMING
__device__ unsigned long long g_cl_ns[16];
__device__ __forceinline__ unsigned long long cl_now() {  // SM clock cycles (globaltimer is too coarse)
  return static_cast<unsigned long long>(clock64());
}
// per-phase globaltimer deltas of CTA 0 thread 0, kept in registers until the kernel ends (a global
// read-modify-write per phase would stall the timed thread and charge the stall to the next phase)
#define CL_T(k)                               \
  do {                                        \
    if (rank == 0 && threadIdx.x == 0) {      \
      const unsigned long long _t = cl_now(); \
      cl_acc[k] += _t - cl_t_last;            \
      cl_t_last = _t;                         \
    }                                         \
  } while (0)
#else
#define CL_T(k) \
  do {          \
  } while (0)
#endif

template <int MODE>
__global__ void __launch_bounds__(kClThreads, 1) dp5_cluster_kernel(const __grid_constant__ GridProblem P,
                                                                      const ClLayout L) {
  __shared__ double s_red[kClThreads / 32];
  __shared__ Ctl c;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int C = gridDim.x;
  const int rank = static_cast<int>(cl_rank());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = kClThreads / 32;
  const int n = P.n, R = L.R;
  const int r0 = rank * R, r1 = min(n, r0 + R);
  const int nsl = (max(0, r1 - r0) + 31) >> 5;  // this CTA's slices
  double2* vec = reinterpret_cast<double2*>(s_dyn + L.vec);
  int* rowlen = reinterpret_cast<int*>(s_dyn + L.rowlen);
  int* soff = reinterpret_cast<int*>(s_dyn + L.soff);
  unsigned* tgt = reinterpret_cast<unsigned*>(s_dyn + L.tgt);
  double2* val = reinterpret_cast<double2*>(s_dyn + L.val);
  double* red = reinterpret_cast<double*>(s_dyn + L.red);  // [0..3] control sums, [4..] observations
  const int kcap = max(1, min(kMaxPending, kObsSlots / (2 * max(1, P.n_e))));
#ifdef QSG_CL_TIMING
  unsigned long long cl_t_last = cl_now(), cl_acc[12] = {};
#endif

  // ---- prologue: the CTA's operator slices into shared memory (columns pre-split by owner) and
  // y0 rows; every other buffer starts uninitialised like the grid engine's
  const DevSell& A = P.gen.A[0];
  for (int i = threadIdx.x; i < L.S * 32; i += kClThreads) {
    const int sl = i >> 5, row = r0 + i;
    rowlen[i] = row < n ? __ldg(A.rowlen + row) : 0;
    if ((i & 31) == 0) soff[sl] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // local slice offsets (in 32-entry columns), the global SELL widths
    int acc = 0;
    for (int sl = 0; sl < L.S; ++sl) {
      soff[sl] = acc;
      const int gs = (r0 >> 5) + sl;
      acc += (r0 + sl * 32 < n) ? static_cast<int>(__ldg(A.slice_off + gs + 1) - __ldg(A.slice_off + gs)) : 0;
    }
    soff[L.S] = acc;
  }
  __syncthreads();
  for (int sl = warp; sl < nsl; sl += W) {
    const int gs = (r0 >> 5) + sl;
    const long long gbase = __ldg(A.slice_off + gs) * 32;
    const int wd = soff[sl + 1] - soff[sl];
    for (int j = 0; j < wd; ++j) {
      const long long gi = gbase + 32LL * j + lane;
      const int col = __ldg(A.col + gi);
      const int own = col / R;
      tgt[(soff[sl] + j) * 32 + lane] = (static_cast<unsigned>(own) << 24) | static_cast<unsigned>(col - own * R);
      val[(soff[sl] + j) * 32 + lane] = __ldg(A.val + gi);
    }
  }
  // events in shared memory (L1 is invalidated by every cluster barrier, so the controller would
  // otherwise fetch them from L2 on each accepted step)
  __shared__ double s_evt[kEvSmem];
  __shared__ int s_evg[kEvSmem], s_evs[kEvSmem];
  const bool ev_sm = P.n_ev <= kEvSmem;
  if (ev_sm)
    for (int i = threadIdx.x; i < P.n_ev; i += kClThreads) {
      s_evt[i] = P.ev_t[i];
      s_evg[i] = P.ev_grid[i];
      s_evs[i] = P.ev_save[i];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 11; ++i) c.p[i] = vec + static_cast<long long>(i) * R;
    c.ev_t = ev_sm ? s_evt : P.ev_t;
    c.ev_grid = ev_sm ? s_evg : P.ev_grid;
    c.ev_save = ev_sm ? s_evs : P.ev_save;
    c.t = c.t_old = P.t0;
    c.h = c.h_last = 0.0;
    c.facold = 1e-4;
    c.steps = c.rejected = c.rhs_evals = c.attempts_total = 0;
    c.status = kRunning;
    c.attempts = c.next = c.np = c.obs_par = c.flush = c.done = 0;
    c.fail_t = 0.0;
    while (c.next < P.n_ev && c.ev_t[c.next] <= P.t0 + P.eps_t && c.np < kcap)
      push_pending(P, c, __longlong_as_double(0x7ff8000000000000ll));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r1 - r0; i += kClThreads) c.p[Y][i] = P.buf[0][r0 + i];  // y0 (host-staged)
  cl_sync();

  // mesolve e_op entries in shared memory when the plan made room (L.n_eo > 0)
  const int* eo_off = P.eo_off;
  const int* eo_i = P.eo_i;
  const int* eo_j = P.eo_j;
  const double2* eo_v = P.eo_v;
  if (MODE == 0 && L.n_eo > 0) {
    int* so = reinterpret_cast<int*>(s_dyn + L.eo);
    double2* sv = reinterpret_cast<double2*>(s_dyn + L.eo + ((4u * (P.n_e + 1) + 15u) & ~15u));
    int* si = reinterpret_cast<int*>(sv + L.n_eo);
    int* sj = si + L.n_eo;
    for (int i = threadIdx.x; i <= P.n_e; i += kClThreads) so[i] = P.eo_off[i];
    for (int i = threadIdx.x; i < L.n_eo; i += kClThreads) {
      sv[i] = P.eo_v[i];
      si[i] = P.eo_i[i];
      sj[i] = P.eo_j[i];
    }
    eo_off = so;
    eo_i = si;
    eo_j = sj;
    eo_v = sv;
    __syncthreads();
  }
  // ---- observation pass: pending events -> expectation partials in red[4 + 2*(q*n_e+e)] and saves
  // bank of observation slots in red[] (double-buffered by c.obs_par, like the grid engine's):
  // a bank is rewritten two observation events later, after at least one more cluster barrier
  auto obs_bank = [&](int par) { return red + 4 + par * kObsSlots; };
  // ow: one warp (the caller, lane = item index) does the whole observation with no block barrier,
  // so it can run beside the other warps' stage-2 pass (MODE 0 only)
  auto observe = [&](bool ow = false) {
    const int tid = ow ? lane : static_cast<int>(threadIdx.x), nthr = ow ? 32 : kClThreads;
    double2* const* p = c.p;
    const int np = c.np;
    const double hl = c.h_last;
    double* bank = obs_bank(c.obs_par);
    const int npairs = np * P.n_e;
    // (event, e_op) pairs reduced together: 2, because every extra pair's unrolled reduction grows
    // the per-event code, and that code plus the per-attempt loop must fit the SM's instruction
    // cache (kV 8 -> 2: Kerr-20 10.8 -> 9.9 us per attempt, profiles/r02_cl_kv.log)
    constexpr int kV = 2;
    for (int b0 = 0; b0 < npairs; b0 += kV) {
      const int nv = min(kV, npairs - b0);
      double2 acc[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) acc[v] = make_double2(0.0, 0.0);
      int tl;  // this CTA's work items (threads with work: the first tl)
      if (MODE == 0) {
        // the pairs' e_op entries as one flat list, item i on CTA i % C: every CTA's DSMEM port
        // carries a share of the dense-output gathers and every pair is in flight at once
        int pre[kV + 1], eb[kV];
        double thv[kV];
        pre[0] = 0;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const int pr = b0 + v;
          int cnt = 0;
          eb[v] = 0;
          thv[v] = 0.0;
          if (v < nv) {
            const int q = pr / P.n_e, e = pr % P.n_e;
            if (c.pend[q].grid_idx >= 0) {
              eb[v] = eo_off[e];
              cnt = eo_off[e + 1] - eo_off[e];
              thv[v] = c.pend[q].theta;
            }
          }
          pre[v + 1] = pre[v] + cnt;
        }
        tl = (pre[kV] - rank + C - 1) / C;
        for (int il = tid; il < tl; il += nthr) {
          const int i = il * C + rank;
          int k = 0;
          double th = 0.0;
#pragma unroll
          for (int v = 0; v < kV; ++v)
            if (i >= pre[v] && i < pre[v + 1]) {
              k = eb[v] + (i - pre[v]);
              th = thv[v];
            }
          const int ei = eo_i[k], ej = eo_j[k];
          const double2 x = cmul(eo_v[k], cscale(0.5, cadd(cl_dense(p, ei * P.d + ej, th, hl, R, L.rmagic),
                                                             cconj(cl_dense(p, ej * P.d + ei, th, hl, R, L.rmagic)))));
#pragma unroll
          for (int v = 0; v < kV; ++v)
            if (i >= pre[v] && i < pre[v + 1]) acc[v] = cadd(acc[v], x);
        }
      } else {
        tl = r1 - r0;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          if (v >= nv) break;
          const int pr = b0 + v;
          const int q = pr / P.n_e, e = pr % P.n_e;
          const double th = c.pend[q].theta;
          if (c.pend[q].grid_idx < 0) continue;
          if (P.n_se_ops == P.n_e) {  // e_op operator stores (r0 and the strides are multiples of 32)
            for (int r = r0 + tid; r < r1; r += nthr) {
              const double2 ev = sell_row(P.se_ops[e], r >> 5, r & 31,
                                          [&](int col) { return cl_dense(p, col, th, hl, R, L.rmagic); });
              acc[v] = cadd(acc[v], cmul(cconj(cl_dense(p, r, th, hl, R, L.rmagic)), ev));
            }
          } else {
            const int* rp = P.se_rowptr + static_cast<long long>(e) * (P.n + 1);
            const long long off = P.se_off[e];
            for (int r = r0 + tid; r < r1; r += nthr) {
              double2 ev = make_double2(0.0, 0.0);
              for (int k = rp[r]; k < rp[r + 1]; ++k)
                ev = cadd(ev, cmul(P.se_val[off + k], cl_dense(p, P.se_col[off + k], th, hl, R, L.rmagic)));
              acc[v] = cadd(acc[v], cmul(cconj(cl_dense(p, r, th, hl, R, L.rmagic)), ev));
            }
          }
        }
      }
      CL_T(7);
      // the CTA's partial of each of the 2 nv values, in a fixed order: warp shuffles, then (more
      // than one warp with work) one smem row per warp folded by warp 0
      const int aw = min(W, (tl + 31) >> 5);  // warps with work (uniform in the CTA)
      if (ow || aw <= 1) {
        if (ow || warp == 0)
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            if (v >= nv) break;
            const double x = warp_sum(acc[v].x), y = warp_sum(acc[v].y);
            if (lane == 0) {
              bank[2 * (b0 + v)] = x;
              bank[2 * (b0 + v) + 1] = y;
            }
          }
      } else {
        __shared__ double s_obs[kClThreads / 32][2 * kV];
        if (warp < aw)
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            if (v >= nv) break;
            const double x = warp_sum(acc[v].x), y = warp_sum(acc[v].y);
            if (lane == 0) {
              s_obs[warp][2 * v] = x;
              s_obs[warp][2 * v + 1] = y;
            }
          }
        __syncthreads();
        if (warp == 0 && lane < 2 * nv) {
          double t = 0.0;
          for (int w = 0; w < aw; ++w) t += s_obs[w][lane];
          bank[2 * b0 + lane] = t;
        }
        __syncthreads();
      }
      CL_T(8);
    }
    for (int q = 0; q < np; ++q) {
      if (c.pend[q].save_idx < 0) continue;
      const double th = c.pend[q].theta;
      double2* out = P.states + static_cast<long long>(c.pend[q].save_idx) * P.n;
      for (int r = r0 + tid; r < r1; r += nthr) {
        if (MODE == 0) {
          const int i = r % P.d, j = r / P.d;
          out[r] = cscale(0.5, cadd(cl_dense(p, r, th, hl, R, L.rmagic), cconj(cl_dense(p, i * P.d + j, th, hl, R, L.rmagic))));
        } else {
          out[r] = cl_dense(p, r, th, hl, R, L.rmagic);
        }
      }
    }
  };
  // after the barrier that follows observe(), in CTA 0: warps w0, w0 + ws, ... fold the C CTA
  // partials of one value each (lane r reads CTA r) and write expect[]. np / par: the observation's
  // pending count and bank parity (captured, since thread 0 may already be resetting them).
  auto observe_commit_cl = [&](int np, int par, int w0, int ws) {
    const int nv = 2 * np * P.n_e;
    const int base = static_cast<int>(obs_bank(par) - red);
    for (int s2 = w0; s2 < nv; s2 += ws) {
      const double v = cl_warp_sum(red, base + s2, C);
      const int q = (s2 / 2) / P.n_e, e = (s2 / 2) % P.n_e;
      if (lane == 0 && c.pend[q].grid_idx >= 0)
        reinterpret_cast<double*>(P.expect + static_cast<long long>(c.pend[q].grid_idx) * P.n_e + e)[s2 & 1] = v;
    }
  };
  // the stage-2 observation's commit: by CTA 0's last warp while the other warps run stage 3 when
  // that warp owns no slice, else by all of CTA 0's warps before stage 3
  const bool defer_commit = nsl <= W - 1;
  const bool obs_ow = MODE == 0 && nsl <= W - 1 && L.obs_ow;
  auto flush = [&]() {
    observe();
    cl_sync();
    if (rank == 0) observe_commit_cl(c.np, c.obs_par, warp, W);
    __syncthreads();
    if (threadIdx.x == 0) {
      c.np = 0;
      c.obs_par ^= 1;
    }
    __syncthreads();
  };

  // ---- start + initial_step (integrator.hpp:61-69,157-187)
  {
    double a0 = 0.0, a1 = 0.0;
    for (int sl = warp; sl < nsl; sl += W) {
      const int lr = sl * 32 + lane;
      const double2 k = cl_row<false>(rowlen, soff, tgt, val, sl, lane, c.p, Y, 0.0);
      if (r0 + lr < r1) {
        c.p[K1][lr] = k;
        const double2 yy = c.p[Y][lr];
        const double sc = P.atol + P.rtol * cabs_(yy);
        a0 += cnorm(make_double2(yy.x / sc, yy.y / sc));
        a1 += cnorm(make_double2(k.x / sc, k.y / sc));
      }
    }
    a0 = block_sum(a0, s_red);
    a1 = block_sum(a1, s_red);
    if (threadIdx.x == 0) {
      red[0] = a0;
      red[1] = a1;
    }
    if (c.np) observe();
    cl_sync();
    if (c.np && rank == 0) observe_commit_cl(c.np, c.obs_par, warp, W);
    __shared__ double s_tot[3];
    if (warp == 0) {
      const double t0 = cl_warp_sum(red, 0, C), t1 = cl_warp_sum(red, 1, C);
      if (lane == 0) {
        s_tot[0] = t0;
        s_tot[1] = t1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double dd0 = sqrt(s_tot[0] / static_cast<double>(n));
      const double dd1 = sqrt(s_tot[1] / static_cast<double>(n));
      if (c.np) c.obs_par ^= 1;
      c.np = 0;
      c.rhs_evals += 1;
      double h0 = (dd0 < 1e-5 || dd1 < 1e-5) ? 1e-6 : 0.01 * dd0 / dd1;
      h0 = fmin(h0, P.tf - c.t);
      if (!(h0 > 0)) h0 = 1e-6;
      c.h0 = h0;
      c.d1 = dd1;
    }
    cl_sync();  // red[0..1] and the observation slots are read before anyone rewrites them
    double a2 = 0.0;
    {
      const double h0 = c.h0;
      for (int sl = warp; sl < nsl; sl += W) {  // SB = y + h0 k1, then G(t0 + h0) SB
        const int lr = sl * 32 + lane;
        if (r0 + lr < r1) {
          const double2 u = c.p[Y][lr], v = c.p[K1][lr];
          c.p[SB][lr] = make_double2(u.x + h0 * v.x, u.y + h0 * v.y);
        }
      }
      cl_sync();
      for (int sl = warp; sl < nsl; sl += W) {
        const int lr = sl * 32 + lane;
        const double2 k = cl_row<false>(rowlen, soff, tgt, val, sl, lane, c.p, SB, 0.0);
        if (r0 + lr < r1) {
          const double2 yy = c.p[Y][lr], kk1 = c.p[K1][lr];
          const double sc = P.atol + P.rtol * cabs_(yy);
          const double2 df = csub(k, kk1);
          a2 += cnorm(make_double2(df.x / sc, df.y / sc));
        }
      }
    }
    a2 = block_sum(a2, s_red);
    if (threadIdx.x == 0) red[2] = a2;
    cl_sync();
    if (warp == 0) {
      const double t2 = cl_warp_sum(red, 2, C);
      if (lane == 0) s_tot[2] = t2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c.rhs_evals += 1;
      const double dd2 = sqrt(s_tot[2] / static_cast<double>(n)) / c.h0;
      double h1;
      if (fmax(c.d1, dd2) <= 1e-15) h1 = fmax(1e-6, c.h0 * 1e-3);
      else h1 = pow(0.01 / fmax(c.d1, dd2), 0.2);
      c.h = fmin(fmin(100.0 * c.h0, h1), P.tf - c.t);
    }
    __syncthreads();
  }

  // ---- solve loop (evolve.cpp:156-167)
  using namespace dp;
#ifdef QSG_CL_TIMING
  if (rank == 0 && threadIdx.x == 0) cl_t_last = cl_now();
#endif
  for (;;) {
    if (threadIdx.x == 0) {
      if (c.next >= P.n_ev) c.done = 1;
      else begin_attempt(P, c);
    }
    __syncthreads();
    CL_T(0);
    if (c.done || c.status != kRunning) break;
    const double hh = c.hh, t = c.t;
    const int np_s = c.np, par_s = c.obs_par;  // the previous step's pending observations
    (void)t;
    // stage passes 2..7 (integrator.hpp:91-102) on local rows, gathers from the cluster
    for (int S = 2; S <= 7; ++S) {
      const int xb = S == 2 ? Y : (S == 3 || S == 5 || S == 7) ? SA : SB;
      const int ko = S == 2 ? K2 : S == 3 ? K3 : S == 4 ? K4 : S == 5 ? K5 : S == 6 ? K6 : K7;
      const int xo = (S == 3 || S == 5) ? SB : SA;
      double esq = 0.0;
      double2* const* p = c.p;
      for (int sl = warp; sl < nsl; sl += W) {
        const int lr = sl * 32 + lane;
        // stage 2 of an autonomous single-term generator: k2 = k1 + (h a21) G k1 (k1 = G y exactly),
        // one gathered vector instead of y and k1 (the grid engine's X2 = 2 form)
        double2 k = S == 2 ? (P.k1g ? cl_row<false>(rowlen, soff, tgt, val, sl, lane, p, K1, hh)
                                    : cl_row<true>(rowlen, soff, tgt, val, sl, lane, p, Y, hh))
                           : cl_row<false>(rowlen, soff, tgt, val, sl, lane, p, xb, hh);
        if (r0 + lr >= r1) continue;
        const double2 yy = p[Y][lr], q1 = p[K1][lr];
        if (S == 2 && P.k1g) k = make_double2(q1.x + (hh * a21) * k.x, q1.y + (hh * a21) * k.y);
        p[ko][lr] = k;
        if (S == 2) {
          p[xo][lr] = make_double2(yy.x + hh * (a31 * q1.x + a32 * k.x), yy.y + hh * (a31 * q1.y + a32 * k.y));
        } else if (S == 3) {
          const double2 q2 = p[K2][lr];
          p[xo][lr] = make_double2(yy.x + hh * (a41 * q1.x + a42 * q2.x + a43 * k.x),
                                   yy.y + hh * (a41 * q1.y + a42 * q2.y + a43 * k.y));
        } else if (S == 4) {
          const double2 q2 = p[K2][lr], q3 = p[K3][lr];
          p[xo][lr] = make_double2(yy.x + hh * (a51 * q1.x + a52 * q2.x + a53 * q3.x + a54 * k.x),
                                   yy.y + hh * (a51 * q1.y + a52 * q2.y + a53 * q3.y + a54 * k.y));
        } else if (S == 5) {
          const double2 q2 = p[K2][lr], q3 = p[K3][lr], q4 = p[K4][lr];
          p[xo][lr] = make_double2(yy.x + hh * (a61 * q1.x + a62 * q2.x + a63 * q3.x + a64 * q4.x + a65 * k.x),
                                   yy.y + hh * (a61 * q1.y + a62 * q2.y + a63 * q3.y + a64 * q4.y + a65 * k.y));
        } else if (S == 6) {
          const double2 q3 = p[K3][lr], q4 = p[K4][lr], q5 = p[K5][lr];
          p[xo][lr] = make_double2(yy.x + hh * (a71 * q1.x + a73 * q3.x + a74 * q4.x + a75 * q5.x + a76 * k.x),
                                   yy.y + hh * (a71 * q1.y + a73 * q3.y + a74 * q4.y + a75 * q5.y + a76 * k.y));
        } else {
          const double2 q3 = p[K3][lr], q4 = p[K4][lr], q5 = p[K5][lr], q6 = p[K6][lr], y1 = p[SA][lr];
          double2 e;
          e.x = hh * (e1 * q1.x + e3 * q3.x + e4 * q4.x + e5 * q5.x + e6 * q6.x + e7 * k.x);
          e.y = hh * (e1 * q1.y + e3 * q3.y + e4 * q4.y + e5 * q5.y + e6 * q6.y + e7 * k.y);
          const double sc = P.atol + P.rtol * fmax(cabs_(yy), cabs_(y1));
          const double qq = cabs_(e) / sc;
          esq += qq * qq;
        }
      }
      CL_T(1);
      // the previous step's events, on the buffers of that step: by the last warp beside the pass
      // when it owns no slice (mesolve), else by the whole CTA after it
      if (S == 2 && np_s) {
        if (!obs_ow) observe();
        else if (warp == W - 1) observe(true);
      }
      CL_T(2);
      if (S == 7) {
        esq = block_sum(esq, s_red);
        if (threadIdx.x == 0) red[3] = esq;
      }
      cl_sync();
      CL_T(3);
      if (S == 2 && np_s) {
        if (rank == 0) {
          if (!defer_commit) {
            observe_commit_cl(np_s, par_s, warp, W);
            __syncthreads();
          } else if (warp == W - 1) {
            observe_commit_cl(np_s, par_s, 0, 1);
          }
        }
        if (threadIdx.x == 0) {  // c.np is next read after the controller's block barrier
          c.np = 0;
          c.obs_par ^= 1;
        }
      }
      CL_T(4);
    }
    if (warp == 0) {
      const double e2 = cl_warp_sum(red, 3, C);
      const double2 pw = controller_pows(attempt_err(P, e2), c.facold);
      if (lane == 0) finish_attempt(P, c, e2, kcap, &pw);
    }
    __syncthreads();
    CL_T(5);
    while (c.flush) {
      flush();
      if (threadIdx.x == 0) {
        while (c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t && c.np < kcap)
          push_pending(P, c, (fmin(c.ev_t[c.next], c.t) - c.t_old) / c.h_last);
        const bool more = c.next < P.n_ev && c.ev_t[c.next] <= c.t + P.eps_t;
        c.flush = more || (c.t >= P.tf - P.eps_t && c.np > 0);
      }
      __syncthreads();
    }
    CL_T(6);
    // red[3] is read by every CTA (finish_attempt above) before the next stage 7 rewrites it:
    // the six stage barriers in between order that
    if (c.done) break;
  }
#ifdef QSG_CL_TIMING
  if (rank == 0 && threadIdx.x == 0)
    for (int k = 0; k < 12; ++k) g_cl_ns[k] += cl_acc[k];
#endif
  if (c.status == kRunning) {
    if (c.np) flush();
    while (c.next < P.n_ev) {
      if (threadIdx.x == 0)
        while (c.next < P.n_ev && c.np < kcap) push_pending(P, c, __longlong_as_double(0x7ff8000000000000ll));
      __syncthreads();
      flush();
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    GridCtl* o = P.ctl;
    o->t = c.t;
    o->h = c.h;
    o->status = c.status == kRunning ? kDone : c.status;
    o->fail_t = c.fail_t;
    o->steps = c.steps;
    o->rejected = c.rejected;
    o->rhs_evals = c.rhs_evals;
    o->attempts = c.attempts_total;
    o->final_buf = 0;
  }
  cl_sync();  // no CTA leaves while another may still read its shared memory
}

template <int MODE>
cudaError_t launch_cluster_one(const GridProblem& P, const ClLayout& L, int C, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(dp5_cluster_kernel<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) ||
      (e = cudaFuncSetAttribute(dp5_cluster_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(L.bytes))))
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dp5_cluster_kernel<MODE>, P, L);
}

template <int MODE, int ST>
cudaLaunchConfig_t cluster_cfg(int grid, size_t smem, cudaLaunchAttribute* at) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(dp5_grid_kernel<MODE, ST>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = grid;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

template <int MODE, int ST>
cudaError_t launch_one(const GridProblem& P, int grid, cudaStream_t s) {
  if (P.cluster) {  // the whole grid as one cluster: co-scheduled by construction
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_cfg<MODE, ST>(grid, grid_smem_bytes(P, ST), at);
    cfg.stream = s;
    return cudaLaunchKernelEx(&cfg, dp5_grid_kernel<MODE, ST>, P);
  }
  void* args[] = {const_cast<GridProblem*>(&P)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dp5_grid_kernel<MODE, ST>), dim3(grid),
                                     dim3(kThreads), args, grid_smem_bytes(P, ST), s);
}

template <int MODE, int ST>
int max_cluster_one(size_t smem) {
  for (int c = 16; c >= 2; c /= 2) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_cfg<MODE, ST>(c, smem, at);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, dp5_grid_kernel<MODE, ST>, &cfg) == cudaSuccess && nc > 0) return c;
    cudaGetLastError();
  }
  return 0;
}

template <int MODE, int ST>
int occupancy_one(size_t smem) {
  int nb = 0;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(dp5_grid_kernel<MODE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp5_grid_kernel<MODE, ST>, kThreads, smem);
  return nb;
}

}  // namespace

int grid_threads() { return kThreads; }

size_t grid_smem_bytes(const GridProblem& P, int st) {
  if (st == 2) {
    const DevSell& A = P.gen.A[0];
    const int W = kThreads / 32;
    return static_cast<size_t>(A.ka_nval) * sizeof(double2) + static_cast<size_t>(2 * W) * A.ka_slot +
           static_cast<size_t>(2 * W) * sizeof(unsigned long long);
  }
  return static_cast<size_t>(P.smem_dict) * (sizeof(double2) + sizeof(int));
}

int grid_max_blocks_per_sm(int mode, int st, size_t dyn_smem) {
  if (mode == 0)
    return st == 2 ? occupancy_one<0, 2>(dyn_smem) : st == 1 ? occupancy_one<0, 1>(dyn_smem) : occupancy_one<0, 0>(dyn_smem);
  return st == 2 ? occupancy_one<1, 2>(dyn_smem) : st == 1 ? occupancy_one<1, 1>(dyn_smem) : occupancy_one<1, 0>(dyn_smem);
}

int grid_max_cluster(int mode, int st, size_t dyn_smem) {
  if (mode == 0)
    return st == 2 ? max_cluster_one<0, 2>(dyn_smem) : st == 1 ? max_cluster_one<0, 1>(dyn_smem) : max_cluster_one<0, 0>(dyn_smem);
  return st == 2 ? max_cluster_one<1, 2>(dyn_smem) : st == 1 ? max_cluster_one<1, 1>(dyn_smem) : max_cluster_one<1, 0>(dyn_smem);
}

// Plans the cluster-resident layout for a single-term plain-store generator: C CTAs of R rows
// each (R a multiple of 32), all state and operator slices in shared memory. Returns false when
// the system does not fit one 16-CTA cluster.
bool plan_cluster_solve(const GridProblem& P, const long long* slice_off_host, int n_obs_slots, int n_eo, int* C_out,
                        ClLayout* plan) {
  if (P.gen.n_terms != 1 || P.gen.A[0].code_bytes != 0) return false;
  const int n = P.n;
  const long long nsl = (n + 31) / 32;
  // as many CTAs as there are slices, up to 16 (one cluster): each CTA's rows are a pass's
  // latency-bound share of work, so the widest cluster is the fastest (profiles/r02_cluster_solve.log)
  const int C0 = static_cast<int>(std::min<long long>(16, nsl));
  for (int C = C0; C >= 2; C = C == C0 ? C0 : C) {
    const int S = static_cast<int>((nsl + C - 1) / C);
    const int R = 32 * S;
    long long E = 0;  // entry capacity: widest CTA
    for (int r = 0; r < C; ++r) {
      const long long a = std::min<long long>(nsl, static_cast<long long>(r) * S), b = std::min<long long>(nsl, a + S);
      E = std::max(E, 32 * (slice_off_host[b] - slice_off_host[a]));
    }
    auto al = [](unsigned x) { return (x + 15u) & ~15u; };
    ClLayout L{};
    L.R = R;
    L.S = S;
    L.E = static_cast<int>(E);
    L.obs_ow = 1;
    if (const char* ow = std::getenv("QSG_CL_OBS_WARP")) L.obs_ow = ow[0] != '0';
    if (R >= (1 << 14)) break;  // cl_elem's multiply-high division needs R < 2^14 (n <= 16 R)
    L.rmagic = static_cast<unsigned>(((1ull << 32) + R - 1) / R);
    unsigned o = 0;
    L.vec = o;
    o = al(o + 11u * R * 16u);
    L.rowlen = o;
    o = al(o + 4u * 32u * S);
    L.soff = o;
    o = al(o + 4u * (S + 1));
    L.tgt = o;
    o = al(o + 4u * static_cast<unsigned>(E));
    L.val = o;
    o = al(o + 16u * static_cast<unsigned>(E));
    L.red = o;
    o = al(o + 8u * (4 + 2 * n_obs_slots));  // control sums + two observation banks
    L.bytes = o;
    const unsigned static_smem = sizeof(double) * (kClThreads / 32) + sizeof(Ctl) + kEvSmem * 16u +
                                 (kClThreads / 32) * 16 * 8 + 64;
    // mesolve e_op entries {value, row, column} in shared memory when they still fit: the
    // observation pass then reads no L2 (each cluster barrier invalidates L1)
    L.eo = o;
    L.n_eo = 0;
    const unsigned eo_bytes = al(4u * (P.n_e + 1)) + al(24u * static_cast<unsigned>(n_eo));
    if (n_eo > 0 && L.bytes + eo_bytes + static_smem <= 226u * 1024u) {
      L.n_eo = n_eo;
      L.bytes = o + eo_bytes;
    }
    // the smallest cluster whose per-CTA share fits (more CTAs only add DSMEM hops and barrier
    // arrivals); 16 slices per CTA at most so every warp owns at most one slice per pass
    if (L.bytes + static_smem <= 226u * 1024u && S <= 64 && R < (1 << 24)) {  // 227 KB per CTA at most
      *C_out = C;
      *plan = L;
      return true;
    }
    break;  // fewer CTAs only means more rows per CTA: it will not fit either
  }
  return false;
}

cudaError_t launch_cluster_dp5(const GridProblem& P, int mode, const ClLayout& L, int C, cudaStream_t s) {
  return mode == 0 ? launch_cluster_one<0>(P, L, C, s) : launch_cluster_one<1>(P, L, C, s);
}

cudaError_t launch_grid_dp5(const GridProblem& P, int mode, int st, int grid, cudaStream_t s) {
  if (mode == 0)
    return st == 2 ? launch_one<0, 2>(P, grid, s) : st == 1 ? launch_one<0, 1>(P, grid, s) : launch_one<0, 0>(P, grid, s);
  return st == 2 ? launch_one<1, 2>(P, grid, s) : st == 1 ? launch_one<1, 1>(P, grid, s) : launch_one<1, 0>(P, grid, s);
}

}  // namespace qsg

#ifdef QSG_CL_TIMING
extern "C" void qsg_debug_cluster_ns(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, qsg::g_cl_ns, sizeof(unsigned long long) * 16);
  if (reset) {
    static const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(qsg::g_cl_ns, z, sizeof(z));
  }
}
#endif

#ifdef QSG_BAR_TIMING
extern "C" void qsg_debug_barrier_ns(unsigned long long* wait_ns, unsigned long long* calls, int reset,
                                     unsigned long long* per_cta) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(wait_ns, qsg::g_bar_wait_ns, sizeof(unsigned long long));
  cudaMemcpyFromSymbol(calls, qsg::g_bar_calls, sizeof(unsigned long long));
  if (per_cta) cudaMemcpyFromSymbol(per_cta, qsg::g_bar_cta_ns, sizeof(unsigned long long) * 1024);
  if (reset) {
    static const unsigned long long z[1024] = {};
    cudaMemcpyToSymbol(qsg::g_bar_wait_ns, z, sizeof(unsigned long long));
    cudaMemcpyToSymbol(qsg::g_bar_calls, z, sizeof(unsigned long long));
    cudaMemcpyToSymbol(qsg::g_bar_cta_ns, z, sizeof(z));
  }
}
#endif
