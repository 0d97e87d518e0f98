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
#include <cstdio>

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

__device__ __forceinline__ void push_pending(const GridProblem& P, Ctl& c, double theta) {
  c.pend[c.np] = Pending{theta, P.ev_grid[c.next], P.ev_save[c.next]};
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

// X2 (stage 2 only): the stage input y + h a21 k1 was materialised in SB by x2_pass, so the SpMV
// gathers one vector instead of two.
// ST: 0 generic rows, 1 coded store (software-pipelined), 2 key-aligned store through the ring.
template <int S, int ST, bool X2 = false>
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
  const double2* __restrict__ x = S == 2 ? (X2 ? gptr(c.p[SB]) : nullptr)
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
    if constexpr (S == 2 && !X2) {
      const double2 a = y[col], q = k1[col];
      return make_double2(a.x + hh * (a21 * q.x), a.y + hh * (a21 * q.y));
    } else {
      return x[col];
    }
  };
  auto epilogue = [&](int row, double2 k, const Ops& o) {
    const double2 yy = o.yy, q1 = o.q1, q2 = o.q2, q3 = o.q3, q4 = o.q4, q5 = o.q5, q6 = o.q6, y1 = o.y1;
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
        const double2 k = sval ? sell_row_coded_smem(cv, sval, soff, row, len, base, xin)
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
__device__ void finish_attempt(const GridProblem& P, Ctl& c, double err_sq, int kcap) {
  using namespace dp;
  double err = sqrt(err_sq / static_cast<double>(P.n));
  if (!isfinite(err)) err = 10.0;
  c.rhs_evals += 6;
  ++c.attempts_total;
  if (err <= 1.0) {
    const double fac11 = pow(err, expo1);
    double fac = fac11 / pow(c.facold, beta);
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
    while (c.next < P.n_ev && P.ev_t[c.next] <= c.t + P.eps_t && c.np < kcap)
      push_pending(P, c, (fmin(P.ev_t[c.next], c.t) - c.t_old) / c.h_last);
    const bool more = c.next < P.n_ev && P.ev_t[c.next] <= c.t + P.eps_t;
    const bool last = c.t >= P.tf - P.eps_t;
    c.flush = more || (last && c.np > 0);
    c.done = last || c.next >= P.n_ev;
  } else {
    ++c.rejected;
    c.h = c.hh / fmin(facc1, pow(err, expo1) / safe);
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
    observe_pass<MODE>(P, c, slots(c.obs_par), s_red, rank, G);
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
    c.t = c.t_old = P.t0;
    c.h = c.h_last = 0.0;
    c.facold = 1e-4;
    c.steps = c.rejected = c.rhs_evals = c.attempts_total = 0;
    c.status = kRunning;
    c.attempts = c.next = c.np = c.obs_par = c.flush = c.done = 0;
    c.fail_t = 0.0;
    // events at t0 observe y0 directly (evolve.cpp:134-137)
    while (c.next < P.n_ev && P.ev_t[c.next] <= P.t0 + P.eps_t && c.np < kcap)
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
    if (PF && P.x2) {
      x2_pass(P, c, s0, s1);
      sync_all(P, G);
      stage_pass<2, ST, true>(P, c, s0, s1, sval, soff, &ring);
    } else {
      stage_pass<2, ST == 2 ? 1 : ST>(P, c, s0, s1, sval, soff, &ring);
    }
    if (c.np) observe_pass<MODE>(P, c, slots(c.obs_par), s_red, rank, G);
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
    if (threadIdx.x == 0) finish_attempt(P, c, s_val[0], kcap);
    __syncthreads();
    while (c.flush) {  // pending list full, or the solve ends with events pending
      flush_obs();
      if (threadIdx.x == 0) {
        while (c.next < P.n_ev && P.ev_t[c.next] <= c.t + P.eps_t && c.np < kcap)
          push_pending(P, c, (fmin(P.ev_t[c.next], c.t) - c.t_old) / c.h_last);
        const bool more = c.next < P.n_ev && P.ev_t[c.next] <= c.t + P.eps_t;
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

cudaError_t launch_grid_dp5(const GridProblem& P, int mode, int st, int grid, cudaStream_t s) {
  if (mode == 0)
    return st == 2 ? launch_one<0, 2>(P, grid, s) : st == 1 ? launch_one<0, 1>(P, grid, s) : launch_one<0, 0>(P, grid, s);
  return st == 2 ? launch_one<1, 2>(P, grid, s) : st == 1 ? launch_one<1, 1>(P, grid, s) : launch_one<1, 0>(P, grid, s);
}

}  // namespace qsg

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
