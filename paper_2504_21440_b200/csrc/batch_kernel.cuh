// Batched Dormand-Prince 5(4) engine for many independent systems: Monte-Carlo trajectories
// (mcsolve, trajectories.cpp:106-249) and parameter-sweep points (one mesolve per point).
//
// Each CTA owns B = 8 "slots"; the state vectors of its slots are interleaved as [n][B] so that
// lane l of a warp works on (row = 4*warp_iter + l/8, slot = l%8): a CSR entry of a row is
// loaded once and broadcast to the 8 slots, and the gather x[col] of the 8 slots is one
// contiguous 128 B line. Slots run their own integrator state machines in lock-step "rounds"
// of passes; a finished slot pulls the next system from a global queue (dynamic load balance),
// trajectory i always drawing from RngStream(seed, i) (trajectories.cpp:42), so results do not
// depend on the CTA, slot or GPU count that ran them.
//
// Round (per slot phase):            P1        P2          P3        P4..P5  P6        P7
//   START  (start + initial_step)    k1,d0,d1  k2,d2       -         -       -         -
//   RUN    (one DP5 attempt)         stage 2   stage 3     stage 4   5, 6    7 + err   commit/Gram
//   JUMP   (trajectories.cpp:177-203) obs+wts  collapse    restart   -       -         -
//   OBS / FINISH                     obs       -           -         -       -         -
// Jump location: |psi(theta)|^2 of the dense output is a polynomial whose coefficients come from
// the Gram matrix of rc1..rc5 (one fused reduction in P7); the reference's <=200-step bisection
// (trajectories.cpp:156-168) then runs on scalars in every thread of the slot.
#pragma once
#include <cstdio>

#include "batch_engine.h"
#include "engine.cuh"

namespace qsg {
namespace {  // internal linkage: every batch_layout_*.cu gets its own copy

constexpr int kMaxB = 32;       // slots per batch (B = 8 CTA-local, 32 grid-wide)
#ifndef QSG_BATCH_THREADS
#define QSG_BATCH_THREADS 512
#endif
constexpr int kThreads = QSG_BATCH_THREADS;  // 16 warps by default
constexpr int W = kThreads / 32;
constexpr int NBUF = 12;
#ifndef QSG_BATCH_KO
#define QSG_BATCH_KO 5  // observation pairs per reduction (2 measured no faster on TFIM-14)
#endif
#ifndef QSG_BATCH_KJ
#define QSG_BATCH_KJ 15  // jump channels per reduction (5 measured no faster)
#endif
#ifndef QSG_BATCH_UNROLL
#define QSG_BATCH_UNROLL 4
#endif
#ifndef QSG_BATCH_MINB
#define QSG_BATCH_MINB 2
#endif

// Y1 (ysti7) shares SA and SC (collapsed state) shares SB: their live ranges never overlap for
// a given slot (SA holds ysti5 until P4, ysti7 from P5 to the P7 commit; a JUMP slot writes SC in
// P2 and consumes it in P3 while it runs no stages).
enum Buf { Y = 0, YO, K1, K1O, K2, K3, K4, K5, K6, K7, SA, SB, Y1 = SA, SC = SB };
enum Phase { FREE = 0, START, RUN, JUMP, OBS, FINISH, DONE };
enum Src { SRC_DENSE = 0, SRC_Y = 1, SRC_SC = 2 };
// Group modes: who shares one batch of slots.
//   GM_CTA:     each CTA runs its own batch over all rows (block barriers only).
//   GM_GRID:    one batch for the whole cooperative grid, rows partitioned over CTAs, passes
//               separated by software grid barriers.
//   GM_CLUSTER: one batch per thread-block cluster, rows partitioned over the cluster's CTAs,
//               passes separated by hardware cluster barriers, slot reductions through DSMEM.
//   GM_DSM:     as GM_CLUSTER, but every state array lives in the shared memory of the CTA that
//               owns the rows (1 << dsm_shift each); gathers read the owner's shared memory
//               (DSMEM), so no pass touches L2 for the state.
enum GroupMode { GM_CTA = 0, GM_GRID = 1, GM_CLUSTER = 2, GM_DSM = 3 };

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// loads from the shared memory of CTA `rank` of this cluster (DSMEM)
__device__ __forceinline__ double dsmem_ld(const double* p, unsigned rank) {
  unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(p)), ra;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long dsmem_ld_u64(const unsigned long long* p, unsigned rank) {
  unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(p)), ra;
  unsigned long long v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
  return v;
}

struct Slot {
  int phase, next_phase, after_obs;
  long long sys;  // index relative to sys_begin
  int status;
  double t, t_old, h, h_last, facold, h0, hh;
  int clamped, attempts, accepted, crossing, fresh;
  long long steps, rejected, rhs_evals;
  unsigned long long rng[4];
  double r, jump_t, d0, d1;
  int channel, njumps, grid;
  double obs_limit;  // grid points <= obs_limit + eps_t are observed from the dense output
  int tail_src;      // -1, or the direct source that takes every later grid point
  int n_pend;
  double pend_theta[kBatchMaxPend];
  int pend_grid[kBatchMaxPend];
  int pend_src[kBatchMaxPend];
  double w[kBatchMaxCops];
  double gram[15];
  double nrm2, err;
};

__device__ __forceinline__ unsigned long long rotl64(unsigned long long x, int k) {
  return (x << k) | (x >> (64 - k));
}
__device__ void rng_init(unsigned long long* s, unsigned long long seed, unsigned long long stream) {
  unsigned long long z = seed ^ ((stream + 1) * 0x9E3779B97F4A7C15ULL);  // rng.cpp:21-25
  for (int i = 0; i < 4; ++i) {
    unsigned long long x = (z += 0x9E3779B97F4A7C15ULL);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    s[i] = x ^ (x >> 31);
  }
  if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
}
__device__ unsigned long long rng_next(unsigned long long* s) {  // rng.cpp:27-37
  const unsigned long long result = rotl64(s[0] + s[3], 23) + s[0];
  const unsigned long long t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}
__device__ double rng_uniform(unsigned long long* s) { return static_cast<double>(rng_next(s) >> 11) * 0x1.0p-53; }
__device__ double rng_uniform_pos(unsigned long long* s) {
  double u = rng_uniform(s);
  while (u == 0.0) u = rng_uniform(s);
  return u;
}

// Logical buffer k of slot s lives in physical array map[s][k]: an accepted step relabels
// (Y, YO, Y1) and (K1, K1O, K7) instead of copying them (FSAL, integrator.hpp:135-137).
template <int BS, bool NA = true, bool DSM = false>
struct Ctx {
  const BatchProblem& P;
  double2* w;  // batch workspace: NBUF arrays of [n][BS] (DSM: this CTA's rows, in shared memory)
  int n;
  const unsigned char (*map)[NBUF];  // shared memory, per slot
  int shift = 0, r_lo = 0;           // DSM: rows per CTA = 1 << shift, first row of this CTA
  __device__ double2* buf(int k, int s) const {
    if constexpr (DSM) return w + (static_cast<long long>(map[s][k]) << shift) * BS;
    else return w + static_cast<long long>(map[s][k]) * n * BS;
  }
  __device__ long long at(int r, int s) const {
    if constexpr (DSM) return static_cast<long long>(r - r_lo) * BS + s;
    else return static_cast<long long>(r) * BS + s;
  }
  // ld: operands streamed once per pass (NA: L1::no_allocate keeps L1 for the gathers; measured
  // +1.8% on TFIM-14 mcsolve, -2.4% on the cluster-layout sweep, so cluster layouts keep L1
  // allocation); ldx: gathers and dense-output reads (L1-allocating; DSM: from the owner CTA)
  __device__ double2 ld(int k, int r, int s) const {
    const double2* p = buf(k, s) + at(r, s);
    if constexpr (NA && !DSM) return ld_na_c2(p);
    else return *p;
  }
  __device__ double2 ldx(int k, int c, int s) const {
    if constexpr (DSM) {
      const unsigned owner = static_cast<unsigned>(c) >> shift;
      const double2* p = buf(k, s) + (static_cast<long long>(c & ((1 << shift) - 1)) * BS + s);
      unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(p)), ra;
      double2 v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(owner));
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
      return v;
    } else {
      return buf(k, s)[static_cast<long long>(c) * BS + s];
    }
  }
  __device__ void st(int k, int r, int s, double2 v) const { buf(k, s)[at(r, s)] = v; }
};

// dense output of slot s at index c (integrator.hpp:127-131,150-154) from the committed step
template <int BS, bool NA, bool DSM>
__device__ __forceinline__ double2 dense_at(const Ctx<BS, NA, DSM>& C, int c, int s, double theta, double h, int src) {
  if (src == SRC_Y) return C.ldx(Y, c, s);
  if (src == SRC_SC) return C.ldx(SC, c, s);
  using namespace dp;
  // after the commit relabelling K1 holds the step's k7 (FSAL) and K1O its k1
  const double2 yo = C.ldx(YO, c, s), y1 = C.ldx(Y, c, s), k1 = C.ldx(K1O, c, s), k7 = C.ldx(K1, c, s);
  const double2 k3 = C.ldx(K3, c, s), k4 = C.ldx(K4, c, s), k5 = C.ldx(K5, c, s), k6 = C.ldx(K6, c, s);
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

// One row of a key-aligned store (engine.cuh DevSell::ka_*; the grid engine's ka_row) when a warp
// holds one slice, i.e. 32 consecutive rows of one slot: the slice block's words are read at
// warp-uniform addresses through L1 (the whole store is a few tens of KB here), the value groups
// sum their gathers before one multiply, and no per-entry column or value is loaded.
template <class XF>
__device__ __forceinline__ double2 ka_row_slot(const DevSell& A, int row, XF&& xf) {
  const unsigned bit = 1u << (row & 31);
  const unsigned* __restrict__ w = reinterpret_cast<const unsigned*>(A.ka_blk) + 4ull * __ldg(A.ka_off + (row >> 5));
  const uint4 h = __ldg(reinterpret_cast<const uint4*>(w));
  const int G = static_cast<int>(h.x), NN = static_cast<int>(h.y), Pu = static_cast<int>(h.z);
  const unsigned* kw_p = w + kKaHdrWords + G;
  const unsigned* mk_p = kw_p + Pu;
  double2 acc = make_double2(0.0, 0.0);
  for (int g = 0; g < G; ++g) {
    const unsigned gw = __ldg(w + kKaHdrWords + g);
    const int cnt = static_cast<int>(gw >> 16);
    double2 sum = make_double2(0.0, 0.0);
    for (int c = 0; c < cnt; c += 4) {
      unsigned kw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) kw[u] = c + u < cnt ? __ldg(kw_p + u) : 0x80000000u;
      double2 x[4];
      int q = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool part = static_cast<int>(kw[u]) < 0;
        const unsigned m = part ? (c + u < cnt ? __ldg(mk_p + q) : 0u) : 0xffffffffu;
        q += (part && c + u < cnt) ? 1 : 0;
        x[u] = (m & bit) ? xf((row ^ static_cast<int>(kw[u])) & 0x7fffffff) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) sum = cadd(sum, x[u]);
      kw_p += 4;
      mk_p += q;
    }
    kw_p += cnt - ((cnt + 3) & ~3);
    cfma(__ldg(A.ka_val + (gw & 0xffffu)), sum, acc);
  }
  const unsigned* ep = mk_p;
  for (int e = 0; e < NN; ++e, ep += kKaNonUniWords) {
    const unsigned key = __ldg(ep), msk = __ldg(ep + 1);
    if (msk & bit) {
      const unsigned short vid = __ldg(reinterpret_cast<const unsigned short*>(ep + 2) + (row & 31));
      cfma(__ldg(A.ka_val + vid), xf(row ^ static_cast<int>(key)), acc);
    }
  }
  return acc;
}

// one row of a SELL operator applied to slot s of a gathered vector (plain or dictionary-coded
// store, engine.cuh DevSell); the row's entries are broadcast to the slots of the warp.
// KA: the caller's warp holds whole slices of one slot, so a key-aligned store may be used.
template <bool KA = false, class XF>
__device__ __forceinline__ double2 sell_row_slot(const DevSell& A, int row, XF&& xf) {
  // QSG_BATCH_LEAN (the batch_layout_lean_*.cu instantiations, chosen when every operator of the
  // batch is a plain SELL store): no key-aligned or dictionary-coded branch in any of the inlined
  // row loops. Their cold code would otherwise sit between the hot passes and push the per-round
  // working set out of the SM's instruction cache (ncu, TFIM-14 mcsolve: no_instruction stalls
  // 5.06 -> 2.09 per issue, 192 -> 171 ms; profiles/r02_batch_lean.log).
#ifndef QSG_BATCH_LEAN
  if constexpr (KA) {
    if (A.ka_nval > 0) return ka_row_slot(A, row, xf);
  }
#endif
  const int sl = row >> 5, ln = row & 31;
  const int len = __ldg(A.rowlen + row);
  double2 acc = make_double2(0.0, 0.0);
#ifdef QSG_BATCH_LEAN
  if (true) {
#else
  if (A.code_bytes == 0) {
#endif
    const long long base = __ldg(A.slice_off + sl) * 32 + ln;
    for (int j = 0; j < len; j += QSG_BATCH_UNROLL) {
      int c[QSG_BATCH_UNROLL];
      double2 v[QSG_BATCH_UNROLL];
#pragma unroll
      for (int u = 0; u < QSG_BATCH_UNROLL; ++u) {
        if (j + u < len) {
          c[u] = __ldg(A.col + base + 32LL * (j + u));
          v[u] = __ldg(A.val + base + 32LL * (j + u));
        } else {
          c[u] = 0;
          v[u] = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < QSG_BATCH_UNROLL; ++u)
        if (j + u < len) cfma(v[u], xf(c[u]), acc);
    }
  } else {
    const long long cb = __ldg(A.code_off + sl);
    const long long base = cb + 8LL * ln;  // interleaved groups of 8 codes (qsg_capi.cu)
    for (int j = 0; j < len; j += 8) {
      uint4 w;
      if (A.code_bytes == 1) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(A.code8 + base + 32LL * j));
        w = make_uint4(v.x, v.y, 0u, 0u);
      } else {
        w = __ldg(reinterpret_cast<const uint4*>(A.code16 + base + 32LL * j));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u < len) {
          unsigned k;
          if (A.code_bytes == 1) k = ((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xffu;
          else k = ((u < 2 ? w.x : u < 4 ? w.y : u < 6 ? w.z : w.w) >> (16 * (u & 1))) & 0xffffu;
          cfma(__ldg(A.dict_val + k), xf(row + __ldg(A.dict_off + k)), acc);
        }
    }
  }
  return acc;
}

// Inlined at each of the 9 call sites: an out-of-line copy per gather source (lambda captures
// through the stack, ABI register saves) measured 595 / 508 traj/s against 785 / 767 (TFIM-14,
// 2,368 trajectories, key-aligned / plain rows; profiles/r02_batch_noinline_ab.log).
template <bool KA = false, class XF>
__device__ __forceinline__ double2 gen_row_slot(const DevGen& g, const double* params, int row, double t,
                                                XF&& xf) {
  double2 s = sell_row_slot<KA>(g.A[0], row, xf);
#if defined(QSG_BATCH_LEAN) && QSG_BATCH_LEAN == 2
  // single-term instantiation (batch_layout_lean1_*.cu): no second inlined row loop
#else
  for (int k = 1; k < g.n_terms; ++k) {
    const double2 sk = sell_row_slot<KA>(g.A[k], row, xf);
    s = cadd(s, cmul(coeff_eval(g.c[k], params, t), sk));
  }
#endif
  return s;
}

__device__ __forceinline__ void prefetch_row(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Deterministic per-slot reduction of NA accumulators -> out[slot*NA + a] (shared memory).
// GRID: the CTA totals go to gpart[value][rank]; the last CTA to arrive sums every value over the
// CTAs in rank order (so the result does not depend on arrival order), publishes gfin and
// releases the others. Every CTA then holds identical totals.
template <int BS, int GM, int NA>
__device__ void slot_reduce(const BatchProblem& P, double (&acc)[NA], double* sred, double* out, double* pub) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, s = lane % BS, rs = lane / BS;
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int off = BS; off < 32; off <<= 1) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], off);
  if (rs == 0)
#pragma unroll
    for (int a = 0; a < NA; ++a) sred[(warp * BS + s) * NA + a] = acc[a];
  __syncthreads();
  if (threadIdx.x < BS * NA) {
    const int ss = threadIdx.x / NA, a = threadIdx.x % NA;
    double v = 0.0;
    for (int w = 0; w < W; ++w) v += sred[(w * BS + ss) * NA + a];
    out[ss * NA + a] = v;
  }
  __syncthreads();
  if constexpr (GM == GM_CLUSTER || GM == GM_DSM) {
    // every CTA publishes its totals in its own shared memory (double-buffered by the caller, so
    // the next reduction cannot overwrite a buffer another CTA is still reading), then sums the
    // cluster's totals in rank order: identical results in every CTA of the cluster. The (<= 16)
    // remote loads are all issued before the in-order sum, so their latencies overlap.
    const int cnt = BS * NA;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) pub[i] = out[i];
    cluster_sync_all();
    const unsigned cs = cluster_size();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      double t[16];
#pragma unroll
      for (unsigned r = 0; r < 16; ++r) t[r] = r < cs ? dsmem_ld(pub + i, r) : 0.0;
      double v = 0.0;
#pragma unroll
      for (unsigned r = 0; r < 16; ++r)
        if (r < cs) v += t[r];
      out[i] = v;
    }
    __syncthreads();
  }
  if constexpr (GM == GM_GRID) {
    // two-phase distributed reduce: every CTA publishes its totals, then value i is summed over
    // the CTAs in rank order by one warp of CTA (i mod G); a second barrier publishes the result.
    const int G = gridDim.x, rank = blockIdx.x, cnt = BS * NA;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) P.gpart[static_cast<long long>(i) * G + rank] = out[i];
    grid_barrier(P.bar, G);
    for (int i = rank + warp * G; i < cnt; i += W * G) {
      double v = 0.0;
      for (int g = lane; g < G; g += 32) v += P.gpart[static_cast<long long>(i) * G + g];
      v = warp_sum(v);
      if (lane == 0) P.gfin[i] = v;
    }
    grid_barrier(P.bar, G);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[i] = P.gfin[i];
    __syncthreads();
  }
}

__device__ double params_at(const BatchProblem& P, const Slot& S, int i) {
  return P.mode == 1 ? P.params[(P.sys_begin + S.sys) * P.n_params + i] : P.params[i];
}

// per-slot parameter pointer for generator coefficients
__device__ __forceinline__ const double* slot_params(const BatchProblem& P, const Slot& S) {
  if (!P.params) return nullptr;
  return P.mode == 1 ? P.params + (P.sys_begin + S.sys) * P.n_params : P.params;
}

// Queue the next grid points of a slot: dense-output points first (<= obs_limit + eps_t), then,
// if a tail source is set, every remaining point from that direct state.
__device__ void refill(Slot& s, const BatchProblem& P) {
  while (s.n_pend < kBatchMaxPend && s.grid < P.n_t) {
    if (P.tlist[s.grid] <= s.obs_limit + P.eps_t) {
      s.pend_theta[s.n_pend] = (fmin(P.tlist[s.grid], s.t) - s.t_old) / s.h_last;
      s.pend_src[s.n_pend] = SRC_DENSE;
    } else if (s.tail_src >= 0) {
      s.pend_theta[s.n_pend] = 0.0;
      s.pend_src[s.n_pend] = s.tail_src;
    } else {
      break;
    }
    s.pend_grid[s.n_pend] = s.grid;
    ++s.n_pend;
    ++s.grid;
  }
}
__device__ bool has_more(const Slot& s, const BatchProblem& P) {
  return s.grid < P.n_t && (P.tlist[s.grid] <= s.obs_limit + P.eps_t || s.tail_src >= 0);
}

// BS slots per batch. !GRID: every CTA runs its own batch over all rows (block barriers only).
// GRID: one batch for the whole cooperative grid, rows partitioned over CTAs, so the state of
// the BS slots (NBUF x n x BS complex) stays L2-resident; passes are separated by grid barriers.
template <int BS, int GM>
__global__ void __launch_bounds__(kThreads, QSG_BATCH_MINB) batch_kernel(const __grid_constant__ BatchProblem P) {
  constexpr bool GRID = GM == GM_GRID;
  constexpr bool DSM = GM == GM_DSM;
  constexpr bool CLU = GM == GM_CLUSTER || DSM;
  constexpr bool PART = GM != GM_CTA;  // rows partitioned over the CTAs of a group
  constexpr int B = BS;
  constexpr int RPW = 32 / BS;
  __shared__ Slot S[BS];
  extern __shared__ double sred[];  // W * BS * 15 (dynamic: up to 61 KB for the grid batch)
  __shared__ double sout[BS * 15];
  __shared__ int s_alldone;
  __shared__ long long s_next;
  __shared__ unsigned char s_map[BS][NBUF];
  __shared__ double s_pub[2][BS * 15];            // cluster mode: published CTA totals
  __shared__ unsigned long long s_assign[BS];     // cluster mode: systems drawn by rank 0

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sl = lane % B, rs = lane / B;
  const int n = P.n;
  const int g_rank = GRID ? static_cast<int>(blockIdx.x) : CLU ? static_cast<int>(cluster_rank()) : 0;
  const int g_size = GRID ? static_cast<int>(gridDim.x) : CLU ? static_cast<int>(cluster_size()) : 1;
  const long long batch_id = GRID ? 0LL : CLU ? static_cast<long long>(blockIdx.x) / g_size : blockIdx.x;
  // DSM: the state arrays follow the reduction scratch in dynamic shared memory (16-B aligned)
  double2* const dsm_w = reinterpret_cast<double2*>(
      reinterpret_cast<unsigned char*>(sred) + ((static_cast<size_t>(W) * BS * 15 * sizeof(double) + 15) & ~size_t(15)));
  const int rows_dsm = 1 << P.dsm_shift;
  const double atol = P.atol, rtol = P.rtol, eps_t = P.eps_t, tf = P.tf, t0 = P.t0;
  const bool out_cta = g_rank == 0;  // the CTA of a group that writes per-system outputs
  const int rpc = DSM ? rows_dsm : PART ? (n + g_size - 1) / g_size : n;
  const int r_lo = PART ? min(n, g_rank * rpc) : 0;
  const int r_hi = PART ? min(n, r_lo + rpc) : n;
  const Ctx<BS, !CLU, DSM> C{P, DSM ? dsm_w : P.work + batch_id * P.work_stride, n, s_map, P.dsm_shift, r_lo};
  int pub_par = 0;
  auto rows = [&](auto&& f) {
    for (int r = r_lo + warp * RPW + rs; r < r_hi; r += W * RPW) f(r);
  };
  // RUN stages: the epilogue operands of this lane's next row (logical buffers in `mask`) are
  // prefetched into L2 while the current row's SpMV chain is in flight
  auto rows_pf = [&](unsigned mask, auto&& f) {
    const int step = W * RPW;
    for (int r = r_lo + warp * RPW + rs; r < r_hi; r += step) {
      const int rn = r + step;
      if (!DSM && rn < r_hi)
        for (int k = 0; k < NBUF; ++k)
          if ((mask >> k) & 1u) prefetch_row(C.buf(k, sl) + static_cast<long long>(rn) * BS + sl);
      f(r);
    }
  };
  auto pass_sync = [&]() {
    if constexpr (GRID) grid_barrier(P.bar, gridDim.x);
    else if constexpr (CLU) cluster_sync_all();
    else __syncthreads();
  };
  auto reduce = [&](auto& acc) {
    slot_reduce<BS, GM>(P, acc, sred, sout, s_pub[pub_par]);
    pub_par ^= 1;
  };

  if (threadIdx.x < B) {
    S[threadIdx.x].phase = FREE;
    S[threadIdx.x].next_phase = FREE;
  }
  if (threadIdx.x == 0) s_next = 0;
  __syncthreads();

  for (;;) {
    // ---------------- slot bookkeeping (one thread per slot) ----------------
    if (GRID && threadIdx.x == 0) {  // deterministic assignment: identical in every CTA
      for (int b = 0; b < B; ++b)
        if (S[b].phase == FREE) S[b].sys = s_next < P.n_systems ? s_next++ : -1;
    }
    if (GRID) __syncthreads();
    if constexpr (CLU) {  // rank 0 draws the next systems from the queue, the cluster reads them
      bool anyfree = false;
      for (int b = 0; b < B; ++b) anyfree |= S[b].phase == FREE;
      if (anyfree) {
        if (g_rank == 0 && threadIdx.x < B && S[threadIdx.x].phase == FREE)
          s_assign[threadIdx.x] = atomicAdd(P.queue, 1ull);
        cluster_sync_all();
      }
    }
    if (threadIdx.x < B) {
      Slot& s = S[threadIdx.x];
      s.fresh = 0;
      if (s.phase == FREE) {
        unsigned long long idx;
        if (GRID) idx = s.sys < 0 ? ~0ull : static_cast<unsigned long long>(s.sys);
        else if (CLU) idx = dsmem_ld_u64(&s_assign[threadIdx.x], 0);
        else idx = atomicAdd(P.queue, 1ull);
        if (idx < static_cast<unsigned long long>(P.n_systems)) {
          s.sys = static_cast<long long>(idx);
          for (int k = 0; k < NBUF; ++k) s_map[threadIdx.x][k] = static_cast<unsigned char>(k);
          s.phase = START;
          s.fresh = 1;
          s.status = kRunning;
          s.t = s.t_old = t0;
          s.h = s.h_last = 0.0;
          s.facold = 1e-4;
          s.steps = s.rejected = s.rhs_evals = 0;
          s.attempts = 0;
          s.njumps = 0;
          s.grid = 0;
          s.n_pend = 0;
          s.obs_limit = -1e300;
          s.tail_src = -1;
          // events at t0 observe y0 directly (evolve.cpp:134-137, trajectories.cpp:142)
          if (P.mode == 0) {
            s.pend_theta[0] = 0.0;
            s.pend_grid[0] = 0;
            s.pend_src[0] = SRC_Y;
            s.n_pend = 1;
            s.grid = 1;
            rng_init(s.rng, P.seed, static_cast<unsigned long long>(P.sys_begin + s.sys));
            s.r = rng_uniform_pos(s.rng);  // trajectories.cpp:144
          } else {
            while (s.grid < P.n_t && P.tlist[s.grid] <= t0 + eps_t && s.n_pend < kBatchMaxPend) {
              s.pend_theta[s.n_pend] = 0.0;
              s.pend_grid[s.n_pend] = s.grid;
              s.pend_src[s.n_pend] = SRC_Y;
              ++s.n_pend;
              ++s.grid;
            }
          }
        } else {
          s.phase = DONE;
        }
      }
      s.next_phase = s.phase;
      if (s.phase == RUN) {
        // Dopri5::step prologue (integrator.hpp:80-89) and the max_steps guard (:157-159)
        if (s.attempts == 0 && s.steps >= P.max_steps) {
          s.status = kFailMaxSteps;
        } else {
          s.hh = fmin(s.h, tf - s.t);
          s.clamped = s.hh < s.h;
          if (!(s.hh > 0.0)) s.status = kFailPastEnd;
          else if (s.hh <= fabs(s.t) * 1e-15 + 1e-300) s.status = kFailUnderflow;
          else if (++s.attempts > 1000) s.status = kFailRejected;
        }
        if (s.status != kRunning) {
          s.phase = FINISH;
          s.n_pend = 0;
        }
      }
    }
    if (threadIdx.x == 0) {
      int all = 1;
      for (int b = 0; b < B; ++b) all &= (S[b].phase == DONE);
      s_alldone = all;
    }
    __syncthreads();
    if (s_alldone) break;
    const int ph = S[sl].phase;

    // fresh slots: y <- y0
    rows([&](int r) {
      if (S[sl].fresh) C.st(Y, r, sl, P.y0[r]);
    });
    pass_sync();

    // ================= P1 =================
    {
      double acc[2] = {0.0, 0.0};
      const double* prm = slot_params(P, S[sl]);
      if (ph == START) {
        rows([&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, t0, [&](int c) { return C.ldx(Y, c, sl); });
          C.st(K1, r, sl, k);
          const double2 yy = C.ld(Y, r, sl);
          const double sc = atol + rtol * cabs_(yy);
          acc[0] += cnorm(make_double2(yy.x / sc, yy.y / sc));
          acc[1] += cnorm(make_double2(k.x / sc, k.y / sc));
        });
      } else if (ph == RUN) {
        const double hh = S[sl].hh, t = S[sl].t;
        using namespace dp;
        rows_pf((1u << Y) | (1u << K1), [&](int r) {
          double2 k;
          if (P.autonomous) {
            // k1 = G y exactly (start / restart, FSAL, unchanged after a rejection), so
            // k2 = G(y + h a21 k1) = k1 + (h a21) G k1: one gathered vector instead of two
            k = gen_row_slot<true>(P.gen, prm, r, t + c2 * hh, [&](int c) { return C.ldx(K1, c, sl); });
          } else {
            k = gen_row_slot<true>(P.gen, prm, r, t + c2 * hh, [&](int c) {
              const double2 a = C.ldx(Y, c, sl), q = C.ldx(K1, c, sl);
              return make_double2(a.x + hh * (a21 * q.x), a.y + hh * (a21 * q.y));
            });
          }
          const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl);
          if (P.autonomous) k = make_double2(q1.x + (hh * a21) * k.x, q1.y + (hh * a21) * k.y);
          C.st(K2, r, sl, k);
          C.st(SA, r, sl, make_double2(yy.x + hh * (a31 * q1.x + a32 * k.x), yy.y + hh * (a31 * q1.y + a32 * k.y)));
        });
      }
      bool any_start = false;
      for (int b = 0; b < B; ++b) any_start |= (S[b].phase == START);
      if (any_start) reduce(acc);
      if (threadIdx.x < B && S[threadIdx.x].phase == START) {
        Slot& s = S[threadIdx.x];
        s.d0 = sqrt(sout[threadIdx.x * 2] / static_cast<double>(n));
        s.d1 = sqrt(sout[threadIdx.x * 2 + 1] / static_cast<double>(n));
        double h0 = (s.d0 < 1e-5 || s.d1 < 1e-5) ? 1e-6 : 0.01 * s.d0 / s.d1;  // integrator.hpp:168-170
        h0 = fmin(h0, tf - s.t);
        if (!(h0 > 0)) h0 = 1e-6;
        s.h0 = h0;
        s.rhs_evals += 1;
      }
      // ---- pending observations (every phase may carry some)
      int maxp = 0;
      for (int b = 0; b < B; ++b) maxp = max(maxp, S[b].phase == DONE ? 0 : S[b].n_pend);
      const int npairs = maxp * P.n_e;
      // KO (event, e_op) pairs x 3 values per reduction
      constexpr int KO = QSG_BATCH_KO;
      for (int c0 = 0; c0 < npairs; c0 += KO) {
        double oa[3 * KO];
#pragma unroll
        for (int a = 0; a < 3 * KO; ++a) oa[a] = 0.0;
#pragma unroll
        for (int u = 0; u < KO; ++u) {
          if (c0 + u >= npairs) continue;
          const int q = (c0 + u) / P.n_e, e = (c0 + u) % P.n_e;
          const bool act = q < S[sl].n_pend && S[sl].phase != DONE;
          if (!act) continue;
          const double th = S[sl].pend_theta[q];
          const int src = S[sl].pend_src[q];
          const double hl = S[sl].h_last;
          if (P.mode == 0) {  // <g|E g> / |g|^2 (trajectories.cpp:133-139)
            rows([&](int r) {
              const double2 ev = sell_row_slot(P.e_ops[e], r, [&](int c) { return dense_at(C, c, sl, th, hl, src); });
              const double2 g = dense_at(C, r, sl, th, hl, src);
              const double2 pr = cmul(cconj(g), ev);
              oa[3 * u] += pr.x;
              oa[3 * u + 1] += pr.y;
              oa[3 * u + 2] += cnorm(g);
            });
          } else {  // sum A(i,j) rho_h(j,i) (evolve.cpp:286-295)
            const int beg = P.eo_off[e], end = P.eo_off[e + 1];
            const int r0 = PART ? beg + (end - beg) * static_cast<long long>(g_rank) / g_size : beg;
            const int r1 = PART ? beg + (end - beg) * static_cast<long long>(g_rank + 1) / g_size : end;
            for (int k = r0 + warp * RPW + rs; k < r1; k += W * RPW) {
              const int i = P.eo_i[k], j = P.eo_j[k];
              const double2 rji = dense_at(C, i * P.d + j, sl, th, hl, src);
              const double2 rij = dense_at(C, j * P.d + i, sl, th, hl, src);
              const double2 v = cmul(P.eo_v[k], cscale(0.5, cadd(rji, cconj(rij))));
              oa[3 * u] += v.x;
              oa[3 * u + 1] += v.y;
            }
          }
        }
        reduce(oa);
        if (threadIdx.x < B && S[threadIdx.x].phase != DONE && out_cta) {
          Slot& s = S[threadIdx.x];
          for (int u = 0; u < KO && c0 + u < npairs; ++u) {
            const int q = (c0 + u) / P.n_e, e = (c0 + u) % P.n_e;
            if (q >= s.n_pend) continue;
            double2 v = make_double2(sout[threadIdx.x * 3 * KO + 3 * u], sout[threadIdx.x * 3 * KO + 3 * u + 1]);
            if (P.mode == 0) {
              const double inv = 1.0 / sout[threadIdx.x * 3 * KO + 3 * u + 2];
              v = make_double2(v.x * inv, v.y * inv);
            }
            P.expect[s.sys * P.n_e * P.n_t + static_cast<long long>(s.pend_grid[q]) * P.n_e + e] = v;
          }
        }
        __syncthreads();
      }
      __syncthreads();
      // ---- jump weights |C_k g(jump_t)|^2 (trajectories.cpp:178-196), chunks of 8 channels
      if (P.mode == 0) {
        bool anyj = false;
        for (int b = 0; b < B; ++b) anyj |= (S[b].phase == JUMP);
        if (anyj) {
          const double thj = (S[sl].jump_t - S[sl].t_old) / S[sl].h_last, hl = S[sl].h_last;
          constexpr int KJ = QSG_BATCH_KJ;  // channels per reduction (each inlines a row loop)
          for (int k0 = 0; k0 < P.n_c; k0 += KJ) {
            double wa[KJ];
#pragma unroll
            for (int u = 0; u < KJ; ++u) wa[u] = 0.0;
            if (ph == JUMP) {
              rows([&](int r) {
#pragma unroll
                for (int u = 0; u < KJ; ++u)
                  if (k0 + u < P.n_c) {
                    const double2 v = sell_row_slot(P.c_ops[k0 + u], r,
                                                    [&](int c) { return dense_at(C, c, sl, thj, hl, SRC_DENSE); });
                    wa[u] += cnorm(v);
                  }
              });
            }
            reduce(wa);
            if (threadIdx.x < B && S[threadIdx.x].phase == JUMP)
              for (int u = 0; u < KJ && k0 + u < P.n_c; ++u) S[threadIdx.x].w[k0 + u] = sout[threadIdx.x * KJ + u];
          }
          __syncthreads();
          if (threadIdx.x < B && S[threadIdx.x].phase == JUMP) {
            Slot& s = S[threadIdx.x];
            double total = 0.0;
            for (int k = 0; k < P.n_c; ++k) total += s.w[k];
            if (total <= 0.0) {
              s.status = kFailJumpWeights;
              s.next_phase = FINISH;
            } else {
              const double u = rng_uniform(s.rng) * total;
              int ch = 0;
              double a = 0.0;
              for (; ch < P.n_c; ++ch) {
                a += s.w[ch];
                if (u < a) break;
              }
              if (ch == P.n_c) ch = P.n_c - 1;
              s.channel = ch;
              if (out_cta && s.njumps < P.jump_cap) {
                P.jump_time[s.sys * P.jump_cap + s.njumps] = s.jump_t;
                P.jump_channel[s.sys * P.jump_cap + s.njumps] = ch;
              }
              ++s.njumps;
              s.r = rng_uniform_pos(s.rng);  // trajectories.cpp:201
            }
          }
        }
      }
      if (threadIdx.x < B) {
        Slot& s = S[threadIdx.x];
        if (s.phase != DONE) s.n_pend = 0;
      }
      pass_sync();
    }

    // ================= P2 =================
    {
      double acc[1] = {0.0};
      const double* prm = slot_params(P, S[sl]);
      const int ph2 = S[sl].phase;
      if (ph2 == START) {
        const double h0 = S[sl].h0;
        rows([&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, t0 + h0, [&](int c) {
            const double2 a = C.ldx(Y, c, sl), q = C.ldx(K1, c, sl);
            return make_double2(a.x + h0 * q.x, a.y + h0 * q.y);
          });
          const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl);
          const double sc = atol + rtol * cabs_(yy);
          const double2 df = csub(k, q1);
          acc[0] += cnorm(make_double2(df.x / sc, df.y / sc));
        });
      } else if (ph2 == RUN) {
        const double hh = S[sl].hh, t = S[sl].t;
        using namespace dp;
        rows_pf((1u << Y) | (1u << K1) | (1u << K2), [&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, t + c3 * hh, [&](int c) { return C.ldx(SA, c, sl); });
          const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl), q2 = C.ld(K2, r, sl);
          C.st(K3, r, sl, k);
          C.st(SB, r, sl, make_double2(yy.x + hh * (a41 * q1.x + a42 * q2.x + a43 * k.x),
                                       yy.y + hh * (a41 * q1.y + a42 * q2.y + a43 * k.y)));
        });
      } else if (ph2 == JUMP && S[sl].next_phase == JUMP) {
        // collapse: psi <- C_ch g / |C_ch g| (trajectories.cpp:198-199)
        const double thj = (S[sl].jump_t - S[sl].t_old) / S[sl].h_last, hl = S[sl].h_last;
        const int ch = S[sl].channel;
        const double nrm = sqrt(S[sl].w[ch]);
        rows([&](int r) {
          const double2 v = sell_row_slot(P.c_ops[ch], r, [&](int c) { return dense_at(C, c, sl, thj, hl, SRC_DENSE); });
          C.st(SC, r, sl, make_double2(v.x / nrm, v.y / nrm));
        });
      }
      bool any_start = false;
      for (int b = 0; b < B; ++b) any_start |= (S[b].phase == START);
      if (any_start) reduce(acc);
      if (threadIdx.x < B && S[threadIdx.x].phase == START) {
        Slot& s = S[threadIdx.x];
        const double d2 = sqrt(sout[threadIdx.x] / static_cast<double>(n)) / s.h0;  // integrator.hpp:180-186
        double h1;
        if (fmax(s.d1, d2) <= 1e-15) h1 = fmax(1e-6, s.h0 * 1e-3);
        else h1 = pow(0.01 / fmax(s.d1, d2), 0.2);
        s.h = fmin(fmin(100.0 * s.h0, h1), tf - s.t);
        s.rhs_evals += 1;
        s.next_phase = RUN;
      }
      pass_sync();
    }

    // ================= P3 =================
    {
      const double* prm = slot_params(P, S[sl]);
      const int ph3 = S[sl].phase;
      if (ph3 == RUN) {
        const double hh = S[sl].hh, t = S[sl].t;
        using namespace dp;
        rows_pf((1u << Y) | (1u << K1) | (1u << K2) | (1u << K3), [&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, t + c4 * hh, [&](int c) { return C.ldx(SB, c, sl); });
          const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl), q2 = C.ld(K2, r, sl), q3 = C.ld(K3, r, sl);
          C.st(K4, r, sl, k);
          C.st(SA, r, sl, make_double2(yy.x + hh * (a51 * q1.x + a52 * q2.x + a53 * q3.x + a54 * k.x),
                                       yy.y + hh * (a51 * q1.y + a52 * q2.y + a53 * q3.y + a54 * k.y)));
        });
      } else if (ph3 == JUMP && S[sl].next_phase == JUMP && S[sl].jump_t < tf - eps_t) {
        // restart: integ.start(jump_t, psi, tf, h_current) (trajectories.cpp:202-203)
        const double tj = S[sl].jump_t;
        rows([&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, tj, [&](int c) { return C.ldx(SC, c, sl); });
          C.st(K1, r, sl, k);
          C.st(Y, r, sl, C.ld(SC, r, sl));
        });
      }
      pass_sync();
      if (threadIdx.x < B && S[threadIdx.x].phase == JUMP && S[threadIdx.x].next_phase == JUMP) {
        Slot& s = S[threadIdx.x];
        if (s.jump_t < tf - eps_t) {
          s.t = s.t_old = s.jump_t;
          s.facold = 1e-4;
          s.rhs_evals += 1;
          s.attempts = 0;
          s.next_phase = RUN;
        } else {  // trajectories.cpp:204-206: fill the rest of the grid with the jumped state
          s.obs_limit = -1e300;
          s.tail_src = SRC_SC;
          refill(s, P);
          s.next_phase = has_more(s, P) ? OBS : FINISH;
          s.after_obs = FINISH;
        }
      }
      __syncthreads();
    }

    // ================= P4, P5 =================
    if (S[sl].phase == RUN) {
      const double* prm = slot_params(P, S[sl]);
      const double hh = S[sl].hh, t = S[sl].t;
      using namespace dp;
      rows_pf((1u << Y) | (1u << K1) | (1u << K2) | (1u << K3) | (1u << K4), [&](int r) {
        const double2 k = gen_row_slot<true>(P.gen, prm, r, t + c5 * hh, [&](int c) { return C.ldx(SA, c, sl); });
        const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl), q2 = C.ld(K2, r, sl), q3 = C.ld(K3, r, sl),
                      q4 = C.ld(K4, r, sl);
        C.st(K5, r, sl, k);
        C.st(SB, r, sl,
             make_double2(yy.x + hh * (a61 * q1.x + a62 * q2.x + a63 * q3.x + a64 * q4.x + a65 * k.x),
                          yy.y + hh * (a61 * q1.y + a62 * q2.y + a63 * q3.y + a64 * q4.y + a65 * k.y)));
      });
    }
    pass_sync();
    if (S[sl].phase == RUN) {
      const double* prm = slot_params(P, S[sl]);
      const double hh = S[sl].hh, t = S[sl].t;
      using namespace dp;
      rows_pf((1u << Y) | (1u << K1) | (1u << K3) | (1u << K4) | (1u << K5), [&](int r) {
        const double2 k = gen_row_slot<true>(P.gen, prm, r, t + hh, [&](int c) { return C.ldx(SB, c, sl); });
        const double2 yy = C.ld(Y, r, sl), q1 = C.ld(K1, r, sl), q3 = C.ld(K3, r, sl), q4 = C.ld(K4, r, sl),
                      q5 = C.ld(K5, r, sl);
        C.st(K6, r, sl, k);
        C.st(Y1, r, sl,
             make_double2(yy.x + hh * (a71 * q1.x + a73 * q3.x + a74 * q4.x + a75 * q5.x + a76 * k.x),
                          yy.y + hh * (a71 * q1.y + a73 * q3.y + a74 * q4.y + a75 * q5.y + a76 * k.y)));
      });
    }
    pass_sync();

    // ================= P6: stage 7 + embedded error =================
    {
      double acc[2] = {0.0, 0.0};
      if (S[sl].phase == RUN) {
        const double* prm = slot_params(P, S[sl]);
        const double hh = S[sl].hh, t = S[sl].t;
        using namespace dp;
        rows_pf((1u << Y) | (1u << Y1) | (1u << K1) | (1u << K3) | (1u << K4) | (1u << K5) | (1u << K6), [&](int r) {
          const double2 k = gen_row_slot<true>(P.gen, prm, r, t + hh, [&](int c) { return C.ldx(Y1, c, sl); });
          const double2 yy = C.ld(Y, r, sl), y1 = C.ld(Y1, r, sl), q1 = C.ld(K1, r, sl), q3 = C.ld(K3, r, sl),
                        q4 = C.ld(K4, r, sl), q5 = C.ld(K5, r, sl), q6 = C.ld(K6, r, sl);
          C.st(K7, r, sl, k);
          double2 e;
          e.x = hh * (e1 * q1.x + e3 * q3.x + e4 * q4.x + e5 * q5.x + e6 * q6.x + e7 * k.x);
          e.y = hh * (e1 * q1.y + e3 * q3.y + e4 * q4.y + e5 * q5.y + e6 * q6.y + e7 * k.y);
          const double sc = atol + rtol * fmax(cabs_(yy), cabs_(y1));
          const double qq = cabs_(e) / sc;
          acc[0] += qq * qq;
          acc[1] += cnorm(y1);
        });
      }
      reduce(acc);
      if (threadIdx.x < B && S[threadIdx.x].phase == RUN) {
        Slot& s = S[threadIdx.x];
        using namespace dp;
        double err = sqrt(sout[threadIdx.x * 2] / static_cast<double>(n));
        if (!isfinite(err)) err = 10.0;
        s.nrm2 = sout[threadIdx.x * 2 + 1];
        s.rhs_evals += 6;
        if (out_cta) atomicAdd(reinterpret_cast<unsigned long long*>(P.attempts_total), 1ull);
        if (err <= 1.0) {  // integrator.hpp:119-142
          const double fac11 = pow(err, expo1);
          double fac = fac11 / pow(s.facold, beta);
          fac = fmax(facc2, fmin(facc1, fac / safe));
          const double h_new = s.hh / fac;
          s.facold = fmax(err, 1e-4);
          s.t_old = s.t;
          s.t += s.hh;
          s.h_last = s.hh;
          ++s.steps;
          if (!s.clamped) s.h = h_new;
          else s.h = fmax(s.h, h_new);
          s.attempts = 0;
          s.accepted = 1;
          s.crossing = (P.mode == 0 && P.n_c > 0 && s.nrm2 < s.r) ? 1 : 0;  // trajectories.cpp:154
        } else {
          ++s.rejected;
          s.h = s.hh / fmin(facc1, pow(err, expo1) / safe);  // integrator.hpp:144-145
          s.accepted = 0;
          s.crossing = 0;
        }
      }
      __syncthreads();
    }

    // ================= P7: commit + Gram of the dense-output basis =================
    {
      double g[15];
#pragma unroll
      for (int a = 0; a < 15; ++a) g[a] = 0.0;
      const bool acc_ok = S[sl].phase == RUN && S[sl].accepted;
      const bool cross = acc_ok && S[sl].crossing;
      if (cross) {
        const double h = S[sl].h_last;
        using namespace dp;
        rows([&](int r) {
          const double2 yo = C.ld(Y, r, sl), y1 = C.ld(Y1, r, sl), k1 = C.ld(K1, r, sl), k7 = C.ld(K7, r, sl);
          {
            const double2 k3 = C.ld(K3, r, sl), k4 = C.ld(K4, r, sl), k5 = C.ld(K5, r, sl), k6 = C.ld(K6, r, sl);
            double2 rc[5];
            rc[0] = yo;
            rc[1] = csub(y1, yo);
            rc[2] = csub(cscale(h, k1), rc[1]);
            rc[3] = csub(csub(rc[1], cscale(h, k7)), rc[2]);
            rc[4].x = h * (d1 * k1.x + d3 * k3.x + d4 * k4.x + d5 * k5.x + d6 * k6.x + d7 * k7.x);
            rc[4].y = h * (d1 * k1.y + d3 * k3.y + d4 * k4.y + d5 * k5.y + d6 * k6.y + d7 * k7.y);
            int q = 0;
#pragma unroll
            for (int a = 0; a < 5; ++a)
#pragma unroll
              for (int b = a; b < 5; ++b) g[q++] += rc[a].x * rc[b].x + rc[a].y * rc[b].y;  // Re <rc_a, rc_b>
          }
        });
      }
      bool anyc = false;
      for (int b = 0; b < B; ++b) anyc |= (S[b].phase == RUN && S[b].accepted && S[b].crossing);
      if (anyc) reduce(g);
      else __syncthreads();
      if (threadIdx.x < B && S[threadIdx.x].phase == RUN && S[threadIdx.x].accepted) {
        Slot& s = S[threadIdx.x];
        // commit by relabelling: YO <- Y, Y <- Y1, Y1 <- old YO; K1O <- K1, K1 <- K7, K7 <- old K1O
        unsigned char* m = s_map[threadIdx.x];
        const unsigned char y = m[Y], yo = m[YO], y1 = m[Y1], k1 = m[K1], k1o = m[K1O], k7 = m[K7];
        m[YO] = y;
        m[Y] = y1;
        m[Y1] = yo;
        m[K1O] = k1;
        m[K1] = k7;
        m[K7] = k1o;
        double jt = s.t;
        if (s.crossing) {
          for (int a = 0; a < 15; ++a) s.gram[a] = sout[threadIdx.x * 15 + a];
          // bisection on |psi(mid)|^2 - r (trajectories.cpp:156-168)
          double lo = s.t_old, hi = s.t;
          for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            const double th = (mid - s.t_old) / s.h_last, t1 = 1.0 - th;
            const double wv[5] = {1.0, th, th * t1, th * th * t1, th * th * t1 * t1};
            double nn = 0.0;
            int q = 0;
            for (int a = 0; a < 5; ++a)
              for (int b = a; b < 5; ++b, ++q) nn += (a == b ? 1.0 : 2.0) * wv[a] * wv[b] * s.gram[q];
            const double gg = nn - s.r;
            if (fabs(gg) < 1e-10) {
              lo = hi = mid;
              break;
            }
            if (gg > 0) lo = mid;
            else hi = mid;
          }
          jt = 0.5 * (lo + hi);
          s.jump_t = jt;
        }
        // observation events reached by this step (evolve.cpp:160-165 / trajectories.cpp:171-175);
        // after the last step the trailing grid points take the final state directly (:169, :207-208)
        s.n_pend = 0;
        s.obs_limit = jt;
        s.tail_src = (!s.crossing && s.t >= tf - eps_t) ? SRC_Y : -1;
        refill(s, P);
        int after;
        if (s.crossing) after = JUMP;
        else if (s.tail_src >= 0 || s.grid >= P.n_t) after = FINISH;
        else after = RUN;
        s.after_obs = after;
        s.next_phase = has_more(s, P) ? OBS : after;
      }
      __syncthreads();
    }

    // ---------------- round end: outputs of finishing slots, phase advance ----------------
    if (threadIdx.x < B) {
      Slot& s = S[threadIdx.x];
      if (s.phase == FINISH) {  // its last observations were taken in this round's P1
        if (out_cta) {
          P.status[s.sys] = s.status == kRunning ? kDone : s.status;
          P.fail_t[s.sys] = s.t;
          P.stats[s.sys * 3] = s.steps;
          P.stats[s.sys * 3 + 1] = s.rejected;
          P.stats[s.sys * 3 + 2] = s.rhs_evals;
          P.jump_count[s.sys] = s.njumps;
        }
        s.next_phase = FREE;
      } else if (s.phase == OBS) {
        refill(s, P);
        s.next_phase = s.n_pend > 0 ? OBS : s.after_obs;
      }
      if (s.phase != DONE) s.phase = s.next_phase;
    }
    __syncthreads();
  }
  // no CTA may leave while another still reads its shared memory (reductions, rank 0's draws)
  if constexpr (CLU) cluster_sync_all();
}

template <int BS, int GM>
size_t dyn_smem() {
  return static_cast<size_t>(W) * BS * 15 * sizeof(double);
}

template <int BS, int GM>
void set_attrs() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(batch_kernel<BS, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(dyn_smem<BS, GM>()));
    if (GM == GM_CLUSTER) cudaFuncSetAttribute(batch_kernel<BS, GM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done = true;
  }
}

template <int BS, int GM>
int occupancy_of() {
  set_attrs<BS, GM>();
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, batch_kernel<BS, GM>, kThreads, dyn_smem<BS, GM>());
  return nb;
}

template <int BS>
cudaError_t launch_cluster(const BatchProblem& P, int grid, int cs, cudaStream_t s) {
  set_attrs<BS, GM_CLUSTER>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = dyn_smem<BS, GM_CLUSTER>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, batch_kernel<BS, GM_CLUSTER>, P);
}

template <int BS>
int cluster_capacity(int cs) {
  set_attrs<BS, GM_CLUSTER>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = dyn_smem<BS, GM_CLUSTER>();
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, batch_kernel<BS, GM_CLUSTER>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

// GM_DSM: the reduction scratch plus the 12 state arrays of this CTA's 1 << shift rows
size_t dsm_smem_bytes(int shift) {
  return ((static_cast<size_t>(W) * 15 * sizeof(double) + 15) & ~size_t(15)) +
         static_cast<size_t>(NBUF) * (size_t(1) << shift) * sizeof(double2);
}

cudaLaunchConfig_t dsm_cfg(int grid, int cs, size_t smem, cudaLaunchAttribute* at) {
  cudaFuncSetAttribute(batch_kernel<1, GM_DSM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(batch_kernel<1, GM_DSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

}  // namespace
}  // namespace qsg

namespace qsg {
namespace {
// Per-layout entry points as templates, so `if constexpr` discards the other group modes and each
// translation unit instantiates exactly one kernel.
template <int BS, int GM>
int layout_occ() {
  if constexpr (GM == GM_DSM) return 1;
  else return occupancy_of<BS, GM>();
}
// cs CTAs per cluster; GM_DSM: cs = clusters' CTA count with `shift` rows each (shift in cs >> 8)
template <int BS, int GM>
int layout_clusters(int cs) {
  if constexpr (GM == GM_CLUSTER) {
    return cluster_capacity<BS>(cs);
  } else if constexpr (GM == GM_DSM) {
    const int c = cs & 0xff, shift = cs >> 8;
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = dsm_cfg(c * 64, c, dsm_smem_bytes(shift), at);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, batch_kernel<1, GM_DSM>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return nc;
  } else {
    return 0;
  }
}
template <int BS, int GM>
cudaError_t layout_launch(const BatchProblem& P, int grid, int cs, cudaStream_t s) {
  if constexpr (GM == GM_DSM) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = dsm_cfg(grid, cs, dsm_smem_bytes(P.dsm_shift), at);
    cfg.stream = s;
    return cudaLaunchKernelEx(&cfg, batch_kernel<1, GM_DSM>, P);
  } else if constexpr (GM == GM_CLUSTER) {
    return launch_cluster<BS>(P, grid, cs, s);
  } else if constexpr (GM == GM_GRID) {
    void* args[] = {const_cast<BatchProblem*>(&P)};
    set_attrs<BS, GM_GRID>();
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(batch_kernel<BS, GM_GRID>), dim3(grid),
                                       dim3(kThreads), args, dyn_smem<BS, GM_GRID>(), s);
  } else {
    set_attrs<BS, GM_CTA>();
    batch_kernel<BS, GM_CTA><<<grid, kThreads, dyn_smem<BS, GM_CTA>(), s>>>(P);
    return cudaGetLastError();
  }
}
}  // namespace
}  // namespace qsg

// Defines the per-layout entry points of one kernel instantiation (one translation unit each, so
// the seven instantiations compile in parallel).
#if defined(QSG_BATCH_LEAN) && QSG_BATCH_LEAN == 2
#define QSG_BATCH_ENTRY(KIND, ID) batch_layout_lean1_##KIND##_##ID
#elif defined(QSG_BATCH_LEAN)
#define QSG_BATCH_ENTRY(KIND, ID) batch_layout_lean_##KIND##_##ID
#else
#define QSG_BATCH_ENTRY(KIND, ID) batch_layout_##KIND##_##ID
#endif
#define QSG_BATCH_LAYOUT(ID, BS, GM)                                                                 \
  namespace qsg {                                                                                    \
  int QSG_BATCH_ENTRY(occ, ID)() { return layout_occ<BS, GM>(); }                                    \
  int QSG_BATCH_ENTRY(clusters, ID)(int cs) { return layout_clusters<BS, GM>(cs); }                  \
  cudaError_t QSG_BATCH_ENTRY(launch, ID)(const BatchProblem& P, int grid, int cs, cudaStream_t s) { \
    return layout_launch<BS, GM>(P, grid, cs, s);                                                    \
  }                                                                                                  \
  }
