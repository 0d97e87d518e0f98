// Shared device-side building blocks of the sm_100a time-evolution engines.
//
// Layout in HBM:
//   operator store: CSR, int32 rowptr/col, complex128 values as double2 (16 B, 128-bit loads),
//                   read with ld.global.nc.L1::no_allocate (streamed, never re-read in a pass);
//   state vectors:  complex128 double2 arrays, one per DP5 register (y, y_old, k1..k7, two
//                   stage-input buffers); every pass touches them coalesced, 32 rows per warp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qsg {

constexpr int kMaxTerms = 8;

// Operator store: SELL-32 ("sliced ELLPACK", slice height 32 = one warp). Slice s holds rows
// [32s, 32s+32); its entries are stored column-major inside the slice, so entry k of the 32 rows
// is 32 consecutive (col, val) pairs — one fully coalesced 512 B value load per warp. Each row
// keeps its true length; loads past it are predicated off, so padding costs no HBM bytes.
struct DevSell {
  const long long* slice_off;  // n_slices + 1, in units of 32-entry columns
  const int* rowlen;           // n_slices * 32 (0 for rows past n)
  const int* col;              // 32 * slice_off[n_slices] (plain store)
  const double2* val;
  int n_rows;
  int n_cols;
  long long nnz;
  // Dictionary-coded store (code_bytes 1 or 2): entry = code into (diagonal offset, value) pairs;
  // column = row + dict_off[code], value = dict_val[code]. Lossless: every distinct pair of the
  // operator is in the dictionary. code_bytes 0 = plain (col, val) store.
  int code_bytes;
  const long long* code_off;  // n_slices + 1, in entries: slice s holds 32 rows x Wp codes, row-contiguous
  const unsigned char* code8;
  const unsigned short* code16;
  const int* dict_off;
  const double2* dict_val;
  int dict_n;  // dictionary entries (0 when plain)
  // plain store small enough that each SM's share of it stays in L1 across passes: its (col, val)
  // entries are loaded through the L1-allocating read-only path instead of L1::no_allocate
  int l1;
  // Key-aligned store (ka_nval 0 = absent). Slice s is one block of 32-bit words at
  // ka_blk + 16 * ka_off[s] bytes. A position is a key: it holds, for every lane (row) in its lane
  // mask, the entry in column row ^ key. Layout: header {G, NN, Pu, Npart}; G group words (value id
  // | count << 16, ascending value id); Pu key words of the uniform positions in group order (bit
  // 31: the lane mask is partial); Npart partial masks in the same order; NN non-uniform positions
  // as {key, mask, 32 uint16 value ids}. Values come from the ka_val table of distinct values.
  const unsigned* ka_off;
  const uint4* ka_blk;
  const double2* ka_val;
  int ka_nval;
  int ka_slot;  // largest block in bytes (ring slot size)
};

constexpr unsigned kKaHdrWords = 4, kKaNonUniWords = 18;
constexpr unsigned kKaNonUniform = 0xffffffffu;

struct DevCoeff {
  int kind;  // qsg_coeff_kind
  int i, j;
  double re, im;
};

struct DevGen {
  int n_terms;
  DevSell A[kMaxTerms];
  DevCoeff c[kMaxTerms];
};

// Dormand-Prince 5(4) tableau, error and dense-output weights, PI controller constants
// (integrator.hpp:28-50). Values are the same double-precision literals.
namespace dp {
constexpr double c2 = 1.0 / 5.0, c3 = 3.0 / 10.0, c4 = 4.0 / 5.0, c5 = 8.0 / 9.0;
constexpr double a21 = 1.0 / 5.0;
constexpr double a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
constexpr double a41 = 44.0 / 45.0, a42 = -56.0 / 15.0, a43 = 32.0 / 9.0;
constexpr double a51 = 19372.0 / 6561.0, a52 = -25360.0 / 2187.0, a53 = 64448.0 / 6561.0,
                 a54 = -212.0 / 729.0;
constexpr double a61 = 9017.0 / 3168.0, a62 = -355.0 / 33.0, a63 = 46732.0 / 5247.0,
                 a64 = 49.0 / 176.0, a65 = -5103.0 / 18656.0;
constexpr double a71 = 35.0 / 384.0, a73 = 500.0 / 1113.0, a74 = 125.0 / 192.0,
                 a75 = -2187.0 / 6784.0, a76 = 11.0 / 84.0;
constexpr double e1 = 71.0 / 57600.0, e3 = -71.0 / 16695.0, e4 = 71.0 / 1920.0,
                 e5 = -17253.0 / 339200.0, e6 = 22.0 / 525.0, e7 = -1.0 / 40.0;
constexpr double d1 = -12715105075.0 / 11282082432.0, d3 = 87487479700.0 / 32700410799.0,
                 d4 = -10690763975.0 / 1880347072.0, d5 = 701980252875.0 / 199316789632.0,
                 d6 = -1453857185.0 / 822651844.0, d7 = 69997945.0 / 29380423.0;
constexpr double beta = 0.04, expo1 = 0.2 - beta * 0.75, safe = 0.9;
constexpr double facc1 = 5.0, facc2 = 0.1;
}  // namespace dp

// failure codes written by the device (mapped to reference messages on the host)
enum DevStatus : int {
  kRunning = 0,
  kDone = 1,
  kFailUnderflow = 2,   // integrator.hpp:84-86
  kFailRejected = 3,    // integrator.hpp:87-89
  kFailMaxSteps = 4,    // evolve.cpp:157-159, trajectories.cpp:147-149
  kFailPastEnd = 5,     // integrator.hpp:83
  kFailJumpWeights = 6, // trajectories.cpp:187-188
  kFailJumpCapacity = 7 // device jump record buffer full (host re-runs with more room)
};

// ---- complex helpers (component order identical to std::complex / Eigen) ----------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// acc += v * x with the product fused into two FMA chains.
__device__ __forceinline__ void cfma(double2 v, double2 x, double2& acc) {
  acc.x = fma(v.x, x.x, acc.x);
  acc.x = fma(-v.y, x.y, acc.x);
  acc.y = fma(v.x, x.y, acc.y);
  acc.y = fma(v.y, x.x, acc.y);
}
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }  // std::abs(complex)
__device__ __forceinline__ double cnorm(double2 a) { return a.x * a.x + a.y * a.y; }

__device__ __forceinline__ double2 coeff_eval(const DevCoeff& c, const double* params, double t) {
  switch (c.kind) {
    case 1: return make_double2(params[c.i], 0.0);
    case 2: return make_double2(params[c.i] * cos(params[c.j] * t), 0.0);
    case 3: return make_double2(params[c.i] * sin(params[c.j] * t), 0.0);
    default: return make_double2(c.re, c.im);
  }
}

// ---- streamed operator loads ----------------------------------------------------------------
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ uint2 ld_stream_u2(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// One row of a SELL-32 operator times a gathered vector (lane-per-row). XF maps col -> x[col].
// Entries are consumed in ascending column order, as Eigen's CSC product accumulates a row.
// Register-resident view of a coded store's streams (kernel-parameter fields would otherwise be
// re-read from the constant bank at every entry).
struct CodedView {
  const unsigned char* __restrict__ code8;
  const unsigned short* __restrict__ code16;
  const double2* __restrict__ dval;
  const int* __restrict__ doff;
  int cbytes;
};
__device__ __forceinline__ CodedView coded_view(const DevSell& A) {
  CodedView v{A.code8, A.code16, A.dict_val, A.dict_off, A.code_bytes};
  __builtin_assume(__isGlobal(v.dval));
  __builtin_assume(__isGlobal(v.doff));
  return v;
}

// Coded row with the dictionary staged in shared memory (sval / soff point into __shared__).
// CB: code bytes fixed at compile time (1 or 2; 0 reads A.cbytes), so the unrolled loop carries
// no per-entry code-width test
template <int CB = 0, class XF>
__device__ __forceinline__ double2 sell_row_coded_smem(const CodedView& A, const double2* sval, const int* soff,
                                                       int row, int len, long long base, XF&& xf) {
  const int cbytes = CB ? CB : A.cbytes;
  __builtin_assume(__isShared(sval));
  __builtin_assume(__isShared(soff));
  double2 acc = make_double2(0.0, 0.0);
  for (int j0 = 0; j0 < len; j0 += 32) {
    uint4 w[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + 8 * c;
      if (j < len) {
        if (cbytes == 1) {
          const uint2 v = ld_stream_u2(reinterpret_cast<const uint2*>(A.code8 + base + 32LL * j));
          w[c] = make_uint4(v.x, v.y, 0u, 0u);
        } else {
          w[c] = ld_stream_u4(reinterpret_cast<const uint4*>(A.code16 + base + 32LL * j));
        }
      } else {
        w[c] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // entries of this group present in the row, compared with the unrolled index (one ISETP per
      // entry, no per-entry add: TFIM-10 solve 23.08 -> 22.51 ms)
      const int rem = len - (j0 + 8 * c);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < rem) {
          unsigned k;
          if (cbytes == 1) k = ((u < 4 ? w[c].x : w[c].y) >> (8 * (u & 3))) & 0xffu;
          else k = ((u < 2 ? w[c].x : u < 4 ? w[c].y : u < 6 ? w[c].z : w[c].w) >> (16 * (u & 1))) & 0xffffu;
          cfma(sval[k], xf(row + soff[k]), acc);
        }
      }
    }
  }
  return acc;
}

// Coded row through a CodedView: `len` entries whose codes start at offset `base`.
template <class XF>
__device__ __forceinline__ double2 sell_row_coded_v(const CodedView& A, int row, int len, long long base, XF&& xf) {
  double2 acc = make_double2(0.0, 0.0);
  for (int j0 = 0; j0 < len; j0 += 32) {
    uint4 w[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + 8 * c;
      if (j < len) {
        if (A.cbytes == 1) {
          const uint2 v = ld_stream_u2(reinterpret_cast<const uint2*>(A.code8 + base + 32LL * j));
          w[c] = make_uint4(v.x, v.y, 0u, 0u);
        } else {
          w[c] = ld_stream_u4(reinterpret_cast<const uint4*>(A.code16 + base + 32LL * j));
        }
      } else {
        w[c] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 8 * c + u;
        if (j < len) {
          unsigned k;
          if (A.cbytes == 1) k = ((u < 4 ? w[c].x : w[c].y) >> (8 * (u & 3))) & 0xffu;
          else k = ((u < 2 ? w[c].x : u < 4 ? w[c].y : u < 6 ? w[c].z : w[c].w) >> (16 * (u & 1))) & 0xffffu;
          cfma(__ldg(A.dval + k), xf(row + __ldg(A.doff + k)), acc);
        }
      }
  }
  return acc;
}

// Coded-store row with its metadata already loaded: `len` entries whose first group of 8 codes
// starts at entry `base` = code_off[slice] + 8 * lane. Codes are interleaved in groups of 8 entries
// (group g of the slice's 32 rows is one contiguous 256-entry run), so 8 codes come in one 8 B
// (uint8) or 16 B (uint16) load, a warp's load is one contiguous 256 / 512 B request, and a
// 32-entry row is in flight after 4 loads.
template <class XF>
__device__ __forceinline__ double2 sell_row_coded(const DevSell& A, int row, int len, long long base, XF&& xf) {
  double2 acc = make_double2(0.0, 0.0);
  for (int j0 = 0; j0 < len; j0 += 32) {
    uint4 w[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + 8 * c;
      if (j < len) {
        if (A.code_bytes == 1) {
          const uint2 v = ld_stream_u2(reinterpret_cast<const uint2*>(A.code8 + base + 32LL * j));
          w[c] = make_uint4(v.x, v.y, 0u, 0u);
        } else {
          w[c] = ld_stream_u4(reinterpret_cast<const uint4*>(A.code16 + base + 32LL * j));
        }
      } else {
        w[c] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 8 * c + u;
        if (j < len) {
          unsigned k;
          if (A.code_bytes == 1) k = ((u < 4 ? w[c].x : w[c].y) >> (8 * (u & 3))) & 0xffu;
          else k = ((u < 2 ? w[c].x : u < 4 ? w[c].y : u < 6 ? w[c].z : w[c].w) >> (16 * (u & 1))) & 0xffffu;
          cfma(__ldg(A.dict_val + k), xf(row + __ldg(A.dict_off + k)), acc);
        }
      }
  }
  return acc;
}

// plain-store row: L1 = entries through the L1-allocating read-only path (DevSell::l1)
template <bool L1, class XF>
__device__ __forceinline__ double2 sell_row_plain(const DevSell& A, int len, long long base, XF&& xf) {
  double2 acc = make_double2(0.0, 0.0);
  for (int j = 0; j < len; j += 8) {
    int c[8];
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j + u < len) {
        c[u] = L1 ? __ldg(A.col + base + 32LL * (j + u)) : ld_stream(A.col + base + 32LL * (j + u));
        v[u] = L1 ? __ldg(A.val + base + 32LL * (j + u)) : ld_stream(A.val + base + 32LL * (j + u));
      } else {
        c[u] = 0;
        v[u] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j + u < len) cfma(v[u], xf(c[u]), acc);
  }
  return acc;
}

template <class XF>
__device__ __forceinline__ double2 sell_row(const DevSell& A, int slice, int lane, XF&& xf) {
  const int len = __ldg(A.rowlen + slice * 32 + lane);
  const long long base = __ldg(A.slice_off + slice) * 32 + lane;
  const int row = slice * 32 + lane;
  if (A.code_bytes != 0) return sell_row_coded(A, row, len, __ldg(A.code_off + slice) + 8LL * lane, xf);
  return A.l1 ? sell_row_plain<true>(A, len, base, xf) : sell_row_plain<false>(A, len, base, xf);
}

// Row `slice*32 + lane` of G(t) x with the reference term order: out = A0 x; out += c_k (A_k x)
// (evolve.cpp:63-69). Rows past n return 0.
template <class XF>
__device__ __forceinline__ double2 gen_row(const DevGen& g, const double* params, int slice, double t,
                                           XF&& xf) {
  const int lane = threadIdx.x & 31;
  double2 s = sell_row(g.A[0], slice, lane, xf);
  for (int k = 1; k < g.n_terms; ++k) {
    const double2 sk = sell_row(g.A[k], slice, lane, xf);
    s = cadd(s, cmul(coeff_eval(g.c[k], params, t), sk));
  }
  return s;
}

// Coherent global load that does not allocate in L1 (streamed operands written by earlier passes
// of the same kernel; keeps L1 for the x-gathers).
__device__ __forceinline__ double2 ld_na_c2(const double2* p) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// ---- bulk asynchronous copies (TMA engine, cp.async.bulk) completing on an mbarrier ------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// One elected thread: expect `bytes` on `bar`, then copy them global -> shared through the async
// proxy; the copy's completion flips the barrier's phase. dst, src and bytes are 16-byte multiples.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// generic-proxy reads of a buffer before the async proxy overwrites it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- block reduction (deterministic order) ----------------------------------------------------
// Returns the block total on every thread. smem needs blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < nw ? smem[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) smem[0] = r;
  }
  __syncthreads();
  r = smem[0];
  return r;
}

// ---- grid barrier for a cooperative launch ------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// All CTAs of the grid participate. `bar` holds 8 bytes, 8-byte aligned, zeroed before the launch.
#ifdef QSG_BAR_TIMING  // development build: total ns CTAs spend waiting in grid barriers
static __device__ unsigned long long g_bar_wait_ns, g_bar_calls, g_bar_cta_ns[1024];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

__device__ __forceinline__ void grid_barrier(unsigned* bar, int G) {
  __syncthreads();
#ifdef QSG_BAR_TIMING
  const unsigned long long t_in = threadIdx.x == 0 ? gtimer() : 0ull;
#endif
#ifdef QSG_BAR_V1
  if (G > 1 && threadIdx.x == 0) {
    const unsigned gen = ld_acquire_gpu(bar + 1);
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == static_cast<unsigned>(G - 1)) {
      atomicExch(bar, 0u);
      __threadfence();
      st_release_gpu(bar + 1, gen + 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
#else
  // One monotone 64-bit arrival counter (bar[0..1], zeroed before the launch): barrier k is open
  // once the counter reaches (k+1)*G. A CTA's own arrival returns a value in [k*G, (k+1)*G), which
  // names k, so no generation word, reset or release store is needed: the last arrival's atomic is
  // the only write between the arrivals and the waiters' next poll.
  if (G > 1 && threadIdx.x == 0) {
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(bar);
    __threadfence();
    const unsigned long long old = atomicAdd(cnt, 1ull);
    const unsigned long long target = (old / static_cast<unsigned long long>(G) + 1) * static_cast<unsigned long long>(G);
    while (ld_acquire_gpu_u64(cnt) < target) {
    }
  }
#endif
#ifdef QSG_BAR_TIMING
  if (threadIdx.x == 0) {
    const unsigned long long dt = gtimer() - t_in;
    atomicAdd(&g_bar_wait_ns, dt);
    atomicAdd(&g_bar_calls, 1ull);
    if (blockIdx.x < 1024) g_bar_cta_ns[blockIdx.x] += dt;
  }
#endif
  __syncthreads();
}

}  // namespace qsg
