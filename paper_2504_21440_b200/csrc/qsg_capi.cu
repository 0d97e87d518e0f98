// C-ABI implementation: context, HBM operator store, generator apply, deterministic solvers.
// Reference seams replaced are cited per entry point in include/qsg.h.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "grid_engine.h"
#include "qsg_internal.h"

namespace qsg {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

qsg_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? QSG_OUT_OF_MEMORY : QSG_CUDA_ERROR;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaError_t upload(DevBuf& b, const void* src, size_t bytes, cudaStream_t s) {
  cudaError_t e = b.alloc(bytes, s);
  if (e != cudaSuccess || bytes == 0) return e;
  return cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyDefault, s);
}

DevSell sell_view(const qsg_op* op, bool use_codes) {
  DevSell v{};
  v.slice_off = op->slice_off;
  v.rowlen = op->rowlen;
  v.col = op->col;
  v.val = op->val;
  v.n_rows = static_cast<int>(op->n_rows);
  v.n_cols = static_cast<int>(op->n_cols);
  v.nnz = op->nnz;
  v.code_bytes = (use_codes || op->col == nullptr) ? op->code_bytes : 0;  // coded-only ops decode
  v.code_off = op->code_off;
  v.code8 = op->code_bytes == 1 ? static_cast<const unsigned char*>(op->code) : nullptr;
  v.code16 = op->code_bytes == 2 ? static_cast<const unsigned short*>(op->code) : nullptr;
  v.dict_off = op->dict_off;
  v.dict_val = op->dict_val;
  v.dict_n = op->dict_n;
  // L1-cached plain entries while the whole plain store is at most QSG_L1OP_MAX_BYTES (default
  // 64 MB; Kerr N=400, 19 MB: 316 -> 251 ms per solve; the 493 MB TFIM-10 plain store streams
  // from HBM and is faster with L1::no_allocate, 55.3 vs 61.4 ms, profiles/r01_l1op_ab.log)
  const char* l1e = std::getenv("QSG_L1OP_MAX_BYTES");
  const long long l1_max = l1e ? std::atoll(l1e) : (64LL << 20);
  v.l1 = v.code_bytes == 0 && 20 * op->nnz <= l1_max;
  v.ka_off = op->ka_off;
  v.ka_blk = op->ka_blk;
  v.ka_val = op->ka_val;
  v.ka_nval = op->ka_nval;  // each engine decides whether to read it (grid: st 2; batch: QSG_BATCH_KA)
  v.ka_slot = op->ka_slot;
  return v;
}

DevGen make_devgen(const qsg_generator* g, bool use_codes) {
  DevGen d{};
  d.n_terms = g->n_terms;
  for (int k = 0; k < g->n_terms; ++k) {
    d.A[k] = sell_view(g->ops[k], use_codes);
    if (k > 0 && g->coeffs) {
      const qsg_coeff& c = g->coeffs[k];
      d.c[k] = DevCoeff{c.kind, c.i, c.j, c.re, c.im};
    } else {
      d.c[k] = DevCoeff{0, 0, 0, 1.0, 0.0};
    }
  }
  return d;
}

qsg_status check_generator(const qsg_generator* g, long long n) {
  if (!g || g->n_terms < 1 || g->n_terms > kMaxTerms || !g->ops) {
    set_error("InvalidGrid: generator needs 1..8 terms");
    return QSG_INVALID_GRID;
  }
  for (int k = 0; k < g->n_terms; ++k) {
    const qsg_op* op = g->ops[k];
    if (!op || op->n_rows != n || op->n_cols != n) {
      set_error("DimsMismatch: generator term shape does not match the state");
      return QSG_DIMS_MISMATCH;
    }
    if (k > 0 && g->coeffs && (g->coeffs[k].kind < 0 || g->coeffs[k].kind > 3)) {
      set_error("InvalidGrid: unknown coefficient kind");
      return QSG_INVALID_GRID;
    }
  }
  return QSG_OK;
}

qsg_status check_tlist(const double* tlist, long long n_t) {  // evolve.cpp:71-75
  if (n_t < 2) {
    set_error("InvalidGrid: tlist needs at least two points");
    return QSG_INVALID_GRID;
  }
  for (long long i = 1; i < n_t; ++i)
    if (!(tlist[i] > tlist[i - 1])) {
      set_error("InvalidGrid: tlist must increase strictly");
      return QSG_INVALID_GRID;
    }
  return QSG_OK;
}

qsg_status build_events(const double* tlist, long long n_t, const qsg_solve_opts* o,
                        bool keep_states, Events& ev) {
  // evolve.cpp:89-118 with the saveat defaulting of :265-272
  struct E {
    double t;
    int grid;
    bool save;
  };
  std::vector<E> v;
  for (long long i = 0; i < n_t; ++i) v.push_back({tlist[i], static_cast<int>(i), false});
  std::vector<double> sv;
  if (o && o->n_saveat > 0) sv.assign(o->saveat, o->saveat + o->n_saveat);
  else if (keep_states) sv.assign(tlist, tlist + n_t);
  if (!sv.empty()) {
    if (!std::is_sorted(sv.begin(), sv.end())) {
      set_error("InvalidGrid: saveat must be sorted");
      return QSG_INVALID_GRID;
    }
    for (double t : sv) {
      if (!(t >= tlist[0] && t <= tlist[n_t - 1])) {
        set_error("InvalidGrid: saveat times must lie within [t0, tf]");
        return QSG_INVALID_GRID;
      }
      v.push_back({t, -1, true});
    }
    std::stable_sort(v.begin(), v.end(), [](const E& a, const E& b) { return a.t < b.t; });
    std::vector<E> merged;
    for (const auto& e : v) {
      if (!merged.empty() && merged.back().t == e.t) {
        if (e.grid >= 0) merged.back().grid = e.grid;
        merged.back().save |= e.save;
      } else {
        merged.push_back(e);
      }
    }
    v.swap(merged);
  }
  ev = Events{};
  for (const auto& e : v) {
    ev.t.push_back(e.t);
    ev.grid.push_back(e.grid);
    ev.save.push_back(e.save ? ev.n_save++ : -1);
  }
  return QSG_OK;
}

static std::string fmt_t(double t) { return std::to_string(t); }  // std::to_string as reference

qsg_status status_from_device(int st, double t) {
  switch (st) {
    case kDone: return QSG_OK;
    case kFailUnderflow: set_error("IntegrationFailure: step size underflow at t = " + fmt_t(t)); break;
    case kFailRejected: set_error("IntegrationFailure: step repeatedly rejected at t = " + fmt_t(t)); break;
    case kFailMaxSteps: set_error("IntegrationFailure: max step count exceeded at t = " + fmt_t(t)); break;
    case kFailPastEnd: set_error("IntegrationFailure: step called past t_end"); break;
    case kFailJumpWeights: set_error("IntegrationFailure: vanishing jump weights at the crossing time"); break;
    default: set_error("IntegrationFailure: solver did not finish"); break;
  }
  return QSG_INTEGRATION_FAILURE;
}

// ---- standalone generator apply (SparseGenerator::apply, evolve.cpp:63-69) ------------------
__global__ void __launch_bounds__(256) gen_apply_kernel(DevGen g, const double* params, int n, double t,
                                                        const double2* __restrict__ y,
                                                        double2* __restrict__ out) {
  const int W = blockDim.x >> 5;
  const int nsl = (n + 31) >> 5;
  for (int sl = blockIdx.x * W + (threadIdx.x >> 5); sl < nsl; sl += gridDim.x * W) {
    const int row = (sl << 5) + (threadIdx.x & 31);
    double2 k = gen_row(g, params, sl, t, [&](int c) { return y[c]; });
    if (row < n) out[row] = k;
  }
}

// Single-term coded generator: the dictionary staged in shared memory and the slice loop
// instantiated per code width, as in the grid engine's stage passes (K-spmv).
template <int CB>
__global__ void __launch_bounds__(256) gen_apply_coded_kernel(const DevSell A, int n, const double2* __restrict__ y,
                                                              double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  double2* sv = reinterpret_cast<double2*>(s_dyn);
  int* so = reinterpret_cast<int*>(sv + A.dict_n);
  for (int i = threadIdx.x; i < A.dict_n; i += blockDim.x) {
    sv[i] = A.dict_val[i];
    so[i] = A.dict_off[i];
  }
  __syncthreads();
  const CodedView cv = coded_view(A);
  const int W = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (n + 31) >> 5;
  for (int sl = blockIdx.x * W + (threadIdx.x >> 5); sl < nsl; sl += gridDim.x * W) {
    const int row = (sl << 5) + lane;
    const int len = __ldg(A.rowlen + row);
    const long long base = __ldg(A.code_off + sl) + 8LL * lane;
    const double2 k = sell_row_coded_smem<CB>(cv, sv, so, row, len, base, [&](int c) { return y[c]; });
    if (row < n) out[row] = k;
  }
}

static cudaError_t launch_apply(const DevGen& dg, const double* params, int n, double t,
                                const double2* y, double2* out, int sms, cudaStream_t s) {
  const int threads = 256;
  const int nsl = (n + 31) / 32;
  const int grid = std::max(1, std::min((nsl + 7) / 8, sms * 8));
  const DevSell& A = dg.A[0];
  if (dg.n_terms == 1 && A.code_bytes > 0 && A.dict_n > 0 && A.dict_n <= 2048) {
    const size_t smem = static_cast<size_t>(A.dict_n) * (sizeof(double2) + sizeof(int));
    if (A.code_bytes == 1) gen_apply_coded_kernel<1><<<grid, threads, smem, s>>>(A, n, y, out);
    else gen_apply_coded_kernel<2><<<grid, threads, smem, s>>>(A, n, y, out);
    return cudaGetLastError();
  }
  gen_apply_kernel<<<grid, threads, 0, s>>>(dg, params, n, t, y, out);
  return cudaGetLastError();
}

// ---- CSR -> SELL-32 conversion on device -----------------------------------------------------
__global__ void sell_widths_kernel(const int* rowptr, int n, int* rowlen, long long* width) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int nsl = (n + 31) >> 5;
  if (r >= nsl * 32) return;
  const int len = r < n ? rowptr[r + 1] - rowptr[r] : 0;
  rowlen[r] = len;
  int m = len;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) width[r >> 5] = m;
}

__global__ void sell_fill_kernel(const int* rowptr, const int* col, const double2* val, int n,
                                 const long long* slice_off, int* scol, double2* sval) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int b = rowptr[r], e = rowptr[r + 1];
  const long long base = slice_off[r >> 5] * 32 + (r & 31);
  for (int k = 0; k < e - b; ++k) {
    scol[base + 32LL * k] = col[b + k];
    sval[base + 32LL * k] = val[b + k];
  }
}

// ---- dictionary of distinct (column - row, value) pairs, built on the device -------------------
// Lock-free open addressing in two launches, with no thread ever waiting on another:
//  claim:  each entry's 64-bit signature claims an empty slot by CAS (or finds it already there);
//          the claiming thread writes the full key into its slot;
//  lookup: after the claim launch has completed, every entry probes again and must find its FULL
//          key (exact bit patterns) under its signature. Two distinct keys sharing a signature
//          leave one of them unfound, which sets `overflow` and keeps the operator plain, so the
//          dictionary is lossless by construction.
// The set of keys is fixed by the operator; which slot (and so which code) a key gets can depend
// on claim order, the decoded operator cannot.
constexpr unsigned kDictSlots = 1u << 17;

__device__ __forceinline__ unsigned long long pair_sig(int off, unsigned long long re, unsigned long long im) {
  unsigned long long h = re * 0x9E3779B97F4A7C15ULL ^ (im + 0x632BE59BD9B4E019ULL) * 0xBF58476D1CE4E5B9ULL ^
                         static_cast<unsigned long long>(static_cast<unsigned>(off)) * 0x94D049BB133111EBULL;
  h ^= h >> 29;
  h *= 0xD6E8FEB86659FD93ULL;
  h ^= h >> 32;
  return h | 1ull;
}

// VALUE_ONLY: key on the value alone (the key-aligned store's table of distinct values)
template <bool VALUE_ONLY = false>
__global__ void dict_claim_kernel(const int* rowptr, const int* col, const double2* val, int n,
                                  unsigned long long* tsig, int* toff, double2* tval, int* overflow) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int p = rowptr[r]; p < rowptr[r + 1]; ++p) {
    const int off = VALUE_ONLY ? 0 : col[p] - static_cast<int>(r);
    const double2 v = val[p];
    const unsigned long long sg =
        pair_sig(off, __double_as_longlong(v.x), __double_as_longlong(v.y));
    unsigned slot = static_cast<unsigned>(sg >> 20) & (kDictSlots - 1);
    bool done = false;
    for (unsigned probe = 0; probe < kDictSlots && !done; ++probe) {
      // read first: with few distinct pairs almost every entry finds its signature in place and
      // needs no atomic; only an empty slot is claimed with CAS (a stale 0 just falls through to it)
      unsigned long long prev = *reinterpret_cast<volatile unsigned long long*>(tsig + slot);
      if (prev == 0ull) {
        prev = atomicCAS(tsig + slot, 0ull, sg);
        if (prev == 0ull) {
          toff[slot] = off;
          tval[slot] = v;
        }
      }
      done = prev == 0ull || prev == sg;
      slot = (slot + 1) & (kDictSlots - 1);
    }
    if (!done) atomicExch(overflow, 1);
  }
}

template <bool VALUE_ONLY = false>
__global__ void dict_lookup_kernel(const int* rowptr, const int* col, const double2* val, int n,
                                   const unsigned long long* tsig, const int* toff, const double2* tval,
                                   unsigned* slot_of, int* overflow) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int p = rowptr[r]; p < rowptr[r + 1]; ++p) {
    const int off = VALUE_ONLY ? 0 : col[p] - static_cast<int>(r);
    const double2 v = val[p];
    const unsigned long long re = __double_as_longlong(v.x), im = __double_as_longlong(v.y);
    const unsigned long long sg = pair_sig(off, re, im);
    unsigned slot = static_cast<unsigned>(sg >> 20) & (kDictSlots - 1);
    bool found = false;
    for (unsigned probe = 0; probe < kDictSlots; ++probe) {
      const unsigned long long t = tsig[slot];
      if (t == 0ull) break;
      if (t == sg) {
        const double2 kv = tval[slot];
        if (toff[slot] == off && static_cast<unsigned long long>(__double_as_longlong(kv.x)) == re &&
            static_cast<unsigned long long>(__double_as_longlong(kv.y)) == im) {
          slot_of[p] = slot;
          found = true;
          break;
        }
      }
      slot = (slot + 1) & (kDictSlots - 1);
    }
    if (!found) atomicExch(overflow, 1);
  }
}

// one block: dense ids in slot order, dictionary arrays, and the number of distinct pairs
__global__ void __launch_bounds__(1024) dict_compact_kernel(const unsigned long long* tsig, const int* toff,
                                                            const double2* tval, unsigned* dense, int* dict_off,
                                                            double2* dict_val, int dict_cap, int* count) {
  __shared__ int part[1024];
  constexpr unsigned per = kDictSlots / 1024;
  const unsigned t = threadIdx.x, lo = t * per;
  int c = 0;
  for (unsigned i = 0; i < per; ++i) c += tsig[lo + i] != 0ull;
  part[t] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan
    const int v = t >= static_cast<unsigned>(o) ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int id = part[t] - c;
  for (unsigned i = 0; i < per; ++i)
    if (tsig[lo + i] != 0ull) {
      dense[lo + i] = static_cast<unsigned>(id);
      if (id < dict_cap) {
        dict_off[id] = toff[lo + i];
        dict_val[id] = tval[lo + i];
      }
      ++id;
    }
  if (t == 1023) *count = part[1023];
}

template <class T>
__global__ void sell_code_fill_dense_kernel(const int* rowptr, const unsigned* slot_of, const unsigned* dense, int n,
                                            const long long* code_off, T* scode) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int b = rowptr[r], e = rowptr[r + 1];
  // interleaved groups of 8 entries: entry k of lane l at code_off[slice] + (k/8)*256 + 8*l + k%8, so
  // a warp's 8-code loads of one group are one contiguous 256-entry run
  const long long base = code_off[r >> 5] + (r & 31) * 8;
  for (int k = 0; k < e - b; ++k) scode[base + (k >> 3) * 256 + (k & 7)] = static_cast<T>(dense[slot_of[b + k]]);
}

// Slice-aligned entry order (coded and plain SELL fills): one warp per 32-row slice. Within each
// row the entries are reordered by (how many rows of the slice hold an entry at the same distance
// |col - row| (descending), that distance, the signed offset), so the rows of a slice put their
// common entries at the same SELL position. A warp's dictionary lookups at one position then touch
// one or two words (a broadcast or a +/- offset pair) instead of up to 32, and its gathers hit one
// contiguous segment. TFIM-10 Liouvillian: 4.70 -> 1.71 distinct codes per (slice, position), 34% ->
// 93% with at most two (scripts/coded_align_stats.py). The row's sum runs in the new order. Slices
// whose rows exceed kAlignMaxRow entries or whose distance set overflows the per-warp table keep
// the CSR order. QSG_SELL_ALIGN=0 keeps the CSR order in the coded store too.
constexpr int kAlignMaxRow = 64;
constexpr int kAlignTab = 256;  // distinct distances per slice (open addressing, per warp)
constexpr int kAlignWarps = 4;

bool sell_align_enabled() {
  const char* al = std::getenv("QSG_SELL_ALIGN");
  return !(al && al[0] == '0');
}
// The plain store keeps the CSR (reference) order unless QSG_PLAIN_ALIGN=1: aligned plain rows
// measured sweep 98.5 -> 95.3 ms, TFIM-14 mcsolve unchanged, K-cluster Kerr-50 9.47 -> 9.54 us per
// attempt (profiles/r02_sell_align.log), not enough to give up the reference summation order.
bool plain_align_enabled() {
  const char* al = std::getenv("QSG_PLAIN_ALIGN");
  return al && al[0] == '1' && sell_align_enabled();
}

// Fills pm[0..len) with the lane's row order (indices into the row's CSR entries); false: keep
// the CSR order for this slice. Every lane of the warp must call it.
__device__ bool slice_aligned_order(const int* __restrict__ col, int r, int b, int len, bool live,
                                    int (*s_key)[kAlignTab], int (*s_cnt)[kAlignTab], int* s_bad,
                                    unsigned char* pm) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < kAlignTab; i += 32) {
    s_key[w][i] = -1;
    s_cnt[w][i] = 0;
  }
  if (lane == 0) s_bad[w] = 0;
  __syncwarp();
  int maxlen = len;
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  if (maxlen > kAlignMaxRow) s_bad[w] = 1;
  auto slot_of_dist = [&](int a, bool insert) {
    unsigned h = (static_cast<unsigned>(a) * 0x9E3779B1u) >> 24;  // kAlignTab = 256
    for (int probe = 0; probe < kAlignTab; ++probe, h = (h + 1) & (kAlignTab - 1)) {
      const int k = insert ? atomicCAS(&s_key[w][h], -1, a) : s_key[w][h];
      if (k == a || (insert && k == -1)) return static_cast<int>(h);
      if (!insert && k == -1) return -1;
    }
    return -1;
  };
  __syncwarp();
  if (!s_bad[w])
    for (int k = 0; k < len; ++k) {
      const int h = slot_of_dist(abs(col[b + k] - r), true);
      if (h < 0) s_bad[w] = 1;
      else atomicAdd(&s_cnt[w][h], 1);
    }
  __syncwarp();
  if (!live || s_bad[w]) return false;
  int fq[kAlignMaxRow], ds[kAlignMaxRow], of[kAlignMaxRow];
  for (int k = 0; k < len; ++k) {
    const int o = col[b + k] - r;
    ds[k] = abs(o);
    fq[k] = s_cnt[w][slot_of_dist(ds[k], false)];
    of[k] = o;
    pm[k] = static_cast<unsigned char>(k);
  }
  auto before = [&](int x, int y) {  // entry x sorts before entry y
    if (fq[x] != fq[y]) return fq[x] > fq[y];
    if (ds[x] != ds[y]) return ds[x] < ds[y];
    return of[x] < of[y];
  };
  for (int i = 1; i < len; ++i) {  // insertion sort (stable)
    const unsigned char v = pm[i];
    int j = i - 1;
    while (j >= 0 && before(v, pm[j])) {
      pm[j + 1] = pm[j];
      --j;
    }
    pm[j + 1] = v;
  }
  return true;
}

template <class T>
__global__ void __launch_bounds__(32 * kAlignWarps) sell_code_fill_aligned_kernel(
    const int* __restrict__ rowptr, const int* __restrict__ col, const unsigned* __restrict__ slot_of,
    const unsigned* __restrict__ dense, int n, const long long* __restrict__ code_off, T* scode) {
  __shared__ int s_key[kAlignWarps][kAlignTab];
  __shared__ int s_cnt[kAlignWarps][kAlignTab];
  __shared__ int s_bad[kAlignWarps];
  const long long r = (static_cast<long long>(blockIdx.x) * kAlignWarps + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31);
  const bool live = r < n;
  const int b = live ? rowptr[r] : 0, len = live ? rowptr[r + 1] - b : 0;
  unsigned char pm[kAlignMaxRow];
  const bool sorted = slice_aligned_order(col, static_cast<int>(r), b, len, live, s_key, s_cnt, s_bad, pm);
  if (!live) return;
  const long long base = code_off[r >> 5] + (r & 31) * 8;
  for (int k = 0; k < len; ++k)
    scode[base + (k >> 3) * 256 + (k & 7)] = static_cast<T>(dense[slot_of[b + (sorted ? pm[k] : k)]]);
}

__global__ void __launch_bounds__(32 * kAlignWarps) sell_fill_aligned_kernel(
    const int* __restrict__ rowptr, const int* __restrict__ col, const double2* __restrict__ val, int n,
    const long long* __restrict__ slice_off, int* scol, double2* sval) {
  __shared__ int s_key[kAlignWarps][kAlignTab];
  __shared__ int s_cnt[kAlignWarps][kAlignTab];
  __shared__ int s_bad[kAlignWarps];
  const long long r = (static_cast<long long>(blockIdx.x) * kAlignWarps + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31);
  const bool live = r < n;
  const int b = live ? rowptr[r] : 0, len = live ? rowptr[r + 1] - b : 0;
  unsigned char pm[kAlignMaxRow];
  const bool sorted = slice_aligned_order(col, static_cast<int>(r), b, len, live, s_key, s_cnt, s_bad, pm);
  if (!live) return;
  const long long base = slice_off[r >> 5] * 32 + (r & 31);
  for (int k = 0; k < len; ++k) {
    const int e = b + (sorted ? pm[k] : k);
    scol[base + 32LL * k] = col[e];
    sval[base + 32LL * k] = val[e];
  }
}

// Builds the coded store of `op` from the staged CSR; leaves op plain when the operator has more
// than 65535 distinct pairs. Returns a CUDA error only for real failures.
static cudaError_t build_coded_store(qsg_op* op, const int* rp, const int* col, const double2* val, long long n,
                                     const std::vector<long long>& w, cudaStream_t s) {
  const long long nsl = static_cast<long long>(w.size());
  cudaError_t e;
  DevBuf tsig, toff, tval, slot_of, dense, cnt, ovf, doff, dval;
  if ((e = tsig.alloc(sizeof(unsigned long long) * kDictSlots, s)) || (e = toff.alloc(sizeof(int) * kDictSlots, s)) ||
      (e = tval.alloc(sizeof(double2) * kDictSlots, s)) ||
      (e = slot_of.alloc(sizeof(unsigned) * op->nnz, s)) || (e = dense.alloc(sizeof(unsigned) * kDictSlots, s)) ||
      (e = cnt.alloc(sizeof(int), s)) || (e = ovf.alloc(sizeof(int), s)) ||
      (e = doff.alloc(sizeof(int) * 65536, s)) || (e = dval.alloc(sizeof(double2) * 65536, s)))
    return e;
  cudaMemsetAsync(tsig.p, 0, sizeof(unsigned long long) * kDictSlots, s);
  cudaMemsetAsync(ovf.p, 0, sizeof(int), s);
  const unsigned nb = static_cast<unsigned>((n + 255) / 256);
  dict_claim_kernel<false><<<nb, 256, 0, s>>>(rp, col, val, static_cast<int>(n), tsig.as<unsigned long long>(),
                                       toff.as<int>(), tval.as<double2>(), ovf.as<int>());
  dict_lookup_kernel<false><<<nb, 256, 0, s>>>(rp, col, val, static_cast<int>(n), tsig.as<unsigned long long>(),
                                        toff.as<int>(), tval.as<double2>(), slot_of.as<unsigned>(), ovf.as<int>());
  dict_compact_kernel<<<1, 1024, 0, s>>>(tsig.as<unsigned long long>(), toff.as<int>(), tval.as<double2>(),
                                         dense.as<unsigned>(), doff.as<int>(), dval.as<double2>(), 65536,
                                         cnt.as<int>());
  int count = 0, overflow = 0;
  if ((e = cudaGetLastError()) || (e = cudaMemcpyAsync(&count, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaMemcpyAsync(&overflow, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, s)) || (e = cudaStreamSynchronize(s)))
    return e;
  if (overflow || count < 1 || count > 65535) return cudaSuccess;  // stays plain
  const int cbytes = count <= 256 ? 1 : 2;
  std::vector<long long> coff(nsl + 1, 0);
  for (long long i = 0; i < nsl; ++i) coff[i + 1] = coff[i] + 32 * ((w[i] + 7) / 8 * 8);
  // + 1024 codes of tail padding: the grid engine prefetches a 1 K-code window per slice
  const size_t pc = static_cast<size_t>(std::max<long long>(1, coff[nsl])) + 1024;
  if ((e = cudaMallocAsync(&op->code, pc * cbytes, s)) ||
      (e = cudaMallocAsync(&op->code_off, sizeof(long long) * (nsl + 1), s)) ||
      (e = cudaMallocAsync(&op->dict_off, sizeof(int) * count, s)) ||
      (e = cudaMallocAsync(&op->dict_val, sizeof(double2) * count, s)))
    return e;
  cudaMemsetAsync(op->code, 0, pc * cbytes, s);
  cudaMemcpyAsync(op->code_off, coff.data(), sizeof(long long) * (nsl + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(op->dict_off, doff.p, sizeof(int) * count, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(op->dict_val, dval.p, sizeof(double2) * count, cudaMemcpyDeviceToDevice, s);
  const bool align = sell_align_enabled();
  const unsigned nba = static_cast<unsigned>((nsl + kAlignWarps - 1) / kAlignWarps);
  if (cbytes == 1) {
    if (align)
      sell_code_fill_aligned_kernel<unsigned char><<<nba, 32 * kAlignWarps, 0, s>>>(
          rp, col, slot_of.as<unsigned>(), dense.as<unsigned>(), static_cast<int>(n), op->code_off,
          static_cast<unsigned char*>(op->code));
    else
      sell_code_fill_dense_kernel<unsigned char><<<nb, 256, 0, s>>>(rp, slot_of.as<unsigned>(), dense.as<unsigned>(),
                                                                    static_cast<int>(n), op->code_off,
                                                                    static_cast<unsigned char*>(op->code));
  } else {
    if (align)
      sell_code_fill_aligned_kernel<unsigned short><<<nba, 32 * kAlignWarps, 0, s>>>(
          rp, col, slot_of.as<unsigned>(), dense.as<unsigned>(), static_cast<int>(n), op->code_off,
          static_cast<unsigned short*>(op->code));
    else
      sell_code_fill_dense_kernel<unsigned short><<<nb, 256, 0, s>>>(rp, slot_of.as<unsigned>(), dense.as<unsigned>(),
                                                                     static_cast<int>(n), op->code_off,
                                                                     static_cast<unsigned short*>(op->code));
  }
  if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(s))) return e;
  op->code_bytes = cbytes;
  op->dict_n = count;
  return cudaSuccess;
}


// ---- key-aligned store, built on the device -------------------------------------
// One warp per 32-row slice. Each lane sorts its row's entries by key = col ^ row; the warp then
// merges the 32 sorted lists: position p takes the warp-minimum head key, the lanes holding it set
// their bit in the position's lane mask and advance. A position whose lanes all carry the same
// value (bit-exact) is "uniform": it joins the group of that value. Lane 0 then writes the slice
// block (engine.cuh kKa* layout): header, one word per group (value id | count << 16), the uniform
// positions' key words grouped by ascending value id (keys ascending inside a group; bit 31 set
// when the lane mask is partial), the partial masks in the same order, then each non-uniform
// position as {key, mask, 32 uint16 value ids}. COUNT pass: block sizes (words); FILL pass: blocks.
constexpr int kKaMaxRow = 64;    // longest row the per-lane sort handles
constexpr int kKaMaxPos = 128;   // widest key union per slice
constexpr int kKaMaxNonUni = 8;  // non-uniform positions per slice
constexpr int kKaMaxVals = 2048;
constexpr int kKaWarps = 4;      // warps per build block

template <bool FILL>
__global__ void __launch_bounds__(32 * kKaWarps) ka_slice_kernel(const int* __restrict__ rowptr,
                                                                 const int* __restrict__ col,
                                                                 const unsigned* __restrict__ slot_of,
                                                                 const unsigned* __restrict__ dense, int n, int nsl,
                                                                 unsigned* __restrict__ words_out,
                                                                 const unsigned* __restrict__ off16,
                                                                 unsigned* __restrict__ blk, int* __restrict__ bad) {
  __shared__ unsigned s_key[kKaWarps][kKaMaxPos], s_mask[kKaWarps][kKaMaxPos], s_vid[kKaWarps][kKaMaxPos];
  __shared__ unsigned short s_ex[kKaWarps][kKaMaxNonUni][32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= nsl) return;
  const int r = s * 32 + lane;
  const int b = r < n ? rowptr[r] : 0;
  const int len = r < n ? rowptr[r + 1] - b : 0;
  if (__any_sync(0xffffffffu, len > kKaMaxRow)) {
    if (lane == 0) atomicExch(bad, 1);
    return;
  }
  unsigned key[kKaMaxRow], vid[kKaMaxRow];
  for (int k = 0; k < len; ++k) {  // insertion sort by key
    const unsigned kk = static_cast<unsigned>(col[b + k]) ^ static_cast<unsigned>(r);
    const unsigned vv = dense[slot_of[b + k]];
    int j = k;
    while (j > 0 && key[j - 1] > kk) {
      key[j] = key[j - 1];
      vid[j] = vid[j - 1];
      --j;
    }
    key[j] = kk;
    vid[j] = vv;
  }
  int np = 0, nn = 0, h = 0;
  bool overflow = false;
  for (;;) {
    const unsigned my = h < len ? key[h] : 0xffffffffu;
    const unsigned m = __reduce_min_sync(0xffffffffu, my);
    if (m == 0xffffffffu) break;
    const bool has = my == m;
    const unsigned mask = __ballot_sync(0xffffffffu, has);
    const unsigned v = has ? vid[h] : 0u;
    const unsigned vmin = __reduce_min_sync(0xffffffffu, has ? v : 0xffffffffu);
    const unsigned vmax = __reduce_max_sync(0xffffffffu, has ? v : 0u);
    const bool uni = vmin == vmax;
    if (np < kKaMaxPos && (uni || nn < kKaMaxNonUni)) {
      if (!uni) s_ex[wl][nn][lane] = static_cast<unsigned short>(v);
      if (lane == 0) {
        s_key[wl][np] = m;
        s_mask[wl][np] = mask;
        s_vid[wl][np] = uni ? vmin : kKaNonUniform;
      }
    } else {
      overflow = true;
    }
    ++np;
    nn += uni ? 0 : 1;
    if (has) ++h;
  }
  if (overflow) {
    if (lane == 0) atomicExch(bad, 1);
    return;
  }
  __syncwarp();
  if (lane != 0) return;
  // groups: distinct uniform value ids, ascending
  unsigned gv[kKaMaxPos], gc[kKaMaxPos];
  int G = 0, Pu = 0, npart = 0;
  for (int p = 0; p < np; ++p) {
    const unsigned v = s_vid[wl][p];
    if (v == kKaNonUniform) continue;
    ++Pu;
    npart += s_mask[wl][p] != 0xffffffffu;
    int g = 0;
    while (g < G && gv[g] < v) ++g;
    if (g < G && gv[g] == v) {
      ++gc[g];
    } else {
      for (int q = G; q > g; --q) {
        gv[q] = gv[q - 1];
        gc[q] = gc[q - 1];
      }
      gv[g] = v;
      gc[g] = 1;
      ++G;
    }
  }
  const unsigned words = (kKaHdrWords + G + Pu + npart + kKaNonUniWords * nn + 3u) & ~3u;
  if (!FILL) {
    words_out[s] = words;
    return;
  }
  unsigned* w = blk + 4ull * off16[s];
  w[0] = G;
  w[1] = nn;
  w[2] = Pu;
  w[3] = npart;
  unsigned kp = kKaHdrWords + G, mp = kp + Pu, ep = mp + npart;
  for (int g = 0; g < G; ++g) {
    w[kKaHdrWords + g] = gv[g] | (gc[g] << 16);
    for (int p = 0; p < np; ++p)  // keys ascending inside the group
      if (s_vid[wl][p] == gv[g]) {
        const bool part = s_mask[wl][p] != 0xffffffffu;
        w[kp++] = s_key[wl][p] | (part ? 0x80000000u : 0u);
        if (part) w[mp++] = s_mask[wl][p];
      }
  }
  int e = 0;
  for (int p = 0; p < np; ++p)
    if (s_vid[wl][p] == kKaNonUniform) {
      w[ep] = s_key[wl][p];
      w[ep + 1] = s_mask[wl][p];
      unsigned short* ids = reinterpret_cast<unsigned short*>(w + ep + 2);
      for (int l = 0; l < 32; ++l) ids[l] = s_ex[wl][e][l];
      ep += kKaNonUniWords;
      ++e;
    }
}

// Builds the key-aligned store of `op` from the staged CSR when it pays: at most kKaMaxVals
// distinct values, rows of at most kKaMaxRow entries, at most kKaMaxPos key positions and
// kKaMaxNonUni non-uniform positions per slice, and blocks smaller than the coded store's
// entries. Otherwise op keeps its other stores.
static cudaError_t build_ka_store(qsg_op* op, const int* rp, const int* col, const double2* val, long long n,
                                  cudaStream_t s) {
  const long long nsl = (n + 31) / 32;
  cudaError_t e;
  DevBuf tsig, toff, tval, slot_of, dense, cnt, ovf, doff, dval, dnp, dbad;
  if ((e = tsig.alloc(sizeof(unsigned long long) * kDictSlots, s)) || (e = toff.alloc(sizeof(int) * kDictSlots, s)) ||
      (e = tval.alloc(sizeof(double2) * kDictSlots, s)) || (e = slot_of.alloc(sizeof(unsigned) * op->nnz, s)) ||
      (e = dense.alloc(sizeof(unsigned) * kDictSlots, s)) || (e = cnt.alloc(sizeof(int), s)) ||
      (e = ovf.alloc(sizeof(int), s)) || (e = doff.alloc(sizeof(int) * kKaMaxVals, s)) ||
      (e = dval.alloc(sizeof(double2) * kKaMaxVals, s)) || (e = dnp.alloc(sizeof(unsigned) * nsl, s)) ||
      (e = dbad.alloc(sizeof(int), s)))
    return e;
  cudaMemsetAsync(tsig.p, 0, sizeof(unsigned long long) * kDictSlots, s);
  cudaMemsetAsync(ovf.p, 0, sizeof(int), s);
  cudaMemsetAsync(dbad.p, 0, sizeof(int), s);
  const unsigned nb = static_cast<unsigned>((n + 255) / 256);
  dict_claim_kernel<true><<<nb, 256, 0, s>>>(rp, col, val, static_cast<int>(n), tsig.as<unsigned long long>(),
                                             toff.as<int>(), tval.as<double2>(), ovf.as<int>());
  dict_lookup_kernel<true><<<nb, 256, 0, s>>>(rp, col, val, static_cast<int>(n), tsig.as<unsigned long long>(),
                                              toff.as<int>(), tval.as<double2>(), slot_of.as<unsigned>(), ovf.as<int>());
  dict_compact_kernel<<<1, 1024, 0, s>>>(tsig.as<unsigned long long>(), toff.as<int>(), tval.as<double2>(),
                                         dense.as<unsigned>(), doff.as<int>(), dval.as<double2>(), kKaMaxVals,
                                         cnt.as<int>());
  int count = 0, overflow = 0;
  if ((e = cudaGetLastError()) || (e = cudaMemcpyAsync(&count, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaMemcpyAsync(&overflow, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, s)) || (e = cudaStreamSynchronize(s)))
    return e;
  if (overflow || count < 1 || count > kKaMaxVals) return cudaSuccess;
  const unsigned kb = static_cast<unsigned>((nsl + kKaWarps - 1) / kKaWarps);
  ka_slice_kernel<false><<<kb, 32 * kKaWarps, 0, s>>>(rp, col, slot_of.as<unsigned>(), dense.as<unsigned>(),
                                                      static_cast<int>(n), static_cast<int>(nsl), dnp.as<unsigned>(),
                                                      nullptr, nullptr, dbad.as<int>());
  std::vector<unsigned> nw(static_cast<size_t>(nsl));
  int bad = 0;
  if ((e = cudaGetLastError()) ||
      (e = cudaMemcpyAsync(nw.data(), dnp.p, sizeof(unsigned) * nsl, cudaMemcpyDeviceToHost, s)) ||
      (e = cudaMemcpyAsync(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, s)) || (e = cudaStreamSynchronize(s)))
    return e;
  if (bad) return cudaSuccess;
  std::vector<unsigned> off(static_cast<size_t>(nsl + 1), 0);
  long long words = 0;
  unsigned slot = 0;
  for (long long i = 0; i < nsl; ++i) {
    off[i] = static_cast<unsigned>(words / 4);
    words += nw[i];
    slot = std::max(slot, 4 * nw[i]);
    if (words / 4 > 0xffffffffLL) return cudaSuccess;
  }
  off[nsl] = static_cast<unsigned>(words / 4);
  // positions per slice ~ words; keep the store only when its blocks are well below the coded
  // store (the coded entries cost op->nnz bytes)
  if (4 * words > op->nnz) return cudaSuccess;
  if ((e = cudaMallocAsync(&op->ka_off, sizeof(unsigned) * (nsl + 1), s)) ||
      (e = cudaMallocAsync(&op->ka_blk, 4 * static_cast<size_t>(words), s)) ||
      (e = cudaMallocAsync(&op->ka_val, sizeof(double2) * count, s)))
    return e;
  cudaMemcpyAsync(op->ka_off, off.data(), sizeof(unsigned) * (nsl + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(op->ka_val, dval.p, sizeof(double2) * count, cudaMemcpyDeviceToDevice, s);
  cudaMemsetAsync(op->ka_blk, 0, 4 * static_cast<size_t>(words), s);
  ka_slice_kernel<true><<<kb, 32 * kKaWarps, 0, s>>>(rp, col, slot_of.as<unsigned>(), dense.as<unsigned>(),
                                                     static_cast<int>(n), static_cast<int>(nsl), nullptr, op->ka_off,
                                                     reinterpret_cast<unsigned*>(op->ka_blk), dbad.as<int>());
  if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(s))) return e;
  op->ka_nval = count;
  op->ka_slot = static_cast<int>(slot);
  op->ka_bytes = 4 * words + 4 * (nsl + 1) + 16LL * count;
  op->ka_positions = words;
  return cudaSuccess;
}

// ---- RNG kernel (rng.cpp:14-47) ---------------------------------------------------------------
__device__ __forceinline__ unsigned long long d_splitmix(unsigned long long& s) {
  unsigned long long z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__global__ void rng_kernel(unsigned long long seed, unsigned long long stream, int kind, int n,
                           double* out_d, unsigned long long* out_u) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long z = seed ^ ((stream + 1) * 0x9E3779B97F4A7C15ULL), s[4];
  for (int i = 0; i < 4; ++i) s[i] = d_splitmix(z);
  if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
  auto next = [&]() {
    const unsigned long long r = ((s[0] + s[3]) << 23 | (s[0] + s[3]) >> 41) + s[0];
    const unsigned long long tt = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= tt;
    s[3] = (s[3] << 45) | (s[3] >> 19);
    return r;
  };
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      out_u[i] = next();
    } else {
      double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
      if (kind == 2)
        while (u == 0.0) u = static_cast<double>(next() >> 11) * 0x1.0p-53;
      out_d[i] = u;
    }
  }
}

// ---- shared deterministic-solver driver ----------------------------------------------------------
// The cluster-resident solver (K-cluster) takes every single-term plain-store system of at least
// 8 slices that fits one 16-CTA cluster's shared memory (Kerr N = 20..100: 13.7 / 12.3 / 12.7 /
// 17.9 us per attempt at N = 20 / 50 / 70 / 100 against 14.6 / 19.1 / 22.5 / 21.5 on the grid
// engine; 4 slices (Kerr N = 10): one CTA is faster, 11.9 vs 14.1; profiles/r02_cluster_solve.log)
constexpr long long kClusterSolveMinSlices = 8;
constexpr long long kClusterSolveRows = 1LL << 30;

static qsg_status run_grid_solve(qsg_ctx* ctx, int mode, const qsg_generator* G, long long d,
                                 const double* y0, const double* tlist, long long n_t, int n_e,
                                 const qsg_csr* e_ops, const double* params, int n_params,
                                 const qsg_solve_opts* opts, double* expect, double* states,
                                 qsg_stats* stats, qsg_timing* timing) {
  if (!ctx) {
    set_error("InvalidGrid: null context");
    return QSG_INVALID_GRID;
  }
  if (qsg_status s = check_tlist(tlist, n_t)) return s;
  const long long n = mode == 0 ? d * d : d;
  if (n <= 0 || n > 0x7fffffffLL) {
    set_error("TooLarge: state length must fit int32 indexing");
    return QSG_TOO_LARGE;
  }
  if (qsg_status s = check_generator(G, n)) return s;
  if (opts && opts->method != 0) {
    set_error("InvalidGrid: only the adaptive Dormand-Prince 5(4) method runs on the device");
    return QSG_UNSUPPORTED;
  }
  const double atol = opts ? opts->abstol : 1e-8, rtol = opts ? opts->reltol : 1e-6;
  if (!(atol > 0 && rtol > 0)) {  // integrator.hpp:55
    set_error("InvalidGrid: tolerances must be positive");
    return QSG_INVALID_GRID;
  }
  const bool keep = (opts && opts->store_states) || n_e == 0;
  Events ev;
  if (qsg_status s = build_events(tlist, n_t, opts, keep, ev)) return s;
  for (int e = 0; e < n_e; ++e)
    if (e_ops[e].n_rows != d || e_ops[e].n_cols != d) {
      set_error("DimsMismatch: e_ops dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
  if (2 * n_e > kObsSlots) {
    set_error("TooLarge: at most 64 e_ops per solve");
    return QSG_TOO_LARGE;
  }
  cudaStream_t s = ctx->stream;
  cudaError_t ce;
  // ---- workspace: 11 state vectors
  const size_t vbytes = static_cast<size_t>(n) * sizeof(double2);
  DevBuf work;
  if ((ce = work.alloc(11 * vbytes, s))) return cuda_fail(ce, "workspace");
  GridProblem P{};
  P.n = static_cast<int>(n);
  P.d = static_cast<int>(d);
  for (int i = 0; i < 11; ++i) P.buf[i] = reinterpret_cast<double2*>(work.as<char>() + i * vbytes);
  if ((ce = cudaMemcpyAsync(P.buf[0], y0, vbytes, cudaMemcpyDefault, s))) return cuda_fail(ce, "y0 copy");
  P.gen = make_devgen(G);
  DevBuf dparams;
  if (n_params > 0) {
    if ((ce = upload(dparams, params, sizeof(double) * n_params, s))) return cuda_fail(ce, "params");
    P.params = dparams.as<double>();
  }
  P.atol = atol;
  P.rtol = rtol;
  P.max_steps = opts ? opts->max_steps : 10000000LL;
  P.t0 = tlist[0];
  P.tf = tlist[n_t - 1];
  P.eps_t = 1e-12 * std::max({1.0, std::fabs(P.tf), std::fabs(P.t0)});  // evolve.cpp:128
  DevBuf dev_t, dev_g, dev_s;
  P.n_ev = static_cast<int>(ev.t.size());
  if ((ce = upload(dev_t, ev.t.data(), ev.t.size() * sizeof(double), s))) return cuda_fail(ce, "events");
  if ((ce = upload(dev_g, ev.grid.data(), ev.grid.size() * sizeof(int), s))) return cuda_fail(ce, "events");
  if ((ce = upload(dev_s, ev.save.data(), ev.save.size() * sizeof(int), s))) return cuda_fail(ce, "events");
  P.ev_t = dev_t.as<double>();
  P.ev_grid = dev_g.as<int>();
  P.ev_save = dev_s.as<int>();
  P.n_e = n_e;
  // ---- observation operators
  std::vector<int> eo_off(1, 0), eo_i, eo_j, se_rowptr;
  std::vector<double> eo_v;
  std::vector<long long> se_off;
  std::vector<int> se_col;
  const char* es = std::getenv("QSG_SE_EOP_STORE");
  const bool se_store = mode == 1 && n_e > 0 && n_e <= kGridMaxSeOps && !(es && es[0] == '0');
  for (int e = 0; e < n_e; ++e) {
    const qsg_csr& A = e_ops[e];
    if (mode == 0) {
      for (long long r = 0; r < A.n_rows; ++r)
        for (int p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) {
          eo_i.push_back(static_cast<int>(r));
          eo_j.push_back(A.col[p]);
          eo_v.push_back(A.val[2 * p]);
          eo_v.push_back(A.val[2 * p + 1]);
        }
      eo_off.push_back(static_cast<int>(eo_i.size()));
    } else if (!se_store) {
      se_off.push_back(static_cast<long long>(se_col.size()));
      se_rowptr.insert(se_rowptr.end(), A.rowptr, A.rowptr + A.n_rows + 1);
      se_col.insert(se_col.end(), A.col, A.col + A.nnz);
      eo_v.insert(eo_v.end(), A.val, A.val + 2 * A.nnz);
    }
  }
  // sesolve: e_ops as operator stores (the coded store shrinks e.g. a 20-spin Sx total from 420 MB
  // to ~25 MB per evaluation); QSG_SE_EOP_STORE=0 keeps the CSR path
  struct OpHold {
    std::vector<qsg_op*> v;
    ~OpHold() {
      for (qsg_op* o : v) qsg_op_destroy(o);
    }
  } se_hold;
  P.n_se_ops = 0;
  if (se_store) {
    for (int e = 0; e < n_e; ++e) {
      qsg_op* o = nullptr;
      if (qsg_status st = qsg_op_create(ctx, &e_ops[e], &o)) return st;
      se_hold.v.push_back(o);
      P.se_ops[e] = sell_view(o, true);
    }
    P.n_se_ops = n_e;
  }
  DevBuf d_eoff, d_ei, d_ej, d_ev, d_srp, d_scol, d_soff;
  if (mode == 0) {
    if ((ce = upload(d_eoff, eo_off.data(), eo_off.size() * sizeof(int), s)) ||
        (ce = upload(d_ei, eo_i.data(), eo_i.size() * sizeof(int), s)) ||
        (ce = upload(d_ej, eo_j.data(), eo_j.size() * sizeof(int), s)) ||
        (ce = upload(d_ev, eo_v.data(), eo_v.size() * sizeof(double), s)))
      return cuda_fail(ce, "e_ops");
    P.eo_off = d_eoff.as<int>();
    P.eo_i = d_ei.as<int>();
    P.eo_j = d_ej.as<int>();
    P.eo_v = d_ev.as<double2>();
  } else if (P.n_se_ops == 0) {
    if ((ce = upload(d_srp, se_rowptr.data(), se_rowptr.size() * sizeof(int), s)) ||
        (ce = upload(d_scol, se_col.data(), se_col.size() * sizeof(int), s)) ||
        (ce = upload(d_ev, eo_v.data(), eo_v.size() * sizeof(double), s)) ||
        (ce = upload(d_soff, se_off.data(), se_off.size() * sizeof(long long), s)))
      return cuda_fail(ce, "e_ops");
    P.se_rowptr = d_srp.as<int>();
    P.se_col = d_scol.as<int>();
    P.se_val = d_ev.as<double2>();
    P.se_off = d_soff.as<long long>();
  }
  // ---- outputs and control
  DevBuf d_exp, d_states, d_ctl, d_red, d_bar;
  if ((ce = d_exp.alloc(std::max<size_t>(1, static_cast<size_t>(n_e) * n_t) * sizeof(double2), s)))
    return cuda_fail(ce, "expect");
  cudaMemsetAsync(d_exp.p, 0, std::max<size_t>(1, static_cast<size_t>(n_e) * n_t) * sizeof(double2), s);
  P.expect = d_exp.as<double2>();
  const bool states_dev = states && is_device_ptr(states);
  if (ev.n_save > 0) {
    if (states_dev) {
      P.states = reinterpret_cast<double2*>(states);
    } else {
      if ((ce = d_states.alloc(static_cast<size_t>(ev.n_save) * vbytes, s))) return cuda_fail(ce, "states");
      P.states = d_states.as<double2>();
    }
  }
  const int lanes = 1;
  const int threads = grid_threads();
  bool pf = true;  // prefetching stage variant when every term uses the coded store
  for (int k = 0; k < G->n_terms; ++k) pf = pf && G->ops[k]->code_bytes > 0;
  // Stage a single-term coded generator's dictionary (<= 2048 entries) in shared memory: its lookups
  // then cost shared-memory wavefronts instead of L1 ones (QSG_SMEM_DICT=0 disables).
  const char* sd = std::getenv("QSG_SMEM_DICT");
  if (pf && G->n_terms == 1 && G->ops[0]->dict_n > 0 && G->ops[0]->dict_n <= 2048 && !(sd && sd[0] == '0'))
    P.smem_dict = G->ops[0]->dict_n;
  // single-term generator with a key-aligned store: stream it through the TMA ring (st 2) when
  // QSG_KA_SOLVE=1. Not the default: on TFIM-10 it cuts L1 wavefronts 35% and DRAM bytes 30% but
  // takes 30.5 ms against 27.6 ms for the coded path (K-grid "key-aligned store").
  const char* ks = std::getenv("QSG_KA_SOLVE");
  const int st = (G->n_terms == 1 && G->ops[0]->ka_nval > 0 && ks && ks[0] == '1') ? 2 : pf ? 1 : 0;
  if (st == 2) P.smem_dict = 0;
  const size_t dyn = grid_smem_bytes(P, st);
  // materialise the stage-2 input for the pipelined single-term path: one extra streaming pass and
  // barrier, half the stage-2 gathers (TFIM-10: 30.2 -> 29.1 ms). QSG_X2=0 disables.
  P.x2 = st >= 1 && G->n_terms == 1;
  if (const char* x2 = std::getenv("QSG_X2")) P.x2 = (x2[0] == '1' && P.x2) || st == 2;
  // an autonomous generator (no time-dependent coefficient): stage 2 then needs neither the x2
  // pass nor a second gathered vector (grid_engine.cu stage_pass, X2 = 2). QSG_K1G=0 keeps the
  // x2 pass. TFIM-10: 27.7 vs 28.2 ms per solve, identical statistics (profiles/r02_k1g.log).
  {
    bool aut = true;  // every term's coefficient time-independent (constant or params[i])
    for (int k = 1; k < G->n_terms; ++k)
      aut = aut && G->coeffs && (G->coeffs[k].kind == QSG_COEFF_CONST || G->coeffs[k].kind == QSG_COEFF_PARAM);
    const char* kg = std::getenv("QSG_K1G");
    P.k1g = aut && !(kg && kg[0] == '0');
    if (P.k1g) P.x2 = 0;
  }
  const int per_sm = grid_max_blocks_per_sm(mode, st, dyn);
  if (per_sm <= 0) return cuda_fail(cudaGetLastError(), "occupancy");
  const int max_grid = per_sm * ctx->sm_count;
  const long long nblk = (n + 31) / 32;
  // ~4 slices (128 rows) per CTA: small systems are latency-bound and gain from spreading out
  // (Kerr N=200: 60 -> 30 us per attempt from 20 to 148 CTAs, profiles/r01_summary.md)
  int grid = static_cast<int>(std::min<long long>(max_grid, std::max<long long>(1, (nblk + 3) / 4)));
  // ... but mid-size operators (up to 2,560 slices) run best on 128 CTAs, under one per SM: Kerr
  // mesolve us per attempt at 128 / 176-296 CTAs: N = 150 22.3 / 23.2, N = 200 23.1 / 24.1,
  // N = 250 24.6 / 25.2, while N = 300 (2,813 slices) wants all 296 (27.3 vs 33.2)
  // (scripts/probe_cl_env.py QSG_GRID=..., profiles/r02_small_grid.log)
  if (nblk < 2560) grid = std::min(grid, 128);
  if (const char* eg = std::getenv("QSG_GRID")) grid = std::max(1, std::min(max_grid, std::atoi(eg)));
  grid = static_cast<int>(std::min<long long>(grid, nblk));
  // Small systems (scripts/probe_small_grid.py, profiles/r02_small_grid.log, Kerr mesolve us per
  // DP5 attempt): every cross-CTA barrier also invalidates L1, so the operator and the state come
  // back from L2 each pass.
  //  * <= 16 slices (Kerr N = 20, 400 rows): ONE CTA, no grid barrier at all: 14.5 us against
  //    23.4 us on 4 CTAs;
  //  * <= 96 slices (Kerr N = 50, 2,500 rows): one 16-CTA thread-block cluster, hardware cluster
  //    barrier: 18.6 us against 22.8 us on a 20-CTA cooperative grid;
  //  * larger (N >= 100): the cooperative grid (N = 100: 21.6 us on 79 CTAs vs 29.5 us as a cluster).
  // QSG_GRID_CLUSTER=1/0 forces/disables the cluster; QSG_GRID still sets the CTA count.
  if (!std::getenv("QSG_GRID") && nblk <= 16) grid = 1;
  {
    const char* gc = std::getenv("QSG_GRID_CLUSTER");
    const bool want = gc ? gc[0] == '1' : (nblk > 16 && nblk <= 96 && !std::getenv("QSG_GRID"));
    const int cmax = want ? grid_max_cluster(mode, st, dyn) : 0;
    if (cmax > 0) {
      P.cluster = 1;
      grid = static_cast<int>(std::min<long long>(cmax, nblk));
      if (const char* cs = std::getenv("QSG_GRID_CLUSTER_SIZE")) grid = std::max(1, std::min(grid, std::atoi(cs)));
    }
  }
  (void)threads;
  if ((ce = d_ctl.alloc(sizeof(GridCtl), s)) || (ce = d_red.alloc(sizeof(double) * kNumSlots * grid, s)) ||
      (ce = d_bar.alloc(2 * sizeof(unsigned), s)))
    return cuda_fail(ce, "control");
  cudaMemsetAsync(d_bar.p, 0, 2 * sizeof(unsigned), s);
  cudaMemsetAsync(d_ctl.p, 0, sizeof(GridCtl), s);
  P.ctl = d_ctl.as<GridCtl>();
  P.red = d_red.as<double>();
  P.bar = d_bar.as<unsigned>();
  // Cluster-resident solve (K-cluster) for small single-term systems: the operator and the state in
  // the shared memory of one thread-block cluster (QSG_CLUSTER_SOLVE=0 disables, =1 forces when it fits)
  ClLayout cl{};
  int cl_ctas = 0;
  {
    const char* cs = std::getenv("QSG_CLUSTER_SOLVE");
    const bool allow = !(cs && cs[0] == '0');
    const bool forced = cs && cs[0] == '1';
    if (allow && G->n_terms == 1 && G->ops[0]->code_bytes == 0 && n <= kClusterSolveRows &&
        (forced || nblk >= kClusterSolveMinSlices) && !std::getenv("QSG_GRID")) {
      std::vector<long long> so(static_cast<size_t>(nblk + 1));
      if ((ce = cudaMemcpyAsync(so.data(), G->ops[0]->slice_off, sizeof(long long) * (nblk + 1), cudaMemcpyDeviceToHost, s)) ||
          (ce = cudaStreamSynchronize(s)))
        return cuda_fail(ce, "slice offsets");
      if (!plan_cluster_solve(P, so.data(), kObsSlots, mode == 0 ? static_cast<int>(eo_i.size()) : 0, &cl_ctas, &cl))
        cl_ctas = 0;
    }
  }
  cudaEventRecord(ctx->ev[0], s);
  if (cl_ctas > 0) {
    grid = cl_ctas;
    if ((ce = launch_cluster_dp5(P, mode, cl, cl_ctas, s))) return cuda_fail(ce, "cluster solver launch");
  } else if ((ce = launch_grid_dp5(P, mode, st, grid, s))) {
    return cuda_fail(ce, "solver launch");
  }
  cudaEventRecord(ctx->ev[1], s);
  GridCtl ctl{};
  if ((ce = cudaMemcpyAsync(&ctl, d_ctl.p, sizeof(GridCtl), cudaMemcpyDeviceToHost, s)))
    return cuda_fail(ce, "ctl copy");
  if ((ce = cudaStreamSynchronize(s))) return cuda_fail(ce, "solver");
  if (stats) *stats = qsg_stats{ctl.steps, ctl.rejected, ctl.rhs_evals};
  if (timing) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    timing->kernel_ms = ms;
    timing->attempts = ctl.attempts;
    timing->grid_ctas = grid;
    timing->lanes = lanes;
    timing->store = st;
    timing->engine = cl_ctas > 0 ? 2 : P.cluster ? 1 : 0;
  }
  if (qsg_status sst = status_from_device(ctl.status, ctl.fail_t)) return sst;
  if (expect && n_e > 0)
    if ((ce = cudaMemcpyAsync(expect, d_exp.p, static_cast<size_t>(n_e) * n_t * sizeof(double2), cudaMemcpyDefault, s)))
      return cuda_fail(ce, "expect copy");
  if (states && ev.n_save > 0 && !states_dev)
    if ((ce = cudaMemcpyAsync(states, P.states, static_cast<size_t>(ev.n_save) * vbytes, cudaMemcpyDefault, s)))
      return cuda_fail(ce, "states copy");
  if ((ce = cudaStreamSynchronize(s))) return cuda_fail(ce, "copy back");
  return QSG_OK;
}

}  // namespace qsg

using namespace qsg;

extern "C" {

const char* qsg_last_error(void) { return g_last_error.c_str(); }

qsg_status qsg_ctx_create(int device, qsg_ctx** out) {
  if (!out) return QSG_INVALID_GRID;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    set_error(std::string("no CUDA device available: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return QSG_CUDA_ERROR;
  }
  if (device < 0 || device >= ndev) {
    set_error("InvalidIndex: device index out of range");
    return QSG_INVALID_INDEX;
  }
  if ((e = cudaSetDevice(device))) return cuda_fail(e, "cudaSetDevice");
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device))) return cuda_fail(e, "device properties");
  if (prop.major < 10) {
    set_error("this build targets sm_100a (B200); device is sm_" + std::to_string(prop.major * 10 + prop.minor));
    return QSG_CUDA_ERROR;
  }
  auto* c = new qsg_ctx;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->l2_bytes = prop.l2CacheSize;
  std::snprintf(c->name, sizeof(c->name), "%s", prop.name);
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking))) {
    delete c;
    return cuda_fail(e, "stream");
  }
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  // All device memory of the library (operator stores, solver workspaces) comes from the device's
  // stream-ordered pool. Keep freed blocks reserved instead of returning them to the driver at
  // every synchronisation: repeated op_create/solve/destroy cycles then cost no remapping.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return QSG_OK;
}

static void ctx_release(qsg_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& ev : ctx->ev) cudaEventDestroy(ev);
  if (ctx->work) cudaFree(ctx->work);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void qsg_ctx_destroy(qsg_ctx* ctx) {
  if (ctx) ctx_release(ctx);
}

qsg_status qsg_device_info(qsg_ctx* ctx, int* sm_count, int64_t* l2_bytes, char* name, int name_len) {
  if (!ctx) return QSG_INVALID_GRID;
  if (sm_count) *sm_count = ctx->sm_count;
  if (l2_bytes) *l2_bytes = ctx->l2_bytes;
  if (name && name_len > 0) std::snprintf(name, name_len, "%s", ctx->name);
  return QSG_OK;
}

qsg_status qsg_op_create(qsg_ctx* ctx, const qsg_csr* a, qsg_op** out) {
  QSG_RANGE("qsg_op_create");
  if (!ctx || !a || !out) {
    set_error("InvalidGrid: null argument");
    return QSG_INVALID_GRID;
  }
  *out = nullptr;
  if (a->n_rows <= 0 || a->n_rows > 0x7fffffffLL || a->nnz < 0 || a->nnz > 0x7fffffffLL) {
    set_error("TooLarge: operator exceeds int32 indexing");
    return QSG_TOO_LARGE;
  }
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const long long n = a->n_rows, nsl = (n + 31) / 32;
  cudaError_t e;
  static const bool trace = std::getenv("QSG_TRACE_OP") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[qsg op] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // stage the CSR in HBM
  // stage the CSR in HBM; input already in this device's memory (e.g. the device-assembled
  // Liouvillian) is read in place instead of copied
  DevBuf d_rp, d_col, d_val, d_w;
  auto stage = [&](DevBuf& b, const void* src, size_t bytes, const void** p) -> cudaError_t {
    cudaPointerAttributes pa;
    if (src && cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeDevice &&
        pa.device == ctx->device) {
      *p = src;
      return cudaSuccess;
    }
    cudaGetLastError();
    const cudaError_t ue = upload(b, src, bytes, s);
    *p = b.p;
    return ue;
  };
  const void *prp = nullptr, *pcol = nullptr, *pval = nullptr;
  if ((e = stage(d_rp, a->rowptr, sizeof(int) * (n + 1), &prp)) ||
      (e = stage(d_col, a->col, sizeof(int) * a->nnz, &pcol)) ||
      (e = stage(d_val, a->val, sizeof(double2) * a->nnz, &pval)) ||
      (e = d_w.alloc(sizeof(long long) * nsl, s)))
    return cuda_fail(e, "operator staging");
  const int* srp = static_cast<const int*>(prp);
  const int* scol = static_cast<const int*>(pcol);
  const double2* sval = static_cast<const double2*>(pval);
  mark("upload");
  auto* op = new qsg_op;
  op->ctx = ctx;
  ctx->refs.fetch_add(1);
  op->n_rows = n;
  op->n_cols = a->n_cols;
  op->nnz = a->nnz;
  op->n_slices = nsl;
  if ((e = cudaMallocAsync(&op->rowlen, sizeof(int) * nsl * 32, s)) ||
      (e = cudaMallocAsync(&op->slice_off, sizeof(long long) * (nsl + 1), s))) {
    qsg_op_destroy(op);
    return cuda_fail(e, "operator store allocation");
  }
  sell_widths_kernel<<<static_cast<unsigned>((nsl * 32 + 255) / 256), 256, 0, s>>>(srp, static_cast<int>(n),
                                                                            op->rowlen, d_w.as<long long>());
  std::vector<long long> w(nsl), off(nsl + 1, 0);
  if ((e = cudaMemcpyAsync(w.data(), d_w.p, sizeof(long long) * nsl, cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s))) {
    qsg_op_destroy(op);
    return cuda_fail(e, "operator widths");
  }
  mark("widths");
  for (long long i = 0; i < nsl; ++i) {
    off[i + 1] = off[i] + w[i];
    op->max_rowlen = std::max<int>(op->max_rowlen, static_cast<int>(w[i]));
  }
  op->padded_cols = off[nsl];
  cudaMemcpyAsync(op->slice_off, off.data(), sizeof(long long) * (nsl + 1), cudaMemcpyHostToDevice, s);
  mark("slice_off");
  // Dictionary-coded store when the operator streams from HBM (otherwise it is L2-resident and
  // the code -> dictionary indirection only adds latency) and has <= 65535 distinct
  // (diagonal offset, value) pairs. QSG_NO_COMPRESS=1 disables, QSG_COMPRESS_MIN_BYTES moves the
  // size threshold.
  const char* nc = std::getenv("QSG_NO_COMPRESS");
  long long min_bytes = 32LL << 20;
  if (const char* mb = std::getenv("QSG_COMPRESS_MIN_BYTES")) min_bytes = std::atoll(mb);
  if (!(nc && nc[0] == '1') && a->nnz > 0 && 20 * a->nnz >= min_bytes) {
    if ((e = build_coded_store(op, srp, scol, sval, n, w, s))) {
      qsg_op_destroy(op);
      return cuda_fail(e, "coded operator store");
    }
    mark("coded");
  }
  // The plain SELL entries, unless the coded store replaces them: every reader of a coded operator
  // (grid engine, generator apply, batch engine via sell_view) then decodes the codes, and the
  // e2e path saves the plain fill and ~20 B per entry of HBM (TFIM-10: 497 MB). QSG_KEEP_PLAIN=1
  // builds both.
  const char* kp = std::getenv("QSG_KEEP_PLAIN");
  if (op->code_bytes == 0 || (kp && kp[0] == '1')) {
    const size_t pe = static_cast<size_t>(std::max<long long>(1, off[nsl] * 32));
    if ((e = cudaMallocAsync(&op->col, sizeof(int) * pe, s)) || (e = cudaMallocAsync(&op->val, sizeof(double2) * pe, s))) {
      qsg_op_destroy(op);
      return cuda_fail(e, "operator store allocation");
    }
    mark("alloc");
    cudaMemsetAsync(op->col, 0, sizeof(int) * pe, s);
    cudaMemsetAsync(op->val, 0, sizeof(double2) * pe, s);
    mark("memset");
    if (plain_align_enabled())
      sell_fill_aligned_kernel<<<static_cast<unsigned>(((n + 31) / 32 + kAlignWarps - 1) / kAlignWarps),
                                 32 * kAlignWarps, 0, s>>>(srp, scol, sval, static_cast<int>(n), op->slice_off,
                                                           op->col, op->val);
    else
      sell_fill_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
          srp, scol, sval, static_cast<int>(n), op->slice_off, op->col, op->val);
    if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(s))) {
      qsg_op_destroy(op);
      return cuda_fail(e, "operator store build");
    }
    mark("sell fill");
  }
  // key-aligned store, built on request (QSG_KA_STORE=1, or QSG_KA_SOLVE=1 for the grid solver)
  const char* kst = std::getenv("QSG_KA_STORE");
  const char* ksv = std::getenv("QSG_KA_SOLVE");
  if (a->nnz > 0 && ((kst && kst[0] == '1') || (ksv && ksv[0] == '1'))) {
    if ((e = build_ka_store(op, srp, scol, sval, n, s))) {
      qsg_op_destroy(op);
      return cuda_fail(e, "key-aligned operator store");
    }
    mark("key-aligned");
  }
  *out = op;
  return QSG_OK;
}

void qsg_op_destroy(qsg_op* op) {
  if (!op) return;
  // stream-ordered frees back into the context's pool: later solves on the same stream reuse the
  // memory without a device synchronisation or an unmap
  cudaSetDevice(op->ctx->device);
  cudaStream_t s = op->ctx->stream;
  for (void* p : {op->code, static_cast<void*>(op->code_off), static_cast<void*>(op->dict_off),
                  static_cast<void*>(op->ka_off), static_cast<void*>(op->ka_blk), static_cast<void*>(op->ka_val),
                  static_cast<void*>(op->dict_val), static_cast<void*>(op->slice_off),
                  static_cast<void*>(op->rowlen), static_cast<void*>(op->col), static_cast<void*>(op->val)})
    if (p) cudaFreeAsync(p, s);
  qsg_ctx* ctx = op->ctx;
  delete op;
  ctx_release(ctx);
}

int64_t qsg_op_nnz(const qsg_op* op) { return op ? op->nnz : 0; }

int32_t qsg_op_code_bytes(const qsg_op* op) { return op ? op->code_bytes : -1; }
int32_t qsg_op_dict_size(const qsg_op* op) { return op ? op->dict_n : -1; }

qsg_status qsg_op_store_info(const qsg_op* op, int64_t* info) {
  if (!op || !info) {
    set_error("InvalidGrid: null argument");
    return QSG_INVALID_GRID;
  }
  const long long nsl = op->n_slices;
  info[0] = op->ka_nval > 0 ? 3 : op->code_bytes;
  info[1] = 20 * op->nnz + 4 * op->n_rows + 8 * nsl;  // plain SELL bytes per SpMV
  info[2] = op->code_bytes ? op->code_bytes * op->nnz + 4 * op->n_rows + 16 * nsl + 20LL * op->dict_n : 0;
  info[3] = op->ka_bytes;
  info[4] = op->ka_nval;
  info[5] = op->ka_positions;
  info[6] = op->dict_n;
  info[7] = op->ka_slot;
  return QSG_OK;
}
int64_t qsg_op_rows(const qsg_op* op) { return op ? op->n_rows : 0; }

qsg_status qsg_generator_apply(qsg_ctx* ctx, const qsg_generator* g, const double* params,
                               int32_t n_params, double t, const double* y, double* out) {
  QSG_RANGE("qsg_generator_apply");
  if (!ctx || !g || g->n_terms < 1) return QSG_INVALID_GRID;
  const long long n = g->ops[0]->n_rows;
  if (qsg_status st = check_generator(g, n)) return st;
  cudaStream_t s = ctx->stream;
  cudaError_t e;
  DevBuf dy, dout, dp;
  const size_t vb = static_cast<size_t>(n) * sizeof(double2);
  if ((e = upload(dy, y, vb, s)) || (e = dout.alloc(vb, s))) return cuda_fail(e, "apply buffers");
  if (n_params > 0 && (e = upload(dp, params, sizeof(double) * n_params, s))) return cuda_fail(e, "params");
  if ((e = launch_apply(make_devgen(g), dp.as<double>(), static_cast<int>(n), t, dy.as<double2>(),
                        dout.as<double2>(), ctx->sm_count, s)))
    return cuda_fail(e, "apply launch");
  if ((e = cudaMemcpyAsync(out, dout.p, vb, cudaMemcpyDefault, s)) || (e = cudaStreamSynchronize(s)))
    return cuda_fail(e, "apply");
  return QSG_OK;
}

qsg_status qsg_generator_apply_timed(qsg_ctx* ctx, const qsg_generator* g, const double* params,
                                     int32_t n_params, double t, const double* y_dev, double* out_dev,
                                     int32_t reps, double* mean_ms) {
  if (!ctx || !g || g->n_terms < 1 || reps < 1) return QSG_INVALID_GRID;
  const long long n = g->ops[0]->n_rows;
  if (qsg_status st = check_generator(g, n)) return st;
  if (!is_device_ptr(y_dev) || !is_device_ptr(out_dev)) {
    set_error("InvalidGrid: timed apply needs device buffers");
    return QSG_INVALID_GRID;
  }
  cudaStream_t s = ctx->stream;
  cudaError_t e;
  DevBuf dp;
  if (n_params > 0 && (e = upload(dp, params, sizeof(double) * n_params, s))) return cuda_fail(e, "params");
  DevGen dg = make_devgen(g);
  cudaEventRecord(ctx->ev[0], s);
  for (int r = 0; r < reps; ++r)
    if ((e = launch_apply(dg, dp.as<double>(), static_cast<int>(n), t,
                          reinterpret_cast<const double2*>(y_dev), reinterpret_cast<double2*>(out_dev),
                          ctx->sm_count, s)))
      return cuda_fail(e, "apply launch");
  cudaEventRecord(ctx->ev[1], s);
  if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "apply");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  if (mean_ms) *mean_ms = ms / reps;
  return QSG_OK;
}

qsg_status qsg_mesolve(qsg_ctx* ctx, const qsg_generator* L, int64_t d, const double* rho0,
                       const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                       const double* params, int32_t n_params, const qsg_solve_opts* opts,
                       double* expect, double* states, qsg_stats* stats, qsg_timing* timing) {
  QSG_RANGE("qsg_mesolve");
  if (ctx) cudaSetDevice(ctx->device);
  return run_grid_solve(ctx, 0, L, d, rho0, tlist, n_t, n_e, e_ops, params, n_params, opts, expect,
                        states, stats, timing);
}

qsg_status qsg_sesolve(qsg_ctx* ctx, const qsg_generator* G, int64_t d, const double* psi0,
                       const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                       const double* params, int32_t n_params, const qsg_solve_opts* opts,
                       double* expect, double* states, qsg_stats* stats, qsg_timing* timing) {
  QSG_RANGE("qsg_sesolve");
  if (ctx) cudaSetDevice(ctx->device);
  return run_grid_solve(ctx, 1, G, d, psi0, tlist, n_t, n_e, e_ops, params, n_params, opts, expect,
                        states, stats, timing);
}

qsg_status qsg_rng_draw(qsg_ctx* ctx, uint64_t seed, uint64_t stream, int32_t kind, int32_t n,
                        double* out_d, uint64_t* out_u) {
  if (!ctx || n < 0) return QSG_INVALID_GRID;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  DevBuf bd, bu;
  cudaError_t e;
  if ((e = bd.alloc(sizeof(double) * std::max(1, n), s)) || (e = bu.alloc(sizeof(uint64_t) * std::max(1, n), s)))
    return cuda_fail(e, "rng buffers");
  rng_kernel<<<1, 32, 0, s>>>(seed, stream, kind, n, bd.as<double>(), bu.as<unsigned long long>());
  if ((e = cudaGetLastError())) return cuda_fail(e, "rng launch");
  if (kind == 0 && out_u) e = cudaMemcpyAsync(out_u, bu.p, sizeof(uint64_t) * n, cudaMemcpyDefault, s);
  if (kind != 0 && out_d) e = cudaMemcpyAsync(out_d, bd.p, sizeof(double) * n, cudaMemcpyDefault, s);
  if (e || (e = cudaStreamSynchronize(s))) return cuda_fail(e, "rng");
  return QSG_OK;
}

}  // extern "C"
