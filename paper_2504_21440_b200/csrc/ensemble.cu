// Ensemble reductions (trajectories.cpp:17-22, 82-83): the device-side pairwise bracket over a
// block's completed trajectories (K7, used by qsg_mcsolve) and the host combine of per-block sums
// gathered from several devices or ranks (qsg_ensemble_combine).
#include <vector>

#include "qsg_internal.h"
#include "ensemble.h"

using namespace qsg;

namespace qsg {

// Completed-trajectory list, in index order (run_ensemble keeps the completed ones, :60-73).
// One block: a chunked exclusive scan over the status flags.
__global__ void __launch_bounds__(1024) ok_compact_kernel(const int* __restrict__ status, long long n,
                                                          int* __restrict__ ok_idx, long long* __restrict__ n_ok) {
  __shared__ int part[1024];
  __shared__ long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (long long c0 = 0; c0 < n; c0 += 1024) {
    const long long i = c0 + threadIdx.x;
    const int ok = i < n && status[i] == kDone;
    part[threadIdx.x] = ok;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int v = threadIdx.x >= static_cast<unsigned>(o) ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += v;
      __syncthreads();
    }
    if (ok) ok_idx[base + part[threadIdx.x] - 1] = static_cast<int>(i);
    __syncthreads();
    if (threadIdx.x == 1023) base += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_ok = base;
}

// pairwise_sum(m, lo, hi) of trajectories.cpp:17-22 for value index v: leaves are whole
// trajectory matrices, the split is lo + (hi - lo)/2, and each node is left + right. Evaluated
// with an explicit stack (a statically sized frame: device recursion would overrun the default
// per-thread stack at ~2^12 trajectories).
__device__ double2 bracket_dev(const double2* __restrict__ per, const int* __restrict__ ok, long long lo0,
                               long long hi0, long long nv, long long v) {
  constexpr int kDepth = 64;
  long long los[kDepth], his[kDepth];
  double2 left[kDepth];
  unsigned char st[kDepth];
  int sp = 0;
  los[0] = lo0;
  his[0] = hi0;
  st[0] = 0;
  double2 ret = make_double2(0.0, 0.0);
  for (;;) {
    const long long lo = los[sp], hi = his[sp];
    if (st[sp] == 0 && hi - lo == 1) {
      ret = per[static_cast<long long>(ok[lo]) * nv + v];
    } else if (st[sp] == 0) {  // descend left
      st[sp] = 1;
      ++sp;
      los[sp] = lo;
      his[sp] = lo + (hi - lo) / 2;
      st[sp] = 0;
      continue;
    } else if (st[sp] == 1) {  // left done: keep it, descend right
      left[sp] = ret;
      st[sp] = 2;
      ++sp;
      los[sp] = lo + (hi - lo) / 2;
      his[sp] = hi;
      st[sp] = 0;
      continue;
    } else {  // both done
      ret = make_double2(left[sp].x + ret.x, left[sp].y + ret.y);
    }
    if (sp == 0) return ret;
    --sp;
  }
}

__global__ void bracket_sums_kernel(const double2* __restrict__ per, const int* __restrict__ ok,
                                    const long long* __restrict__ n_ok, const long long* __restrict__ lo,
                                    const long long* __restrict__ hi, int n_ranges, long long nv,
                                    double2* __restrict__ out) {
  const long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int r = blockIdx.y;
  if (v >= nv) return;
  // hi < 0: up to the end of the completed list
  const long long a = n_ranges > 0 ? lo[r] : 0, b = n_ranges > 0 && hi[r] >= 0 ? hi[r] : *n_ok;
  out[static_cast<long long>(r) * nv + v] = b > a ? bracket_dev(per, ok, a, b, nv, v) : make_double2(0.0, 0.0);
}

cudaError_t device_bracket_sums(const double2* per, const int* status, long long n_sys, long long nv,
                                int n_ranges, const long long* range_lo, const long long* range_hi,
                                cudaStream_t s, long long& n_ok, std::vector<double2>& sums) {
  cudaError_t e;
  DevBuf ok, nok, dlo, dhi, out;
  const int nr = n_ranges > 0 ? n_ranges : 1;
  if ((e = ok.alloc(sizeof(int) * std::max(1LL, n_sys), s)) || (e = nok.alloc(sizeof(long long), s)) ||
      (e = out.alloc(sizeof(double2) * nv * nr, s)))
    return e;
  if (n_ranges > 0 && ((e = upload(dlo, range_lo, sizeof(long long) * n_ranges, s)) ||
                       (e = upload(dhi, range_hi, sizeof(long long) * n_ranges, s))))
    return e;
  ok_compact_kernel<<<1, 1024, 0, s>>>(status, n_sys, ok.as<int>(), nok.as<long long>());
  const dim3 grid(static_cast<unsigned>((nv + 127) / 128), static_cast<unsigned>(nr));
  bracket_sums_kernel<<<grid, 128, 0, s>>>(per, ok.as<int>(), nok.as<long long>(), dlo.as<long long>(),
                                           dhi.as<long long>(), n_ranges, nv, out.as<double2>());
  sums.resize(static_cast<size_t>(nv * nr));
  if ((e = cudaGetLastError()) ||
      (e = cudaMemcpyAsync(&n_ok, nok.p, sizeof(long long), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaMemcpyAsync(sums.data(), out.p, sizeof(double2) * nv * nr, cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return e;
  return cudaSuccess;
}

}  // namespace qsg

namespace {

// pairwise_sum bracket over [lo, hi) where leaves are whole blocks [begin_k, end_k) whose
// pre-summed values sit in block_sums. The recursion splits at lo + (hi - lo)/2 exactly as the
// reference; a split that falls inside a block is not representable and is rejected.
bool bracket(long long lo, long long hi, int nb, const long long* b, const long long* e,
             const double* sums, long long nv, std::vector<double>& out) {
  for (int k = 0; k < nb; ++k)
    if (b[k] == lo && e[k] == hi) {
      out.assign(sums + 2 * nv * k, sums + 2 * nv * (k + 1));
      return true;
    }
  if (hi - lo <= 1) return false;
  const long long mid = lo + (hi - lo) / 2;
  std::vector<double> l, r;
  if (!bracket(lo, mid, nb, b, e, sums, nv, l) || !bracket(mid, hi, nb, b, e, sums, nv, r)) return false;
  out.resize(l.size());
  for (size_t i = 0; i < l.size(); ++i) out[i] = l[i] + r[i];
  return true;
}

}  // namespace

extern "C" qsg_status qsg_ensemble_combine(int32_t n_blocks, const int64_t* block_begin,
                                           const int64_t* block_end, const double* block_sums,
                                           int64_t n_vals, int64_t n_ok_total, double* mean) {
  QSG_RANGE("qsg_ensemble_combine");
  if (n_blocks < 1 || n_ok_total < 1) {
    set_error("EnsembleFailure: every trajectory failed");
    return QSG_ENSEMBLE_FAILURE;
  }
  std::vector<long long> b(block_begin, block_begin + n_blocks), e(block_end, block_end + n_blocks);
  long long lo = b[0], hi = e[0];
  for (int k = 1; k < n_blocks; ++k) {
    lo = std::min(lo, b[k]);
    hi = std::max(hi, e[k]);
  }
  std::vector<double> tot;
  if (!bracket(lo, hi, n_blocks, b.data(), e.data(), block_sums, n_vals, tot)) {
    set_error("InvalidGrid: blocks do not align with the pairwise bracket");
    return QSG_INVALID_GRID;
  }
  // Eigen: matrix / Complex(N, 0) — complex division of every entry
  for (long long i = 0; i < n_vals; ++i) {
    const double re = tot[2 * i], im = tot[2 * i + 1], c = static_cast<double>(n_ok_total);
    mean[2 * i] = re / c;
    mean[2 * i + 1] = im / c;
  }
  return QSG_OK;
}
