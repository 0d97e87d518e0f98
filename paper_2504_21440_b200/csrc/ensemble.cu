// Ensemble combine (trajectories.cpp:17-22, 82-83) — placeholder entry points filled in by the
// batched trajectory engine (batch_engine.cu).
#include <vector>

#include "qsg_internal.h"

using namespace qsg;

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
