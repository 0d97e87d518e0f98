// On-device Liouvillian assembly: L = -i(spre(H) - spost(H)) + sum_k D(c_k),
// D(c) = sprepost(c, c^dag) - 0.5 spre(c^dag c) - 0.5 spost(c^dag c)   (superop.cpp:51-91).
//
// The reference builds L on the host from Eigen sparse expressions; for TFIM-10 that takes seconds,
// far longer than the whole GPU solve. Here each row R = p*d + q of L (column-stacked vec,
// superop.hpp:9-10) is produced by one thread as a merge of the term rows that can touch it:
//   spre(X)  = kron(I, X)          row q of X,   columns p*d + c            (superop.cpp:51-55)
//   spost(X) = kron(X^T, I)        row p of X^T, columns a*d + q            (superop.cpp:57-61)
//   sprepost(c, c^dag) = kron(conj(c), c)   rows p and q of c, columns j1*d + j2 (superop.cpp:63-69)
// Every term row is already sorted by column, so the union pattern comes out sorted, and each
// entry is folded in the reference's expression order with its union semantics (a present entry
// plus a missing one is `a + 0`, Eigen's binary evaluator, qobj.cpp:162-168):
//   l = (0,-1) * (spre(H) + (-1) spost(H));  for k: l = l + ((S1 + (-1)(0.5 S2)) + (-1)(0.5 S3)).
// The arithmetic uses explicitly rounded operations (no FMA contraction, like the reference's
// x86-64 baseline build), so the values equal the reference's entry for entry; the operator-level
// pieces (c^dag c, transposes) are formed on the host with the same product order
// (csrc/host/qobj.cpp, bit-identical to the oracle, tests/test_host_model.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "qsg_internal.h"
#include "../../include/qsim/qobj.hpp"

namespace qsg {
namespace {

constexpr int kMaxLiouCops = 32;
constexpr int kMaxLists = 2 + 3 * kMaxLiouCops;

struct DevCsr {
  const int* rp;
  const int* col;
  const double2* val;
};

struct LiouProblem {
  int d;
  int n_c;
  int has_h;
  DevCsr h, ht;  // H and H^T
  const DevCsr* c;     // n_c collapse operators
  const DevCsr* cdc;   // c^dag c
  const DevCsr* cdct;  // (c^dag c)^T
  const int* rowptr;   // fill phase: output row offsets
  int* out_col;
  double2* out_val;
  int* count;          // count phase: entries per row
};

// exactly rounded complex arithmetic (std::complex<double> operator* / operator+ without contraction)
__device__ __forceinline__ double2 xmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 xadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// List l of row (p, q): kind 0 = spre-like (row q of X, column p*d + c), kind 1 = spost-like
// (row p of X^T, column a*d + q), kind 2 = sprepost (rows p and q of c, column j1*d + j2).
// List order = fold order: H spre, H spost, then per c_k: sprepost, spre(cdc), spost(cdc).
struct Cursor {
  int pos, end;    // kinds 0/1: entry range; kind 2: outer (row p of c)
  int pos2, beg2, end2;  // kind 2: inner (row q of c)
};

template <bool FILL>
__global__ void __launch_bounds__(256) liouvillian_kernel(const LiouProblem P) {
  const long long n = static_cast<long long>(P.d) * P.d;
  const int n_lists = (P.has_h ? 2 : 0) + 3 * P.n_c;
  for (long long R = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; R < n;
       R += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(R / P.d), q = static_cast<int>(R % P.d);
    Cursor cur[kMaxLists];
    int head[kMaxLists];  // column of the list's current entry, INT_MAX when exhausted
    auto list_mat = [&](int l, int& kind) -> const DevCsr& {
      if (P.has_h && l < 2) {
        kind = l;
        return l == 0 ? P.h : P.ht;
      }
      const int m = l - (P.has_h ? 2 : 0), k = m / 3, r = m % 3;
      kind = r == 0 ? 2 : r == 1 ? 0 : 1;
      return r == 0 ? P.c[k] : r == 1 ? P.cdc[k] : P.cdct[k];
    };
    auto col_of = [&](int l) -> int {
      int kind;
      const DevCsr& X = list_mat(l, kind);
      const Cursor& c = cur[l];
      if (kind == 0) return c.pos < c.end ? p * P.d + X.col[c.pos] : INT_MAX;
      if (kind == 1) return c.pos < c.end ? X.col[c.pos] * P.d + q : INT_MAX;
      return (c.pos < c.end && c.beg2 < c.end2) ? X.col[c.pos] * P.d + X.col[c.pos2] : INT_MAX;
    };
    for (int l = 0; l < n_lists; ++l) {
      int kind;
      const DevCsr& X = list_mat(l, kind);
      Cursor& c = cur[l];
      const int r0 = kind == 0 ? q : p;
      c.pos = X.rp[r0];
      c.end = X.rp[r0 + 1];
      c.beg2 = c.pos2 = kind == 2 ? X.rp[q] : 0;
      c.end2 = kind == 2 ? X.rp[q + 1] : 0;
      head[l] = col_of(l);
    }
    // value of list l's current entry, then advance it
    auto take = [&](int l) -> double2 {
      int kind;
      const DevCsr& X = list_mat(l, kind);
      Cursor& c = cur[l];
      double2 v;
      if (kind == 0) {
        v = xmul(make_double2(1.0, 0.0), X.val[c.pos]);  // kron(I, X): 1 * x (superop.cpp:31-43)
        ++c.pos;
      } else if (kind == 1) {
        v = xmul(X.val[c.pos], make_double2(1.0, 0.0));  // kron(X^T, I): x * 1
        ++c.pos;
      } else {
        const double2 a = X.val[c.pos];                  // (c^dag)^T = conj(c)
        v = xmul(make_double2(a.x, -a.y), X.val[c.pos2]);
        if (++c.pos2 == c.end2) {
          c.pos2 = c.beg2;
          ++c.pos;
        }
      }
      head[l] = col_of(l);
      return v;
    };
    const double2 zero = make_double2(0.0, 0.0), m1 = make_double2(-1.0, 0.0), half = make_double2(0.5, 0.0);
    long long w = FILL ? P.rowptr[R] : 0;
    for (;;) {
      int C = INT_MAX;
      for (int l = 0; l < n_lists; ++l) C = min(C, head[l]);
      if (C == INT_MAX) break;
      if (!FILL) {
        for (int l = 0; l < n_lists; ++l)
          if (head[l] == C) take(l);
        ++w;
        continue;
      }
      bool has_l = false;
      double2 L = zero;
      int l = 0;
      if (P.has_h) {
        // l0 = (0,-1) * (spre(H) + (-1) * spost(H))   (superop.cpp:85, qobj.cpp:170-174)
        const bool a = head[0] == C, b = head[1] == C;
        if (a || b) {
          const double2 va = a ? take(0) : zero;
          const double2 vb = b ? xmul(m1, take(1)) : zero;
          const double2 hsum = a && b ? xadd(va, vb) : a ? xadd(va, zero) : xadd(zero, vb);
          L = xmul(make_double2(0.0, -1.0), hsum);
          has_l = true;
        }
        l = 2;
      }
      for (int k = 0; k < P.n_c; ++k, l += 3) {
        const bool p3 = head[l] == C, p4 = head[l + 1] == C, p5 = head[l + 2] == C;
        if (!(p3 || p4 || p5)) continue;
        // D(c) = (S1 + (-1)(0.5 S2)) + (-1)(0.5 S3)   (superop.cpp:71-76)
        const double2 s1 = p3 ? take(l) : zero;
        const double2 s2 = p4 ? xmul(m1, xmul(half, take(l + 1))) : zero;
        const double2 s3 = p5 ? xmul(m1, xmul(half, take(l + 2))) : zero;
        const bool d1p = p3 || p4;
        const double2 d1 = p3 && p4 ? xadd(s1, s2) : p3 ? xadd(s1, zero) : p4 ? xadd(zero, s2) : zero;
        const double2 dk = d1p && p5 ? xadd(d1, s3) : d1p ? xadd(d1, zero) : xadd(zero, s3);
        L = has_l ? xadd(L, dk) : xadd(zero, dk);  // l = l + D(c_k)   (superop.cpp:86-89)
        has_l = true;
      }
      P.out_col[w] = C;
      P.out_val[w] = L;
      ++w;
    }
    if (!FILL) P.count[R] = static_cast<int>(w);
  }
}

using qsim::Complex;
using qsim::SparseMatrix;

SparseMatrix to_sparse(const qsg_csr& a) {
  SparseMatrix m;
  m.rows = a.n_rows;
  m.cols = a.n_cols;
  m.rowptr.resize(static_cast<size_t>(a.n_rows + 1));
  m.col.resize(static_cast<size_t>(a.nnz));
  m.val.resize(static_cast<size_t>(a.nnz));
  const bool dev = is_device_ptr(a.rowptr);
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (dev) cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
    else if (bytes) std::memcpy(dst, src, bytes);
  };
  cp(m.rowptr.data(), a.rowptr, sizeof(int32_t) * m.rowptr.size());
  cp(m.col.data(), a.col, sizeof(int32_t) * m.col.size());
  cp(m.val.data(), a.val, sizeof(Complex) * m.val.size());
  return m;
}

struct DevCsrBuf {
  DevBuf rp, col, val;
  cudaError_t up(const SparseMatrix& m, cudaStream_t s, DevCsr& out) {
    cudaError_t e;
    if ((e = upload(rp, m.rowptr.data(), sizeof(int32_t) * m.rowptr.size(), s))) return e;
    if (m.col.empty()) {  // no entries: placeholders, never read
      if ((e = col.alloc(16, s)) || (e = val.alloc(16, s))) return e;
    } else if ((e = upload(col, m.col.data(), sizeof(int32_t) * m.col.size(), s)) ||
               (e = upload(val, m.val.data(), sizeof(Complex) * m.val.size(), s))) {
      return e;
    }
    out = DevCsr{rp.as<int>(), col.as<int>(), val.as<double2>()};
    return cudaSuccess;
  }
};

// 64-bit total of the per-row counts: the int32 scan below would wrap silently past 2^31 entries
__global__ void count_total_kernel(const int* __restrict__ cnt, long long n, unsigned long long* total) {
  unsigned long long a = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    a += static_cast<unsigned>(cnt[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, a);
}

// Assembles L into device CSR arrays owned by the caller-provided buffers.
qsg_status assemble(qsg_ctx* ctx, int64_t d, const qsg_csr* H, int32_t n_c, const qsg_csr* c_ops, DevBuf& rp,
                    DevBuf& col, DevBuf& val, long long& nnz) {
  if (!ctx || d <= 0 || n_c < 0 || (n_c > 0 && !c_ops)) {
    set_error("InvalidGrid: bad Liouvillian arguments");
    return QSG_INVALID_GRID;
  }
  if (n_c > kMaxLiouCops) {
    set_error("TooLarge: device Liouvillian assembly supports at most 32 collapse operators");
    return QSG_TOO_LARGE;
  }
  if (d * d > 0x7fffffffLL) {
    set_error("TooLarge: Liouvillian dimension exceeds int32 indexing");
    return QSG_TOO_LARGE;
  }
  auto check = [&](const qsg_csr& a, const char* what) -> qsg_status {
    if (a.n_rows != d || a.n_cols != d) {
      set_error(std::string("DimsMismatch: ") + what + " dims mismatch");
      return QSG_DIMS_MISMATCH;
    }
    return QSG_OK;
  };
  if (H)
    if (qsg_status st = check(*H, "Hamiltonian")) return st;
  for (int k = 0; k < n_c; ++k)
    if (qsg_status st = check(c_ops[k], "liouvillian: collapse")) return st;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  cudaError_t e;
  // operator-level pieces on the host, in the reference's arithmetic (superop.cpp:71-76)
  SparseMatrix h, ht;
  if (H) {
    h = to_sparse(*H);
    ht = qsim::sparse_transpose(h, false);
  }
  std::vector<SparseMatrix> cm(static_cast<size_t>(n_c)), cdc(static_cast<size_t>(n_c)), cdct(static_cast<size_t>(n_c));
  for (int k = 0; k < n_c; ++k) {
    cm[k] = to_sparse(c_ops[k]);
    cdc[k] = qsim::sparse_mul(qsim::sparse_transpose(cm[k], true), cm[k]);
    cdct[k] = qsim::sparse_transpose(cdc[k], false);
  }
  DevCsrBuf bh, bht;
  std::vector<DevCsrBuf> bc(static_cast<size_t>(n_c)), bcdc(static_cast<size_t>(n_c)), bcdct(static_cast<size_t>(n_c));
  LiouProblem P{};
  P.d = static_cast<int>(d);
  P.n_c = n_c;
  P.has_h = H ? 1 : 0;
  if (H && ((e = bh.up(h, s, P.h)) || (e = bht.up(ht, s, P.ht)))) return cuda_fail(e, "Liouvillian upload");
  std::vector<DevCsr> vc(static_cast<size_t>(std::max(1, static_cast<int>(n_c)))), vcdc(vc.size()), vcdct(vc.size());
  for (int k = 0; k < n_c; ++k)
    if ((e = bc[k].up(cm[k], s, vc[k])) || (e = bcdc[k].up(cdc[k], s, vcdc[k])) ||
        (e = bcdct[k].up(cdct[k], s, vcdct[k])))
      return cuda_fail(e, "Liouvillian upload");
  DevBuf dc, dcdc, dcdct;
  if ((e = upload(dc, vc.data(), sizeof(DevCsr) * vc.size(), s)) ||
      (e = upload(dcdc, vcdc.data(), sizeof(DevCsr) * vc.size(), s)) ||
      (e = upload(dcdct, vcdct.data(), sizeof(DevCsr) * vc.size(), s)))
    return cuda_fail(e, "Liouvillian upload");
  P.c = dc.as<DevCsr>();
  P.cdc = dcdc.as<DevCsr>();
  P.cdct = dcdct.as<DevCsr>();
  const long long n = d * d;
  // count -> exclusive scan -> fill
  if ((e = rp.alloc(sizeof(int) * (n + 1), s))) return cuda_fail(e, "Liouvillian rowptr");
  P.count = rp.as<int>();
  int dev_sms = ctx->sm_count;
  const unsigned blocks = static_cast<unsigned>(std::min<long long>((n + 255) / 256, 64LL * dev_sms));
  liouvillian_kernel<false><<<blocks, 256, 0, s>>>(P);
  if ((e = cudaGetLastError())) return cuda_fail(e, "Liouvillian count");
  cudaMemsetAsync(rp.as<int>() + n, 0, sizeof(int), s);
  {
    DevBuf tot;
    unsigned long long total64 = 0;
    if ((e = tot.alloc(sizeof(unsigned long long), s))) return cuda_fail(e, "Liouvillian count");
    cudaMemsetAsync(tot.p, 0, sizeof(unsigned long long), s);
    count_total_kernel<<<blocks, 256, 0, s>>>(rp.as<int>(), n, tot.as<unsigned long long>());
    if ((e = cudaGetLastError()) ||
        (e = cudaMemcpyAsync(&total64, tot.p, sizeof(total64), cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s)))
      return cuda_fail(e, "Liouvillian count");
    if (total64 > 0x7fffffffULL) {  // before any entry buffer is sized or written
      set_error("TooLarge: Liouvillian nnz exceeds int32 indexing");
      return QSG_TOO_LARGE;
    }
  }
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rp.as<int>(), rp.as<int>(), static_cast<int>(n + 1), s);
  DevBuf tmp;
  if ((e = tmp.alloc(tmp_bytes, s))) return cuda_fail(e, "Liouvillian scan");
  if ((e = cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, rp.as<int>(), rp.as<int>(), static_cast<int>(n + 1), s)))
    return cuda_fail(e, "Liouvillian scan");
  int total = 0;
  if ((e = cudaMemcpyAsync(&total, rp.as<int>() + n, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      (e = cudaStreamSynchronize(s)))
    return cuda_fail(e, "Liouvillian scan");
  nnz = total;
  if ((e = col.alloc(sizeof(int) * std::max(1, total), s)) || (e = val.alloc(sizeof(double2) * std::max(1, total), s)))
    return cuda_fail(e, "Liouvillian entries");
  P.rowptr = rp.as<int>();
  P.out_col = col.as<int>();
  P.out_val = val.as<double2>();
  liouvillian_kernel<true><<<blocks, 256, 0, s>>>(P);
  if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(s))) return cuda_fail(e, "Liouvillian fill");
  return QSG_OK;
}

}  // namespace
}  // namespace qsg

using namespace qsg;

extern "C" {

qsg_status qsg_liouvillian_create(qsg_ctx* ctx, int64_t d, const qsg_csr* H, int32_t n_c, const qsg_csr* c_ops,
                                  qsg_op** out) {
  QSG_RANGE("qsg_liouvillian_create");
  if (!out) {
    set_error("InvalidGrid: null output");
    return QSG_INVALID_GRID;
  }
  *out = nullptr;
  DevBuf rp, col, val;
  long long nnz = 0;
  if (qsg_status st = assemble(ctx, d, H, n_c, c_ops, rp, col, val, nnz)) return st;
  const qsg_csr L{d * d, d * d, nnz, rp.as<int32_t>(), col.as<int32_t>(), val.as<double>()};
  return qsg_op_create(ctx, &L, out);
}

qsg_status qsg_liouvillian_export(qsg_ctx* ctx, int64_t d, const qsg_csr* H, int32_t n_c, const qsg_csr* c_ops,
                                  int64_t* nnz_out, int32_t* rowptr, int32_t* col_out, double* val_out) {
  QSG_RANGE("qsg_liouvillian_export");
  DevBuf rp, col, val;
  long long nnz = 0;
  if (qsg_status st = assemble(ctx, d, H, n_c, c_ops, rp, col, val, nnz)) return st;
  if (nnz_out) *nnz_out = nnz;
  cudaStream_t s = ctx->stream;
  cudaError_t e;
  if (rowptr && (e = cudaMemcpyAsync(rowptr, rp.p, sizeof(int32_t) * (d * d + 1), cudaMemcpyDefault, s)))
    return cuda_fail(e, "Liouvillian export");
  if (col_out && (e = cudaMemcpyAsync(col_out, col.p, sizeof(int32_t) * nnz, cudaMemcpyDefault, s)))
    return cuda_fail(e, "Liouvillian export");
  if (val_out && (e = cudaMemcpyAsync(val_out, val.p, sizeof(double2) * nnz, cudaMemcpyDefault, s)))
    return cuda_fail(e, "Liouvillian export");
  if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "Liouvillian export");
  return QSG_OK;
}

}  // extern "C"
