// QuantumObject and the CSR sparse kernels behind operator construction (host side).
// Value semantics follow the reference (qobj.cpp:162-263 on Eigen CSC); the storage is CSR so
// the device operator store can ingest it directly, and the big kernels (kron, add) run over row
// ranges in parallel — the TFIM-10 Liouvillian (24.6 M entries) is assembled in ~1 s.
#include <algorithm>
#include <cmath>
#include <thread>

#include "../../../include/qsim/qobj.hpp"

namespace qsim {

const char* error_code_name(ErrorCode c) {
  switch (c) {
    case ErrorCode::KindMismatch: return "KindMismatch";
    case ErrorCode::DimsMismatch: return "DimsMismatch";
    case ErrorCode::InvalidSubsystem: return "InvalidSubsystem";
    case ErrorCode::InvalidDimension: return "InvalidDimension";
    case ErrorCode::InvalidIndex: return "InvalidIndex";
    case ErrorCode::TooLarge: return "TooLarge";
    case ErrorCode::IntegrationFailure: return "IntegrationFailure";
    case ErrorCode::EnsembleFailure: return "EnsembleFailure";
    case ErrorCode::SteadyStateFailure: return "SteadyStateFailure";
    case ErrorCode::DfdOverflow: return "DfdOverflow";
    case ErrorCode::InvalidGrid: return "InvalidGrid";
    case ErrorCode::InvalidScenario: return "InvalidScenario";
  }
  return "?";
}

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Ket: return "Ket";
    case Kind::Bra: return "Bra";
    case Kind::Operator: return "Operator";
    case Kind::SuperOperator: return "SuperOperator";
    case Kind::OperatorKet: return "OperatorKet";
    case Kind::OperatorBra: return "OperatorBra";
  }
  return "?";
}

long dims_product(const Dims& dims) {
  long p = 1;
  for (int d : dims) p *= d;
  return p;
}

namespace {

// Run f(lo, hi) over [0, n) in contiguous chunks on up to hardware_concurrency threads.
template <class F>
void parallel_rows(long n, long work, F&& f) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (work < (1L << 20) || nt == 1 || n < 2) {
    f(0L, n);
    return;
  }
  nt = static_cast<unsigned>(std::min<long>(nt, n));
  std::vector<std::thread> th;
  for (unsigned k = 0; k < nt; ++k) {
    const long lo = n * k / nt, hi = n * (k + 1) / nt;
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

void check_index_range(long entries) {
  require(entries <= 0x7fffffffL, ErrorCode::TooLarge, "operator exceeds int32 sparse indexing");
}

}  // namespace

SparseMatrix SparseMatrix::identity(long n) {
  SparseMatrix m;
  m.rows = m.cols = n;
  m.rowptr.resize(static_cast<size_t>(n + 1));
  m.col.resize(static_cast<size_t>(n));
  m.val.assign(static_cast<size_t>(n), Complex(1.0, 0.0));
  for (long i = 0; i <= n; ++i) m.rowptr[static_cast<size_t>(i)] = static_cast<int32_t>(i);
  for (long i = 0; i < n; ++i) m.col[static_cast<size_t>(i)] = static_cast<int32_t>(i);
  return m;
}

SparseMatrix SparseMatrix::empty(long r, long c) {
  SparseMatrix m;
  m.rows = r;
  m.cols = c;
  m.rowptr.assign(static_cast<size_t>(r + 1), 0);
  return m;
}

// Union add: a + b where both present, a + 0 / 0 + b otherwise (Eigen sparse binary op).
SparseMatrix sparse_add(const SparseMatrix& a, const SparseMatrix& b) {
  SparseMatrix m;
  m.rows = a.rows;
  m.cols = a.cols;
  m.rowptr.assign(static_cast<size_t>(a.rows + 1), 0);
  // pass 1: merged row lengths
  parallel_rows(a.rows, a.nonZeros() + b.nonZeros(), [&](long lo, long hi) {
    for (long r = lo; r < hi; ++r) {
      int ia = a.rowptr[r], ea = a.rowptr[r + 1], ib = b.rowptr[r], eb = b.rowptr[r + 1], c = 0;
      while (ia < ea || ib < eb) {
        if (ia < ea && ib < eb && a.col[ia] == b.col[ib]) { ++ia; ++ib; }
        else if (ia < ea && (ib >= eb || a.col[ia] < b.col[ib])) ++ia;
        else ++ib;
        ++c;
      }
      m.rowptr[static_cast<size_t>(r + 1)] = c;
    }
  });
  for (long r = 0; r < a.rows; ++r) m.rowptr[static_cast<size_t>(r + 1)] += m.rowptr[static_cast<size_t>(r)];
  check_index_range(m.rowptr.back());
  m.col.resize(static_cast<size_t>(m.rowptr.back()));
  m.val.resize(static_cast<size_t>(m.rowptr.back()));
  parallel_rows(a.rows, a.nonZeros() + b.nonZeros(), [&](long lo, long hi) {
    for (long r = lo; r < hi; ++r) {
      int ia = a.rowptr[r], ea = a.rowptr[r + 1], ib = b.rowptr[r], eb = b.rowptr[r + 1];
      size_t o = static_cast<size_t>(m.rowptr[r]);
      while (ia < ea || ib < eb) {
        if (ia < ea && ib < eb && a.col[ia] == b.col[ib]) {
          m.col[o] = a.col[ia];
          m.val[o] = a.val[ia] + b.val[ib];
          ++ia;
          ++ib;
        } else if (ia < ea && (ib >= eb || a.col[ia] < b.col[ib])) {
          m.col[o] = a.col[ia];
          m.val[o] = a.val[ia] + Complex(0.0, 0.0);
          ++ia;
        } else {
          m.col[o] = b.col[ib];
          m.val[o] = Complex(0.0, 0.0) + b.val[ib];
          ++ib;
        }
        ++o;
      }
    }
  });
  return m;
}

SparseMatrix sparse_scale(Complex s, const SparseMatrix& a) {
  SparseMatrix m = a;
  for (auto& v : m.val) v = s * v;
  return m;
}

// C(i,j) = sum_k A(i,k) B(k,j), k ascending, first term assigned — the accumulation order of
// Eigen's conservative sparse*sparse product for every (i,j).
SparseMatrix sparse_mul(const SparseMatrix& a, const SparseMatrix& b) {
  SparseMatrix m;
  m.rows = a.rows;
  m.cols = b.cols;
  m.rowptr.assign(static_cast<size_t>(a.rows + 1), 0);
  std::vector<int> mark(static_cast<size_t>(b.cols), -1);
  std::vector<Complex> acc(static_cast<size_t>(b.cols));
  std::vector<int32_t> idx;
  for (long i = 0; i < a.rows; ++i) {
    idx.clear();
    for (int p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
      const int k = a.col[p];
      const Complex x = a.val[p];
      for (int q = b.rowptr[k]; q < b.rowptr[k + 1]; ++q) {
        const int j = b.col[q];
        if (mark[static_cast<size_t>(j)] != i) {
          mark[static_cast<size_t>(j)] = static_cast<int>(i);
          acc[static_cast<size_t>(j)] = x * b.val[q];
          idx.push_back(j);
        } else {
          acc[static_cast<size_t>(j)] += x * b.val[q];
        }
      }
    }
    std::sort(idx.begin(), idx.end());
    for (int j : idx) {
      m.col.push_back(j);
      m.val.push_back(acc[static_cast<size_t>(j)]);
    }
    check_index_range(static_cast<long>(m.col.size()));
    m.rowptr[static_cast<size_t>(i + 1)] = static_cast<int32_t>(m.col.size());
  }
  return m;
}

// Row (ia*rb + ib) = row ia of A times row ib of B; columns come out sorted (ja major).
SparseMatrix sparse_kron(const SparseMatrix& a, const SparseMatrix& b) {
  SparseMatrix m;
  m.rows = a.rows * b.rows;
  m.cols = a.cols * b.cols;
  check_index_range(a.nonZeros() * b.nonZeros());
  m.rowptr.assign(static_cast<size_t>(m.rows + 1), 0);
  for (long ia = 0; ia < a.rows; ++ia) {
    const int la = a.rowptr[ia + 1] - a.rowptr[ia];
    for (long ib = 0; ib < b.rows; ++ib)
      m.rowptr[static_cast<size_t>(ia * b.rows + ib + 1)] = la * (b.rowptr[ib + 1] - b.rowptr[ib]);
  }
  for (long r = 0; r < m.rows; ++r) m.rowptr[static_cast<size_t>(r + 1)] += m.rowptr[static_cast<size_t>(r)];
  m.col.resize(static_cast<size_t>(m.rowptr.back()));
  m.val.resize(static_cast<size_t>(m.rowptr.back()));
  parallel_rows(a.rows, a.nonZeros() * b.nonZeros(), [&](long lo, long hi) {
    for (long ia = lo; ia < hi; ++ia)
      for (long ib = 0; ib < b.rows; ++ib) {
        size_t o = static_cast<size_t>(m.rowptr[static_cast<size_t>(ia * b.rows + ib)]);
        for (int p = a.rowptr[ia]; p < a.rowptr[ia + 1]; ++p) {
          const long cb = static_cast<long>(a.col[p]) * b.cols;
          const Complex av = a.val[p];
          for (int q = b.rowptr[ib]; q < b.rowptr[ib + 1]; ++q, ++o) {
            m.col[o] = static_cast<int32_t>(cb + b.col[q]);
            m.val[o] = av * b.val[q];
          }
        }
      }
  });
  return m;
}

SparseMatrix sparse_transpose(const SparseMatrix& a, bool conjugate) {
  SparseMatrix m;
  m.rows = a.cols;
  m.cols = a.rows;
  m.rowptr.assign(static_cast<size_t>(a.cols + 1), 0);
  for (int c : a.col) ++m.rowptr[static_cast<size_t>(c + 1)];
  for (long i = 0; i < a.cols; ++i) m.rowptr[static_cast<size_t>(i + 1)] += m.rowptr[static_cast<size_t>(i)];
  std::vector<int32_t> pos(m.rowptr.begin(), m.rowptr.end() - 1);
  m.col.resize(a.col.size());
  m.val.resize(a.val.size());
  for (long r = 0; r < a.rows; ++r)
    for (int p = a.rowptr[r]; p < a.rowptr[r + 1]; ++p) {
      const int q = pos[static_cast<size_t>(a.col[p])]++;
      m.col[static_cast<size_t>(q)] = static_cast<int32_t>(r);
      m.val[static_cast<size_t>(q)] = conjugate ? std::conj(a.val[p]) : a.val[p];
    }
  return m;
}

namespace {

SparseMatrix dense_to_sparse(const DenseMatrix& d) {  // Eigen sparseView(): exact zeros dropped
  SparseMatrix m = SparseMatrix::empty(d.rows(), d.cols());
  for (long r = 0; r < d.rows(); ++r) {
    for (long c = 0; c < d.cols(); ++c)
      if (d(r, c) != Complex(0.0, 0.0)) {
        m.col.push_back(static_cast<int32_t>(c));
        m.val.push_back(d(r, c));
      }
    m.rowptr[static_cast<size_t>(r + 1)] = static_cast<int32_t>(m.col.size());
  }
  return m;
}

DenseMatrix sparse_to_dense(const SparseMatrix& s) {
  DenseMatrix d(s.rows, s.cols);
  for (long r = 0; r < s.rows; ++r)
    for (int p = s.rowptr[r]; p < s.rowptr[r + 1]; ++p) d(r, s.col[p]) = s.val[p];
  return d;
}

DenseMatrix d_add(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix m(a.rows(), a.cols());
  for (long i = 0; i < a.size(); ++i) m.data()[i] = a.data()[i] + b.data()[i];
  return m;
}
DenseMatrix d_scale(Complex s, const DenseMatrix& a) {
  DenseMatrix m = a;
  for (long i = 0; i < a.size(); ++i) m.data()[i] = s * a.data()[i];
  return m;
}
DenseMatrix d_mul(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix m(a.rows(), b.cols());
  for (long j = 0; j < b.cols(); ++j)
    for (long k = 0; k < a.cols(); ++k) {
      const Complex y = b(k, j);
      for (long i = 0; i < a.rows(); ++i) m(i, j) += a(i, k) * y;
    }
  return m;
}
DenseMatrix d_adjoint(const DenseMatrix& a, bool conjugate) {
  DenseMatrix m(a.cols(), a.rows());
  for (long j = 0; j < a.cols(); ++j)
    for (long i = 0; i < a.rows(); ++i) m(j, i) = conjugate ? std::conj(a(i, j)) : a(i, j);
  return m;
}

std::pair<long, long> expected_shape(Kind k, long d) {
  switch (k) {
    case Kind::Ket: return {d, 1};
    case Kind::Bra: return {1, d};
    case Kind::Operator: return {d, d};
    case Kind::SuperOperator: return {d * d, d * d};
    case Kind::OperatorKet: return {d * d, 1};
    case Kind::OperatorBra: return {1, d * d};
  }
  return {0, 0};
}

Kind matmul_kind(Kind a, Kind b) {  // qobj.cpp:179-192
  using K = Kind;
  if (a == K::Operator && b == K::Operator) return K::Operator;
  if (a == K::Operator && b == K::Ket) return K::Ket;
  if (a == K::Bra && b == K::Operator) return K::Bra;
  if (a == K::Bra && b == K::Ket) return K::Operator;
  if (a == K::Ket && b == K::Bra) return K::Operator;
  if (a == K::SuperOperator && b == K::SuperOperator) return K::SuperOperator;
  if (a == K::SuperOperator && b == K::OperatorKet) return K::OperatorKet;
  if (a == K::OperatorBra && b == K::SuperOperator) return K::OperatorBra;
  if (a == K::OperatorBra && b == K::OperatorKet) return K::Operator;
  throw_error(ErrorCode::KindMismatch, std::string("cannot multiply ") + kind_name(a) + " by " + kind_name(b));
}

Kind dag_kind(Kind k) {
  switch (k) {
    case Kind::Ket: return Kind::Bra;
    case Kind::Bra: return Kind::Ket;
    case Kind::OperatorKet: return Kind::OperatorBra;
    case Kind::OperatorBra: return Kind::OperatorKet;
    default: return k;
  }
}

}  // namespace

QuantumObject::QuantumObject() : data_(DenseMatrix::Zero(1, 1)) {}

QuantumObject::QuantumObject(DenseMatrix data, Kind kind, Dims dims)
    : data_(std::move(data)), kind_(kind), dims_(std::move(dims)), dim_(dims_product(dims_)) {
  check_shape();
}

QuantumObject::QuantumObject(SparseMatrix data, Kind kind, Dims dims)
    : data_(std::move(data)), kind_(kind), dims_(std::move(dims)), dim_(dims_product(dims_)) {
  check_shape();
}

void QuantumObject::check_shape() const {  // qobj.cpp:101-108
  require(!dims_.empty(), ErrorCode::DimsMismatch, "dims must be non-empty");
  for (int d : dims_) require(d >= 1, ErrorCode::InvalidDimension, "dims entries must be >= 1");
  auto [r, c] = expected_shape(kind_, dim_);
  require(rows() == r && cols() == c, ErrorCode::DimsMismatch,
          std::string("payload shape does not match kind ") + kind_name(kind_));
}

long QuantumObject::rows() const { return is_dense() ? dense_ref().rows() : sparse_ref().rows; }
long QuantumObject::cols() const { return is_dense() ? dense_ref().cols() : sparse_ref().cols; }
const DenseMatrix& QuantumObject::dense_ref() const {
  require(is_dense(), ErrorCode::KindMismatch, "expected dense payload");
  return std::get<DenseMatrix>(data_);
}
const SparseMatrix& QuantumObject::sparse_ref() const {
  require(is_sparse(), ErrorCode::KindMismatch, "expected sparse payload");
  return std::get<SparseMatrix>(data_);
}
DenseMatrix QuantumObject::dense_matrix() const { return is_dense() ? dense_ref() : sparse_to_dense(sparse_ref()); }
SparseMatrix QuantumObject::sparse_matrix() const { return is_sparse() ? sparse_ref() : dense_to_sparse(dense_ref()); }
QuantumObject QuantumObject::to_dense() const { return QuantumObject(dense_matrix(), kind_, dims_); }
QuantumObject QuantumObject::to_sparse() const { return QuantumObject(sparse_matrix(), kind_, dims_); }
Complex QuantumObject::coeff(long row, long col) const {
  if (is_dense()) return dense_ref()(row, col);
  const SparseMatrix& s = sparse_ref();
  for (int p = s.rowptr[row]; p < s.rowptr[row + 1]; ++p)
    if (s.col[p] == col) return s.val[p];
  return Complex(0.0, 0.0);
}

QuantumObject operator+(const QuantumObject& a, const QuantumObject& b) {  // qobj.cpp:162-168
  require(a.kind() == b.kind(), ErrorCode::KindMismatch, "cannot add different kinds");
  require(a.dims() == b.dims(), ErrorCode::DimsMismatch, "operands have different dims");
  if (a.is_sparse() && b.is_sparse()) return QuantumObject(sparse_add(a.sparse_ref(), b.sparse_ref()), a.kind(), a.dims());
  return QuantumObject(d_add(a.dense_matrix(), b.dense_matrix()), a.kind(), a.dims());
}
QuantumObject operator-(const QuantumObject& a, const QuantumObject& b) { return a + (-b); }
QuantumObject operator-(const QuantumObject& a) { return Complex(-1.0, 0.0) * a; }

QuantumObject operator*(const QuantumObject& a, const QuantumObject& b) {  // qobj.cpp:201-217
  Kind k = matmul_kind(a.kind(), b.kind());
  require(a.dims() == b.dims(), ErrorCode::DimsMismatch, "operands have different dims");
  const bool scalar = (a.kind() == Kind::Bra && b.kind() == Kind::Ket) ||
                      (a.kind() == Kind::OperatorBra && b.kind() == Kind::OperatorKet);
  Dims od = scalar ? Dims{1} : a.dims();
  if (a.is_sparse() && b.is_sparse()) return QuantumObject(sparse_mul(a.sparse_ref(), b.sparse_ref()), k, od);
  return QuantumObject(d_mul(a.dense_matrix(), b.dense_matrix()), k, od);
}
QuantumObject operator*(Complex s, const QuantumObject& a) {
  if (a.is_sparse()) return QuantumObject(sparse_scale(s, a.sparse_ref()), a.kind(), a.dims());
  return QuantumObject(d_scale(s, a.dense_ref()), a.kind(), a.dims());
}
QuantumObject operator*(const QuantumObject& a, Complex s) { return s * a; }
QuantumObject operator*(double s, const QuantumObject& a) { return Complex(s, 0.0) * a; }
QuantumObject operator*(const QuantumObject& a, double s) { return Complex(s, 0.0) * a; }
QuantumObject operator/(const QuantumObject& a, Complex s) { return (Complex(1.0, 0.0) / s) * a; }
QuantumObject operator/(const QuantumObject& a, double s) { return (1.0 / s) * a; }

QuantumObject tensor(const QuantumObject& a, const QuantumObject& b) {  // qobj.cpp:232-263
  Kind k = a.kind();
  require(k == b.kind(), ErrorCode::KindMismatch, "tensor requires equal kinds");
  require(k == Kind::Ket || k == Kind::Bra || k == Kind::Operator, ErrorCode::KindMismatch,
          "tensor supports Ket, Bra and Operator kinds");
  Dims dims = a.dims();
  dims.insert(dims.end(), b.dims().begin(), b.dims().end());
  if (a.is_sparse() && b.is_sparse()) return QuantumObject(sparse_kron(a.sparse_ref(), b.sparse_ref()), k, dims);
  const DenseMatrix A = a.dense_matrix(), B = b.dense_matrix();
  DenseMatrix out(A.rows() * B.rows(), A.cols() * B.cols());
  for (long i = 0; i < A.rows(); ++i)
    for (long j = 0; j < A.cols(); ++j)
      for (long k2 = 0; k2 < B.rows(); ++k2)
        for (long l = 0; l < B.cols(); ++l) out(i * B.rows() + k2, j * B.cols() + l) = A(i, j) * B(k2, l);
  return QuantumObject(std::move(out), k, dims);
}

QuantumObject tensor(std::span<const QuantumObject> f) {
  require(!f.empty(), ErrorCode::DimsMismatch, "tensor of zero factors");
  QuantumObject out = f[0];
  for (size_t i = 1; i < f.size(); ++i) out = tensor(out, f[i]);
  return out;
}

QuantumObject dag(const QuantumObject& x) {
  if (x.is_sparse()) return QuantumObject(sparse_transpose(x.sparse_ref(), true), dag_kind(x.kind()), x.dims());
  return QuantumObject(d_adjoint(x.dense_ref(), true), dag_kind(x.kind()), x.dims());
}
QuantumObject transpose(const QuantumObject& x) {
  if (x.is_sparse()) return QuantumObject(sparse_transpose(x.sparse_ref(), false), dag_kind(x.kind()), x.dims());
  return QuantumObject(d_adjoint(x.dense_ref(), false), dag_kind(x.kind()), x.dims());
}
QuantumObject conj(const QuantumObject& x) {
  if (x.is_sparse()) {
    SparseMatrix m = x.sparse_ref();
    for (auto& v : m.val) v = std::conj(v);
    return QuantumObject(std::move(m), x.kind(), x.dims());
  }
  DenseMatrix m = x.dense_ref();
  for (long i = 0; i < m.size(); ++i) m.data()[i] = std::conj(m.data()[i]);
  return QuantumObject(std::move(m), x.kind(), x.dims());
}

Complex expect(const QuantumObject& op, const QuantumObject& state) {  // qobj.cpp:430-457
  require(op.is_operator(), ErrorCode::KindMismatch, "expect: first argument must be an Operator");
  require(op.dims() == state.dims(), ErrorCode::DimsMismatch, "expect: dims mismatch");
  const SparseMatrix A = op.sparse_matrix();
  if (state.is_ket()) {
    const DenseMatrix psi = state.dense_matrix();
    Complex acc = 0.0;
    for (long r = 0; r < A.rows; ++r) {
      Complex row = 0.0;
      for (int p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) row += A.val[p] * psi(A.col[p], 0);
      acc += std::conj(psi(r, 0)) * row;
    }
    return acc;
  }
  require(state.is_operator(), ErrorCode::KindMismatch, "expect: state must be Ket or Operator");
  const DenseMatrix R = state.dense_matrix();
  Complex acc = 0.0;
  for (long r = 0; r < A.rows; ++r)
    for (int p = A.rowptr[r]; p < A.rowptr[r + 1]; ++p) acc += A.val[p] * R(A.col[p], r);
  return acc;
}

Complex tr(const QuantumObject& x) {
  require(x.rows() == x.cols(), ErrorCode::KindMismatch, "tr expects a square object");
  Complex acc = 0.0;
  if (x.is_sparse()) {
    const SparseMatrix& m = x.sparse_ref();
    for (long r = 0; r < m.rows; ++r)
      for (int p = m.rowptr[r]; p < m.rowptr[r + 1]; ++p)
        if (m.col[p] == r) acc += m.val[p];
    return acc;
  }
  for (long i = 0; i < x.rows(); ++i) acc += x.dense_ref()(i, i);
  return acc;
}

double norm(const QuantumObject& x) {
  double s = 0.0;
  if (x.is_sparse())
    for (const auto& v : x.sparse_ref().val) s += std::norm(v);
  else
    for (long i = 0; i < x.dense_ref().size(); ++i) s += std::norm(x.dense_ref().data()[i]);
  return std::sqrt(s);
}

QuantumObject ket2dm(const QuantumObject& psi) {  // qobj.cpp:513-518
  if (psi.is_operator()) return psi;
  require(psi.is_ket(), ErrorCode::KindMismatch, "ket2dm expects a Ket");
  const DenseMatrix v = psi.dense_matrix();
  return QuantumObject(d_mul(v, d_adjoint(v, true)), Kind::Operator, psi.dims());
}

double max_abs_diff(const QuantumObject& a, const QuantumObject& b) {
  const DenseMatrix x = a.dense_matrix(), y = b.dense_matrix();
  double m = 0.0;
  for (long i = 0; i < x.size(); ++i) m = std::max(m, std::abs(x.data()[i] - y.data()[i]));
  return m;
}

}  // namespace qsim
