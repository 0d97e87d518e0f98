// qsim — C++ host API of the B200 engine, source-compatible with the reference's
// core/include/qsim/{errors,qobj}.hpp (errors.hpp:8-44, qobj.hpp:15-151).
//
// Differences from the reference, all deliberate:
//   * no Eigen: DenseMatrix is a small column-major complex matrix, SparseMatrix is CSR
//     (row-major, sorted columns, int32 indices) — the layout the device operator store ingests;
//   * sparse arithmetic follows the reference's value semantics exactly (union add, kron value
//     a*b, products accumulated over k ascending with the first term assigned), so operators
//     built here are bit-identical to the reference's; see tests/test_host_model.py;
//   * ptrace / expm / eigenstates / trace-norm are not part of the time-evolution path and are
//     not provided (SURVEY.md §2 marks them out of scope).
#pragma once

#include <complex>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace qsim {

// ---- errors.hpp:8-44 -------------------------------------------------------------------
enum class ErrorCode {
  KindMismatch,
  DimsMismatch,
  InvalidSubsystem,
  InvalidDimension,
  InvalidIndex,
  TooLarge,
  IntegrationFailure,
  EnsembleFailure,
  SteadyStateFailure,
  DfdOverflow,
  InvalidGrid,
  InvalidScenario,
};

const char* error_code_name(ErrorCode code);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void throw_error(ErrorCode code, const std::string& message) {
  throw Error(code, message);
}
inline void require(bool condition, ErrorCode code, const std::string& message) {
  if (!condition) throw_error(code, message);
}

// ---- containers ------------------------------------------------------------------------------
using Complex = std::complex<double>;
using Dims = std::vector<int>;

/// Column-major dense complex matrix (Eigen::MatrixXcd layout).
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(long rows, long cols) : rows_(rows), cols_(cols), v_(static_cast<size_t>(rows * cols)) {}
  long rows() const { return rows_; }
  long cols() const { return cols_; }
  long size() const { return rows_ * cols_; }
  Complex& operator()(long i, long j) { return v_[static_cast<size_t>(i + j * rows_)]; }
  const Complex& operator()(long i, long j) const { return v_[static_cast<size_t>(i + j * rows_)]; }
  Complex* data() { return v_.data(); }
  const Complex* data() const { return v_.data(); }
  static DenseMatrix Zero(long r, long c) { return DenseMatrix(r, c); }
  static DenseMatrix Identity(long n) {
    DenseMatrix m(n, n);
    for (long i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }

 private:
  long rows_ = 0, cols_ = 0;
  std::vector<Complex> v_;
};

/// Compressed sparse row matrix, columns sorted within each row, int32 indices.
struct SparseMatrix {
  long rows = 0, cols = 0;
  std::vector<int32_t> rowptr;  // rows + 1
  std::vector<int32_t> col;
  std::vector<Complex> val;
  long nonZeros() const { return static_cast<long>(val.size()); }
  static SparseMatrix identity(long n);
  static SparseMatrix empty(long r, long c);
};

enum class Kind { Ket, Bra, Operator, SuperOperator, OperatorKet, OperatorBra };
const char* kind_name(Kind kind);
long dims_product(const Dims& dims);

/// Quantum state / operator / superoperator on a truncated Hilbert space (qobj.hpp:33-79).
class QuantumObject {
 public:
  QuantumObject();
  QuantumObject(DenseMatrix data, Kind kind, Dims dims);
  QuantumObject(SparseMatrix data, Kind kind, Dims dims);

  Kind kind() const noexcept { return kind_; }
  const Dims& dims() const noexcept { return dims_; }
  long dim() const noexcept { return dim_; }
  long rows() const;
  long cols() const;
  bool is_dense() const noexcept { return std::holds_alternative<DenseMatrix>(data_); }
  bool is_sparse() const noexcept { return !is_dense(); }
  const DenseMatrix& dense_ref() const;
  const SparseMatrix& sparse_ref() const;
  DenseMatrix dense_matrix() const;
  SparseMatrix sparse_matrix() const;  // dense payloads drop exact zeros (Eigen sparseView)
  QuantumObject to_dense() const;
  QuantumObject to_sparse() const;
  Complex coeff(long row, long col) const;
  bool is_ket() const noexcept { return kind_ == Kind::Ket; }
  bool is_operator() const noexcept { return kind_ == Kind::Operator; }
  bool is_superoperator() const noexcept { return kind_ == Kind::SuperOperator; }

 private:
  std::variant<DenseMatrix, SparseMatrix> data_;
  Kind kind_ = Kind::Operator;
  Dims dims_{1};
  long dim_ = 1;
  void check_shape() const;
};

using Qobj = QuantumObject;

QuantumObject operator+(const QuantumObject& a, const QuantumObject& b);
QuantumObject operator-(const QuantumObject& a, const QuantumObject& b);
QuantumObject operator-(const QuantumObject& a);
QuantumObject operator*(const QuantumObject& a, const QuantumObject& b);
QuantumObject operator*(Complex s, const QuantumObject& a);
QuantumObject operator*(const QuantumObject& a, Complex s);
QuantumObject operator*(double s, const QuantumObject& a);
QuantumObject operator*(const QuantumObject& a, double s);
QuantumObject operator/(const QuantumObject& a, Complex s);
QuantumObject operator/(const QuantumObject& a, double s);

QuantumObject tensor(const QuantumObject& a, const QuantumObject& b);
QuantumObject tensor(std::span<const QuantumObject> factors);
QuantumObject dag(const QuantumObject& x);
QuantumObject transpose(const QuantumObject& x);
QuantumObject conj(const QuantumObject& x);
Complex expect(const QuantumObject& op, const QuantumObject& state);
Complex tr(const QuantumObject& x);
/// L2 (Frobenius) norm; the reference's trace norm (SVD) is not provided.
double norm(const QuantumObject& x);
QuantumObject ket2dm(const QuantumObject& psi);
double max_abs_diff(const QuantumObject& a, const QuantumObject& b);

// sparse kernels used by superop / factories (exposed for tests)
SparseMatrix sparse_add(const SparseMatrix& a, const SparseMatrix& b);
SparseMatrix sparse_scale(Complex s, const SparseMatrix& a);
SparseMatrix sparse_mul(const SparseMatrix& a, const SparseMatrix& b);
SparseMatrix sparse_kron(const SparseMatrix& a, const SparseMatrix& b);
SparseMatrix sparse_transpose(const SparseMatrix& a, bool conjugate);

}  // namespace qsim
