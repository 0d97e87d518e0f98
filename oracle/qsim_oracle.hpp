// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// Plain-C++ CPU restatement of the reference hot path (QuantumToolbox.jl desk-scale C++
// reference, /root/reference/proj/core). It exists so that tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg have a checker. The product (paper_2504_21440_b200) never
// links, imports or calls anything in this directory.
//
// The reference itself cannot be compiled here: proj/CMakeLists.txt:14 requires Eigen3 >= 3.4,
// which is absent from this image (and vendor/ doctest/CLI11/json are git-ignored and not
// shipped, proj/.gitignore:2). This file therefore restates, in reference arithmetic order,
//   * the Eigen sparse semantics the reference relies on (CSC storage, setFromTriplets
//     duplicate summation, union sparse add, conservative sparse*sparse product, CSC SpMV),
//   * qobj.cpp:162-263,410-414,513-518 (arithmetic, tensor, dag, ket2dm),
//   * factories.cpp:23-98,192-246 (operators, states, embed_site, ising_model),
//   * superop.cpp:5-91 (mat2vec, kron_sparse, spre/spost/sprepost, dissipator, liouvillian),
//   * integrator.hpp:23-195 (Dopri5),
//   * evolve.cpp:39-299 (td Liouvillian, SparseGenerator, events, sesolve, mesolve),
//   * trajectories.cpp:11-249 (run_ensemble, pairwise_sum, ensemble_stddev, mcsolve),
//   * rng.cpp:8-61 (splitmix64 / xoshiro256++ RngStream).
// Parity pinning: see oracle/README.md and tests/test_oracle_pinning.py.
#pragma once

#include <complex>
#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using cd = std::complex<double>;

// errors.hpp:8-21
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
const char* error_code_name(ErrorCode c);

// errors.hpp:26-36
class Error : public std::runtime_error {
 public:
  Error(ErrorCode c, const std::string& m)
      : std::runtime_error(std::string(error_code_name(c)) + ": " + m), code_(c) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};
[[noreturn]] void throw_error(ErrorCode c, const std::string& m);
inline void require(bool ok, ErrorCode c, const std::string& m) {
  if (!ok) throw_error(c, m);
}

// ---- containers with Eigen semantics -------------------------------------------------

/// Column-major dense complex matrix (Eigen::MatrixXcd layout).
struct Dense {
  long rows = 0, cols = 0;
  std::vector<cd> v;
  Dense() = default;
  Dense(long r, long c) : rows(r), cols(c), v(static_cast<size_t>(r * c)) {}
  cd& operator()(long i, long j) { return v[static_cast<size_t>(i + j * rows)]; }
  const cd& operator()(long i, long j) const { return v[static_cast<size_t>(i + j * rows)]; }
};

/// Compressed sparse column matrix, row indices sorted within each column
/// (Eigen::SparseMatrix<complex<double>> after makeCompressed(), qobj.hpp:17).
struct Csc {
  long rows = 0, cols = 0;
  std::vector<int> outer;  // cols + 1
  std::vector<int> inner;  // row index per entry
  std::vector<cd> val;
  long nnz() const { return static_cast<long>(val.size()); }
};

struct Triplet {
  long r, c;
  cd v;
};

Csc from_triplets(long rows, long cols, std::vector<Triplet> trips);
Csc sp_identity(long n);
Csc sp_add(const Csc& a, const Csc& b);
Csc sp_scale(cd s, const Csc& a);
Csc sp_mul(const Csc& a, const Csc& b);
Csc sp_transpose(const Csc& a);
Csc sp_adjoint(const Csc& a);
Csc sp_kron(const Csc& a, const Csc& b);
Dense sp_to_dense(const Csc& a);
Csc dense_to_sp(const Dense& a);  // sparseView(): drops exact zeros
/// out = A * y, Eigen CSC product order (per column, scatter into rows).
void sp_gemv(const Csc& a, const cd* y, cd* out);

// ---- QuantumObject (qobj.hpp:21-79) --------------------------------------------------

enum class Kind { Ket, Bra, Operator, SuperOperator, OperatorKet, OperatorBra };
using Dims = std::vector<int>;

struct QObj {
  bool is_sparse = false;
  Dense d;
  Csc s;
  Kind kind = Kind::Operator;
  Dims dims{1};
  long dim = 1;

  QObj() : d(1, 1) {}
  QObj(Dense m, Kind k, Dims ds);
  QObj(Csc m, Kind k, Dims ds);
  long rows() const { return is_sparse ? s.rows : d.rows; }
  long cols() const { return is_sparse ? s.cols : d.cols; }
  Dense dense() const { return is_sparse ? sp_to_dense(s) : d; }
  Csc sparse() const { return is_sparse ? s : dense_to_sp(d); }
  bool is_ket() const { return kind == Kind::Ket; }
  bool is_operator() const { return kind == Kind::Operator; }
};

QObj operator+(const QObj& a, const QObj& b);
QObj operator-(const QObj& a, const QObj& b);
QObj operator-(const QObj& a);
QObj operator*(const QObj& a, const QObj& b);
QObj operator*(cd s, const QObj& a);
QObj operator*(double s, const QObj& a);
QObj operator/(const QObj& a, double s);
QObj tensor(const QObj& a, const QObj& b);
QObj dag(const QObj& x);
QObj ket2dm(const QObj& psi);
double ket_norm(const QObj& psi);

// ---- factories.cpp ---------------------------------------------------------------------
QObj destroy(int n);
QObj create(int n);
QObj num(int n);
QObj qeye(int n);
QObj sigmax();
QObj sigmay();
QObj sigmaz();
QObj sigmap();
QObj sigmam();
QObj basis(int n, int i);
QObj fock(int n, int i);
QObj fock_dm(int n, int i);
QObj embed_site(const Dims& dims, int site, const QObj& op);
/// factories.cpp:204-246; `cap_sites` reproduces the reference's 12-site cap when true.
std::pair<QObj, std::vector<QObj>> ising_model(int nx, int ny, double jz, double hx,
                                               double gamma, bool periodic, bool cap_sites);

// ---- superop.cpp -----------------------------------------------------------------------
QObj spre(const QObj& a);
QObj spost(const QObj& b);
QObj sprepost(const QObj& a, const QObj& b);
QObj lindblad_dissipator(const QObj& c);
QObj liouvillian(const QObj& h, std::span<const QObj> c_ops);

// ---- evolve.hpp ------------------------------------------------------------------------
using Params = std::vector<double>;
using CoeffFn = std::function<cd(const Params&, double)>;
struct TdTerm {
  QObj op;
  CoeffFn coeff;
};
struct TdOp {
  QObj constant;
  std::vector<TdTerm> terms;
};
TdOp liouvillian_td(const TdOp& h, std::span<const QObj> c_ops);  // evolve.cpp:39-47

struct SolveOptions {
  double abstol = 1e-8;
  double reltol = 1e-6;
  bool store_states = false;
  std::optional<std::vector<double>> saveat;
  long max_steps = 10'000'000;
};
struct SolveStats {
  long steps = 0, rejected = 0, rhs_evals = 0;
  std::vector<std::string> warnings;
};
struct SolveResult {
  std::vector<double> times;
  Dense expect;  // n_e x n_t
  std::vector<QObj> states;
  SolveStats stats;
};

/// evolve.hpp:96-111 / evolve.cpp:53-69
// Worker threads for the element-wise loops and row-parallel SpMV of a single solve
// (bench.py's reference arm: "all the host threads it can use"). Every result is bit-identical
// to the 1-thread run: element-wise expressions are unchanged, each SpMV row accumulates its
// entries in the same ascending-column order as the CSC scatter, and every reduction (error
// norm, initial-step norms) is still summed sequentially in index order. Default 1.
void set_threads(int n);
int threads();

// Row-major copy of a Csc (columns ascending within a row) for the row-parallel product.
struct CsrRows {
  long rows = 0;
  std::vector<long> ptr;
  std::vector<int> col;
  std::vector<cd> val;
};

class SparseGenerator {
 public:
  SparseGenerator() = default;
  SparseGenerator(const TdOp& op, cd prefactor, const Params& params);
  void apply(double t, const std::vector<cd>& y, std::vector<cd>& out) const;
  long size() const { return const_part_.rows; }
  const Csc& const_part() const { return const_part_; }

 private:
  Csc const_part_;
  std::vector<std::pair<Csc, CoeffFn>> terms_;
  Params params_;
  mutable std::vector<cd> tmp_;
  // threads() > 1 at construction: row-major copies used by apply()
  CsrRows const_rows_;
  std::vector<CsrRows> term_rows_;
};

SolveResult sesolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                    std::span<const QObj> e_ops, const Params& params, const SolveOptions& opt);
SolveResult mesolve(const TdOp& h_or_l, const QObj& rho0, std::span<const double> tlist,
                    std::span<const QObj> c_ops, std::span<const QObj> e_ops,
                    const Params& params, const SolveOptions& opt);

// ---- rng.cpp ---------------------------------------------------------------------------
std::uint64_t splitmix64_next(std::uint64_t& state);
class RngStream {
 public:
  explicit RngStream(std::uint64_t master_seed, std::uint64_t stream = 0);
  std::uint64_t next_u64();
  double uniform();
  double uniform_pos();
  double normal();

 private:
  std::uint64_t s_[4];
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// ---- trajectories ----------------------------------------------------------------------
struct JumpEvent {
  double time;
  int channel;
};
struct EnsembleOptions {
  int ntraj = 100;
  std::uint64_t seed = 0;
  int n_threads = 0;
  bool store_per_traj = true;
  bool store_measurement = false;  // trajectories.hpp:31 (stochastic solvers)
  double dt_max = 0.0;             // trajectories.hpp:32 (<= 0: span / 1e4)
};
// Wiener record of one stochastic trajectory (trajectories.hpp:18-24): n_ch x n_steps, col-major.
struct WienerRecord {
  double dt = 0.0;
  long n_ch = 0, n_steps = 0;
  std::vector<double> increments, expectation, current;
};
struct TrajectoryData {
  Dense expect;
  std::vector<JumpEvent> jumps;
  bool failed = false;
  std::string failure;
  long steps = 0, rejected = 0, rhs_evals = 0;
  bool has_wiener = false;
  WienerRecord wiener;
};
struct EnsembleResult {
  std::vector<double> times;
  Dense mean_expect;
  std::vector<Dense> per_traj_expect;
  std::vector<std::vector<JumpEvent>> jump_records;
  std::vector<int> traj_indices;
  std::vector<TrajectoryData> raw;  // every slot, failed or not (oracle extension)
  int ntraj = 0;
  int failed_trajectories = 0;
  SolveStats stats;
};
EnsembleResult run_ensemble(const std::function<TrajectoryData(int, RngStream&)>& sim,
                            int n_e, std::span<const double> tlist, const EnsembleOptions& ens);
std::vector<double> ensemble_stddev(const EnsembleResult& r);  // n_e x n_t, col-major
EnsembleResult mcsolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                       std::span<const QObj> c_ops, std::span<const QObj> e_ops,
                       const EnsembleOptions& ens, const Params& params,
                       const SolveOptions& opt);
// Euler-Maruyama stochastic Schroedinger / master equations (trajectories.cpp:251-503)
struct EmGrid {
  long substeps_per_interval = 1;
  double dt = 0.0;
  long n_steps = 0;
};
EmGrid make_em_grid(std::span<const double> tlist, double dt_max);
EnsembleResult ssesolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                        std::span<const QObj> sc_ops, std::span<const QObj> e_ops,
                        const EnsembleOptions& ens, const Params& params);
EnsembleResult smesolve(const TdOp& h, const QObj& rho0, std::span<const double> tlist,
                        std::span<const QObj> c_ops, std::span<const QObj> sc_ops,
                        std::span<const QObj> e_ops, const EnsembleOptions& ens, const Params& params);

// ---- model zoo (scenario.cpp:247-395 style assembly) -------------------------------------
struct Model {
  std::string name;
  TdOp h;             // Hamiltonian (constant + parameter terms)
  std::vector<QObj> c_ops;
  std::vector<QObj> e_ops;
  QObj psi0;          // ket or density operator
  Params params;      // default parameter vector for td terms
};
Model build_model(const std::string& name, std::span<const double> p);

}  // namespace orc
