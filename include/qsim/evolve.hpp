// Solver API — same entry points, options and results as the reference's
// core/include/qsim/evolve.hpp:13-117 and trajectories.hpp:13-95, executed on a B200.
//
// CoeffFn: the reference takes an arbitrary std::function<Complex(const Params&, double)>.
// Device solvers can only evaluate coefficients from the device library below; a Coeff built
// from an arbitrary callable still works for TimeDependentOperator::evaluate on the host, but a
// solve with it throws InvalidGrid (there is no CPU fallback by design).
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "factories.hpp"

namespace qsim {

using Params = std::vector<double>;

/// Time-dependent coefficient c(params, t).
class Coeff {
 public:
  enum class Kind { Const = 0, Param = 1, ParamCos = 2, ParamSin = 3, HostOnly = -1 };
  Coeff() = default;
  template <class F, class = std::enable_if_t<std::is_invocable_r_v<Complex, F, const Params&, double>>>
  Coeff(F f) : kind_(Kind::HostOnly), fn_(std::move(f)) {}  // NOLINT: implicit like std::function
  static Coeff constant(Complex c);
  static Coeff param(int i);                   // params[i]
  static Coeff param_cos(int i, int j);        // params[i] * cos(params[j] * t)
  static Coeff param_sin(int i, int j);        // params[i] * sin(params[j] * t)
  Complex operator()(const Params& p, double t) const;
  explicit operator bool() const { return kind_ != Kind::HostOnly || static_cast<bool>(fn_); }
  Kind kind() const { return kind_; }
  int i() const { return i_; }
  int j() const { return j_; }
  Complex value() const { return c_; }

 private:
  Kind kind_ = Kind::HostOnly;
  int i_ = 0, j_ = 0;
  Complex c_ = 0.0;
  std::function<Complex(const Params&, double)> fn_;
};
using CoeffFn = Coeff;

struct TdTerm {
  QuantumObject op;
  CoeffFn coeff;
};

/// Constant part plus (operator, coefficient) terms (evolve.hpp:23-43).
class TimeDependentOperator {
 public:
  TimeDependentOperator() = default;
  TimeDependentOperator(QuantumObject constant);  // NOLINT: implicit like the reference
  TimeDependentOperator(QuantumObject constant, std::vector<TdTerm> terms);
  void add_term(QuantumObject op, CoeffFn coeff);
  const QuantumObject& constant() const { return constant_; }
  std::span<const TdTerm> terms() const { return terms_; }
  bool is_constant() const { return terms_.empty(); }
  qsim::Kind kind() const { return constant_.kind(); }
  const Dims& dims() const { return constant_.dims(); }
  QuantumObject evaluate(const Params& params, double t) const;

 private:
  QuantumObject constant_;
  std::vector<TdTerm> terms_;
};

TimeDependentOperator liouvillian(const TimeDependentOperator& h, std::span<const QuantumObject> c_ops);

struct SolveOptions {  // evolve.hpp:55-64 (+ device selection)
  enum class Method { AdaptiveRK45, FixedRK4 };
  Method method = Method::AdaptiveRK45;
  double abstol = 1e-8;
  double reltol = 1e-6;
  double dt_fixed = 1e-3;
  bool store_states = false;
  std::optional<std::vector<double>> saveat;
  long max_steps = 10'000'000;
  int device = 0;
};

struct SolveStats {
  long steps = 0;
  long rejected = 0;
  long rhs_evals = 0;
  std::vector<std::string> warnings;
};

struct SolveResult {
  std::vector<double> times;
  DenseMatrix expect;  // n_e_ops x n_times
  std::vector<QuantumObject> states;
  SolveStats stats;
  double device_ms = 0.0;  // solver kernel time
};

SolveResult sesolve(const TimeDependentOperator& h, const QuantumObject& psi0, std::span<const double> tlist,
                    std::span<const QuantumObject> e_ops = {}, const Params& params = {},
                    const SolveOptions& options = {});

SolveResult mesolve(const TimeDependentOperator& h_or_l, const QuantumObject& rho0, std::span<const double> tlist,
                    std::span<const QuantumObject> c_ops = {}, std::span<const QuantumObject> e_ops = {},
                    const Params& params = {}, const SolveOptions& options = {});

// ---- trajectories.hpp -------------------------------------------------------------------------
struct JumpEvent {
  double time;
  int channel;
};

struct EnsembleOptions {
  int ntraj = 100;
  std::uint64_t seed = 0;
  int n_threads = 0;            // accepted for source compatibility; device work is not threaded
  bool store_per_traj = true;
  bool store_measurement = false;
  double dt_max = 0.0;
  std::vector<int> devices;     // GPUs to shard trajectories over (empty: SolveOptions::device)
};

/// Per-trajectory continuous-measurement record on the Euler-Maruyama grid (trajectories.hpp:18-24).
/// Eigen::MatrixXd there; here column-major n_channels x n_steps arrays of doubles.
struct WienerRecord {
  double dt = 0.0;
  long n_channels = 0, n_steps = 0;
  std::vector<double> increments;   // dW_n(t_k)
  std::vector<double> expectation;  // e_n(t_k) on the pre-step state
  std::vector<double> current;      // J_n(t_k) = expectation + increments / dt
  double at(const std::vector<double>& m, long n, long k) const { return m[static_cast<size_t>(n + n_channels * k)]; }
};

struct TrajectoryEnsembleResult {
  std::vector<double> times;
  DenseMatrix mean_expect;
  std::vector<DenseMatrix> per_traj_expect;
  std::vector<std::vector<JumpEvent>> jump_records;
  std::vector<WienerRecord> measurement;
  std::vector<int> traj_indices;
  int ntraj = 0;
  std::uint64_t master_seed = 0;
  int failed_trajectories = 0;
  SolveStats stats;
  double device_ms = 0.0;
};

std::vector<double> ensemble_stddev(const TrajectoryEnsembleResult& result);  // n_e x n_t col-major

// Sharding of trajectories [0, ntraj) over nshards devices or ranks: each shard is a contiguous
// run of whole subtrees ("leaves") of run_ensemble's pairwise bracket (trajectories.cpp:17-22), so
// per-leaf sums combine into the single-device mean bit for bit (qsg_ensemble_combine).
struct EnsembleShard {
  long begin = 0, end = 0;
  std::vector<std::pair<long, long>> leaves;
};
std::vector<EnsembleShard> ensemble_shards(long ntraj, int nshards);

TrajectoryEnsembleResult mcsolve(const TimeDependentOperator& h, const QuantumObject& psi0,
                                 std::span<const double> tlist, std::span<const QuantumObject> c_ops,
                                 std::span<const QuantumObject> e_ops, const EnsembleOptions& ens = {},
                                 const Params& params = {}, const SolveOptions& options = {});

/// Homodyne stochastic Schroedinger equation, Euler-Maruyama in Ito form, state renormalised after
/// every step (trajectories.cpp:367-393); tlist must be uniform. Runs on the device.
TrajectoryEnsembleResult ssesolve(const TimeDependentOperator& h, const QuantumObject& psi0,
                                  std::span<const double> tlist, std::span<const QuantumObject> sc_ops,
                                  std::span<const QuantumObject> e_ops, const EnsembleOptions& ens = {},
                                  const Params& params = {}, const SolveOptions& options = {});

/// Homodyne stochastic master equation; c_ops are unmonitored loss channels (trajectories.cpp:474-503).
/// The Liouvillian over c_ops followed by sc_ops is assembled on the device.
TrajectoryEnsembleResult smesolve(const TimeDependentOperator& h, const QuantumObject& rho0,
                                  std::span<const double> tlist, std::span<const QuantumObject> c_ops,
                                  std::span<const QuantumObject> sc_ops, std::span<const QuantumObject> e_ops,
                                  const EnsembleOptions& ens = {}, const Params& params = {},
                                  const SolveOptions& options = {});

// ---- rng.hpp (host copy, for re-deriving thresholds as the reference tests do) -----------------
class RngStream {
 public:
  explicit RngStream(std::uint64_t master_seed, std::uint64_t stream = 0);
  std::uint64_t next_u64();
  double uniform();
  double uniform_pos();

 private:
  std::uint64_t s_[4];
};

}  // namespace qsim
