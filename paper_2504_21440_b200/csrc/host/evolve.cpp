// Host side of sesolve / mesolve / mcsolve: builds the generator exactly as the reference
// (evolve.cpp:191-299, trajectories.cpp:217-249), uploads it into the HBM operator store and
// runs the device engines through the C-ABI (include/qsg.h). No CPU integration path exists.
#include <cmath>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "../../../include/qsg.h"
#include "../../../include/qsim/evolve.hpp"

namespace qsim {

// ---- device plumbing ----------------------------------------------------------------------------
namespace {

std::mutex g_ctx_mu;
std::map<int, qsg_ctx*>& ctx_map() {
  static std::map<int, qsg_ctx*> m;
  return m;
}

[[noreturn]] void throw_status(qsg_status st) {
  const std::string msg = qsg_last_error();
  if (st >= 1 && st <= 12) {
    // the device library already prefixes "<CodeName>: "; strip it to avoid doubling
    const std::string pre = std::string(error_code_name(static_cast<ErrorCode>(st - 1))) + ": ";
    throw Error(static_cast<ErrorCode>(st - 1), msg.rfind(pre, 0) == 0 ? msg.substr(pre.size()) : msg);
  }
  throw std::runtime_error("qsim device error: " + msg);
}

void check(qsg_status st) {
  if (st != QSG_OK) throw_status(st);
}

qsg_ctx* device_ctx(int dev) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto& m = ctx_map();
  auto it = m.find(dev);
  if (it != m.end()) return it->second;
  qsg_ctx* c = nullptr;
  check(qsg_ctx_create(dev, &c));
  m[dev] = c;
  return c;
}

qsg_csr csr_view(const SparseMatrix& m) {
  return qsg_csr{m.rows, m.cols, m.nonZeros(), m.rowptr.data(), m.col.data(),
                 reinterpret_cast<const double*>(m.val.data())};
}

struct OpHandle {
  qsg_op* op = nullptr;
  ~OpHandle() { qsg_op_destroy(op); }
};

// Device generator: SparseGenerator(op, prefactor, params) (evolve.cpp:53-61).
struct DeviceGenerator {
  std::vector<std::unique_ptr<OpHandle>> ops;
  std::vector<const qsg_op*> raw;
  std::vector<qsg_coeff> coeffs;
  qsg_generator g{};

  DeviceGenerator() = default;
  DeviceGenerator(qsg_ctx* ctx, const TimeDependentOperator& op, Complex prefactor) {
    add(ctx, (prefactor * op.constant()).sparse_matrix(), qsg_coeff{QSG_COEFF_CONST, 0, 0, 1.0, 0.0});
    for (const auto& t : op.terms()) {
      require(t.coeff.kind() != Coeff::Kind::HostOnly, ErrorCode::InvalidGrid,
              "time-dependent coefficient is a host function; the device solvers accept "
              "qsim::Coeff::constant/param/param_cos/param_sin");
      add(ctx, (prefactor * t.op).sparse_matrix(),
          qsg_coeff{static_cast<int32_t>(t.coeff.kind()), t.coeff.i(), t.coeff.j(), t.coeff.value().real(),
                    t.coeff.value().imag()});
    }
    g.n_terms = static_cast<int32_t>(raw.size());
    g.ops = raw.data();
    g.coeffs = coeffs.data();
  }
  // takes ownership of a store built elsewhere (device Liouvillian assembly)
  void adopt(qsg_op* op, qsg_coeff c) {
    auto h = std::make_unique<OpHandle>();
    h->op = op;
    raw.push_back(op);
    ops.push_back(std::move(h));
    coeffs.push_back(c);
    g.n_terms = static_cast<int32_t>(raw.size());
    g.ops = raw.data();
    g.coeffs = coeffs.data();
  }
  void add(qsg_ctx* ctx, const SparseMatrix& m, qsg_coeff c) {
    auto h = std::make_unique<OpHandle>();
    const qsg_csr v = csr_view(m);
    check(qsg_op_create(ctx, &v, &h->op));
    raw.push_back(h->op);
    ops.push_back(std::move(h));
    coeffs.push_back(c);
  }
};

void check_tlist(std::span<const double> tlist) {  // evolve.cpp:71-75
  require(tlist.size() >= 2, ErrorCode::InvalidGrid, "tlist needs at least two points");
  for (size_t i = 1; i < tlist.size(); ++i)
    require(tlist[i] > tlist[i - 1], ErrorCode::InvalidGrid, "tlist must increase strictly");
}

std::vector<SparseMatrix> to_sparse_ops(std::span<const QuantumObject> ops, const Dims& dims, const char* who) {
  std::vector<SparseMatrix> out;
  for (const auto& op : ops) {
    require(op.dims() == dims, ErrorCode::DimsMismatch, std::string(who) + ": operator dims mismatch");
    out.push_back(op.sparse_matrix());
  }
  return out;
}

qsg_solve_opts to_opts(const SolveOptions& o) {
  qsg_solve_opts q{};
  require(o.method == SolveOptions::Method::AdaptiveRK45, ErrorCode::InvalidGrid,
          "the device engine implements the adaptive Dormand-Prince 5(4) method");
  q.method = 0;
  q.abstol = o.abstol;
  q.reltol = o.reltol;
  q.dt_fixed = o.dt_fixed;
  q.store_states = o.store_states ? 1 : 0;
  q.n_saveat = o.saveat ? static_cast<int64_t>(o.saveat->size()) : 0;
  q.saveat = o.saveat ? o.saveat->data() : nullptr;
  q.max_steps = o.max_steps;
  return q;
}

size_t count_saves(std::span<const double> tlist, const SolveOptions& o, bool keep) {
  // merged event list of evolve.cpp:89-118: saveat points are unique after merging
  if (o.saveat) {
    std::vector<double> v = *o.saveat;
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v.size();
  }
  return keep ? tlist.size() : 0;
}

}  // namespace

// ---- Coeff / TimeDependentOperator ----------------------------------------------------------------
Coeff Coeff::constant(Complex c) {
  Coeff k;
  k.kind_ = Kind::Const;
  k.c_ = c;
  return k;
}
Coeff Coeff::param(int i) {
  Coeff k;
  k.kind_ = Kind::Param;
  k.i_ = i;
  return k;
}
Coeff Coeff::param_cos(int i, int j) {
  Coeff k;
  k.kind_ = Kind::ParamCos;
  k.i_ = i;
  k.j_ = j;
  return k;
}
Coeff Coeff::param_sin(int i, int j) {
  Coeff k = param_cos(i, j);
  k.kind_ = Kind::ParamSin;
  return k;
}
Complex Coeff::operator()(const Params& p, double t) const {
  switch (kind_) {
    case Kind::Const: return c_;
    case Kind::Param: return Complex(p.at(static_cast<size_t>(i_)), 0.0);
    case Kind::ParamCos: return Complex(p.at(static_cast<size_t>(i_)) * std::cos(p.at(static_cast<size_t>(j_)) * t));
    case Kind::ParamSin: return Complex(p.at(static_cast<size_t>(i_)) * std::sin(p.at(static_cast<size_t>(j_)) * t));
    case Kind::HostOnly: return fn_(p, t);
  }
  return 0.0;
}

TimeDependentOperator::TimeDependentOperator(QuantumObject constant) : constant_(std::move(constant)) {}
TimeDependentOperator::TimeDependentOperator(QuantumObject constant, std::vector<TdTerm> terms)
    : constant_(std::move(constant)), terms_(std::move(terms)) {
  for (const auto& t : terms_) {
    require(t.op.kind() == constant_.kind() && t.op.dims() == constant_.dims(), ErrorCode::DimsMismatch,
            "time-dependent terms must share kind and dims");
    require(static_cast<bool>(t.coeff), ErrorCode::InvalidGrid, "time-dependent term without coefficient function");
  }
}
void TimeDependentOperator::add_term(QuantumObject op, CoeffFn coeff) {
  require(op.kind() == constant_.kind() && op.dims() == constant_.dims(), ErrorCode::DimsMismatch,
          "time-dependent terms must share kind and dims");
  require(static_cast<bool>(coeff), ErrorCode::InvalidGrid, "time-dependent term without coefficient function");
  terms_.push_back({std::move(op), std::move(coeff)});
}
QuantumObject TimeDependentOperator::evaluate(const Params& params, double t) const {
  QuantumObject out = constant_;
  for (const auto& [op, coeff] : terms_) out = out + coeff(params, t) * op;
  return out;
}

TimeDependentOperator liouvillian(const TimeDependentOperator& h, std::span<const QuantumObject> c_ops) {
  QuantumObject l0 = liouvillian(h.constant(), c_ops);  // evolve.cpp:39-47
  std::vector<TdTerm> terms;
  for (const auto& [op, coeff] : h.terms()) terms.push_back({Complex(0, -1) * (spre(op) - spost(op)), coeff});
  return TimeDependentOperator(std::move(l0), std::move(terms));
}

// ---- sesolve / mesolve ---------------------------------------------------------------------------
SolveResult sesolve(const TimeDependentOperator& h, const QuantumObject& psi0, std::span<const double> tlist,
                    std::span<const QuantumObject> e_ops, const Params& params, const SolveOptions& options) {
  check_tlist(tlist);  // evolve.cpp:191-233
  require(psi0.is_ket(), ErrorCode::KindMismatch, "sesolve expects a Ket initial state");
  require(h.kind() == Kind::Operator, ErrorCode::KindMismatch, "sesolve expects an Operator");
  require(h.dims() == psi0.dims(), ErrorCode::DimsMismatch, "H and psi0 dims differ");
  SolveResult res;
  res.times.assign(tlist.begin(), tlist.end());
  const long ne = static_cast<long>(e_ops.size()), nt = static_cast<long>(tlist.size());
  res.expect = DenseMatrix(ne, nt);
  if (std::abs(norm(psi0) - 1.0) > 1e-10) res.stats.warnings.push_back("initial state is not normalized");
  qsg_ctx* ctx = device_ctx(options.device);
  DeviceGenerator gen(ctx, h, Complex(0, -1));
  auto e_mats = to_sparse_ops(e_ops, psi0.dims(), "sesolve e_ops");
  std::vector<qsg_csr> ev;
  for (const auto& m : e_mats) ev.push_back(csr_view(m));
  const DenseMatrix y0 = psi0.dense_matrix();
  const bool keep = options.store_states || e_ops.empty();
  const size_t nsave = count_saves(tlist, options, keep);
  const long d = psi0.dim();
  std::vector<Complex> states(nsave * static_cast<size_t>(d));
  const qsg_solve_opts o = to_opts(options);
  qsg_stats st{};
  qsg_timing tm{};
  check(qsg_sesolve(ctx, &gen.g, d, reinterpret_cast<const double*>(y0.data()), tlist.data(), nt,
                    static_cast<int32_t>(ne), ev.data(), params.data(), static_cast<int32_t>(params.size()), &o,
                    reinterpret_cast<double*>(res.expect.data()), nsave ? reinterpret_cast<double*>(states.data()) : nullptr,
                    &st, &tm));
  res.stats.steps = st.steps;
  res.stats.rejected = st.rejected;
  res.stats.rhs_evals = st.rhs_evals;
  res.device_ms = tm.kernel_ms;
  for (size_t s = 0; s < nsave; ++s) {
    DenseMatrix m(d, 1);
    std::copy(states.begin() + static_cast<long>(s) * d, states.begin() + static_cast<long>(s + 1) * d, m.data());
    res.states.emplace_back(std::move(m), Kind::Ket, psi0.dims());
  }
  return res;
}

SolveResult mesolve(const TimeDependentOperator& h_or_l, const QuantumObject& rho0_in, std::span<const double> tlist,
                    std::span<const QuantumObject> c_ops, std::span<const QuantumObject> e_ops, const Params& params,
                    const SolveOptions& options) {
  check_tlist(tlist);  // evolve.cpp:237-299
  TimeDependentOperator l_td;
  // An Operator generator with <= 32 collapse operators gets its Liouvillian assembled on the
  // device (qsg_liouvillian_create, equal to liouvillian() entry for entry); otherwise on the host.
  const bool device_l = h_or_l.kind() == Kind::Operator && c_ops.size() <= 32;
  if (device_l) {
    for (const auto& c : c_ops)  // superop.cpp:87
      require(c.dims() == h_or_l.dims(), ErrorCode::DimsMismatch, "liouvillian: collapse dims mismatch");
    l_td = h_or_l;
  } else if (h_or_l.kind() == Kind::Operator) {
    l_td = liouvillian(h_or_l, c_ops);
  } else {
    require(h_or_l.kind() == Kind::SuperOperator, ErrorCode::KindMismatch,
            "mesolve expects an Operator or SuperOperator generator");
    require(c_ops.empty(), ErrorCode::KindMismatch, "c_ops must be empty when a SuperOperator is supplied");
    l_td = h_or_l;
  }
  QuantumObject rho0 = rho0_in.is_ket() ? ket2dm(rho0_in) : rho0_in;
  require(rho0.is_operator(), ErrorCode::KindMismatch, "mesolve expects a Ket or Operator state");
  require(rho0.dims() == l_td.dims(), ErrorCode::DimsMismatch, "state dims do not match L");
  SolveResult res;
  res.times.assign(tlist.begin(), tlist.end());
  const long ne = static_cast<long>(e_ops.size()), nt = static_cast<long>(tlist.size());
  res.expect = DenseMatrix(ne, nt);
  qsg_ctx* ctx = device_ctx(options.device);
  DeviceGenerator gen;
  if (device_l) {
    const SparseMatrix h0 = h_or_l.constant().sparse_matrix();
    const qsg_csr hv = csr_view(h0);
    std::vector<SparseMatrix> cm;
    for (const auto& c : c_ops) cm.push_back(c.sparse_matrix());
    std::vector<qsg_csr> cv;
    for (const auto& m : cm) cv.push_back(csr_view(m));
    qsg_op* op = nullptr;
    check(qsg_liouvillian_create(ctx, h_or_l.constant().dim(), &hv, static_cast<int32_t>(cv.size()), cv.data(), &op));
    gen.adopt(op, qsg_coeff{QSG_COEFF_CONST, 0, 0, 1.0, 0.0});
    for (const auto& t : h_or_l.terms()) {  // -i(spre(op) - spost(op)) per term (evolve.cpp:39-47)
      require(t.coeff.kind() != Coeff::Kind::HostOnly, ErrorCode::InvalidGrid,
              "time-dependent coefficient is a host function; the device solvers accept "
              "qsim::Coeff::constant/param/param_cos/param_sin");
      const SparseMatrix tm = t.op.sparse_matrix();
      const qsg_csr tv = csr_view(tm);
      qsg_op* top = nullptr;
      check(qsg_liouvillian_create(ctx, h_or_l.constant().dim(), &tv, 0, nullptr, &top));
      gen.adopt(top, qsg_coeff{static_cast<int32_t>(t.coeff.kind()), t.coeff.i(), t.coeff.j(),
                               t.coeff.value().real(), t.coeff.value().imag()});
    }
  } else {
    gen = DeviceGenerator(ctx, l_td, Complex(1, 0));
  }
  auto e_mats = to_sparse_ops(e_ops, rho0.dims(), "mesolve e_ops");
  std::vector<qsg_csr> ev;
  for (const auto& m : e_mats) ev.push_back(csr_view(m));
  const long d = rho0.dim();
  const DenseMatrix m0 = rho0.dense_matrix();  // column-major == column stacking (:274-277)
  const bool keep = options.store_states || e_ops.empty();
  const size_t nsave = count_saves(tlist, options, keep);
  std::vector<Complex> states(nsave * static_cast<size_t>(d * d));
  const qsg_solve_opts o = to_opts(options);
  qsg_stats st{};
  qsg_timing tm{};
  check(qsg_mesolve(ctx, &gen.g, d, reinterpret_cast<const double*>(m0.data()), tlist.data(), nt,
                    static_cast<int32_t>(ne), ev.data(), params.data(), static_cast<int32_t>(params.size()), &o,
                    reinterpret_cast<double*>(res.expect.data()), nsave ? reinterpret_cast<double*>(states.data()) : nullptr,
                    &st, &tm));
  res.stats.steps = st.steps;
  res.stats.rejected = st.rejected;
  res.stats.rhs_evals = st.rhs_evals;
  res.device_ms = tm.kernel_ms;
  for (size_t s = 0; s < nsave; ++s) {
    DenseMatrix m(d, d);
    std::copy(states.begin() + static_cast<long>(s) * d * d, states.begin() + static_cast<long>(s + 1) * d * d, m.data());
    res.states.emplace_back(std::move(m), Kind::Operator, rho0.dims());
  }
  return res;
}

// ---- mcsolve --------------------------------------------------------------------------------------
namespace {
DenseMatrix pairwise_sum(const std::vector<const DenseMatrix*>& m, size_t lo, size_t hi) {  // :17-22
  if (hi - lo == 1) return *m[lo];
  const size_t mid = lo + (hi - lo) / 2;
  DenseMatrix a = pairwise_sum(m, lo, mid), b = pairwise_sum(m, mid, hi);
  for (long i = 0; i < a.size(); ++i) a.data()[i] += b.data()[i];
  return a;
}
}  // namespace

TrajectoryEnsembleResult mcsolve(const TimeDependentOperator& h, const QuantumObject& psi0,
                                 std::span<const double> tlist, std::span<const QuantumObject> c_ops,
                                 std::span<const QuantumObject> e_ops, const EnsembleOptions& ens,
                                 const Params& params, const SolveOptions& options) {
  check_tlist(tlist);  // trajectories.cpp:217-249
  require(psi0.is_ket(), ErrorCode::KindMismatch, "mcsolve expects a Ket initial state");
  require(h.kind() == Kind::Operator, ErrorCode::KindMismatch, "mcsolve expects an Operator H");
  require(h.dims() == psi0.dims(), ErrorCode::DimsMismatch, "H and psi0 dims differ");
  require(ens.ntraj >= 1, ErrorCode::InvalidGrid, "ntraj must be >= 1");
  QuantumObject heff_const = h.constant();
  for (const auto& c : c_ops) {
    require(c.dims() == psi0.dims(), ErrorCode::DimsMismatch, "collapse operator dims mismatch");
    heff_const = heff_const + Complex(0, -0.5) * (dag(c) * c);
  }
  TimeDependentOperator heff(heff_const, std::vector<TdTerm>(h.terms().begin(), h.terms().end()));
  std::vector<SparseMatrix> c_mats, e_mats;
  for (const auto& c : c_ops) c_mats.push_back(c.sparse_matrix());
  for (const auto& e : e_ops) {
    require(e.dims() == psi0.dims(), ErrorCode::DimsMismatch, "e_op dims mismatch");
    e_mats.push_back(e.sparse_matrix());
  }
  std::vector<qsg_csr> cv, ev;
  for (const auto& m : c_mats) cv.push_back(csr_view(m));
  for (const auto& m : e_mats) ev.push_back(csr_view(m));
  const DenseMatrix y0 = psi0.dense_matrix();
  const long ne = static_cast<long>(e_ops.size()), nt = static_cast<long>(tlist.size());
  const long ntraj = ens.ntraj, blk = ne * nt;
  const qsg_solve_opts o = to_opts(options);
  std::vector<int> devs = ens.devices.empty() ? std::vector<int>{options.device} : ens.devices;
  const int nd = static_cast<int>(std::min<long>(static_cast<long>(devs.size()), ntraj));
  // jump records kept per trajectory by the batched call; longer logs are re-run below
  // (QSG_MC_JUMP_CAP lowers the capacity so tests can exercise that path)
  const long kJumpCap = [] {
    const char* e = std::getenv("QSG_MC_JUMP_CAP");
    const long v = e ? std::atol(e) : 0;
    return v > 0 ? v : 256L;
  }();
  // Shards: whole subtrees of the pairwise bracket (trajectories.cpp:17-22), so every shard's
  // device-side subtree sums combine into exactly the single-device mean (ensemble_shards).
  const std::vector<EnsembleShard> shards = ensemble_shards(ntraj, nd);
  // per-trajectory expectations come back when stored, or when several shards might need the
  // host bracket (a failed trajectory shifts the bracket over the completed list)
  const bool fetch_per = ens.store_per_traj || nd > 1;
  std::vector<Complex> per(fetch_per ? static_cast<size_t>(ntraj * blk) : 0);
  std::vector<int32_t> failed(static_cast<size_t>(ntraj)), jcount(static_cast<size_t>(ntraj));
  std::vector<double> ftime(static_cast<size_t>(ntraj)), jtime(static_cast<size_t>(ntraj * kJumpCap));
  std::vector<int32_t> jch(static_cast<size_t>(ntraj * kJumpCap));
  std::vector<int64_t> tstats(static_cast<size_t>(ntraj * 3));
  std::vector<std::vector<Complex>> leaf_sums(static_cast<size_t>(nd));
  std::vector<Complex> bsum(static_cast<size_t>(std::max<long>(1, blk)) * static_cast<size_t>(nd));
  std::vector<int64_t> nok(static_cast<size_t>(nd));
  std::vector<qsg_status> rcs(static_cast<size_t>(nd), QSG_OK);
  std::vector<std::string> errs(static_cast<size_t>(nd));
  std::vector<double> dev_ms(static_cast<size_t>(nd));
  // NCCL communicator over distinct devices (the all-gather of leaf sums); QSG_MC_NCCL=1 uses it
  // for a single device too. Duplicate device ids run one context per shard and combine on the host.
  std::vector<qsg_comm*> comms;
  bool distinct = true;
  for (int i = 0; i < nd; ++i)
    for (int j = 0; j < i; ++j) distinct = distinct && devs[static_cast<size_t>(i)] != devs[static_cast<size_t>(j)];
  const char* force = std::getenv("QSG_MC_NCCL");
  if (distinct && (nd > 1 || (force && force[0] == '1'))) {
    comms.assign(static_cast<size_t>(nd), nullptr);
    check(qsg_comm_init_all(nd, devs.data(), comms.data()));
  }
  struct CommGuard {
    std::vector<qsg_comm*>& c;
    ~CommGuard() {
      for (auto* x : c) qsg_comm_destroy(x);
    }
  } comm_guard{comms};
  std::vector<std::vector<Complex>> gathered(static_cast<size_t>(nd));
  int max_leaves = 0;
  for (const auto& sh : shards) max_leaves = std::max(max_leaves, static_cast<int>(sh.leaves.size()));
  const long gcount = 2 * (2 + static_cast<long>(max_leaves) * blk);  // doubles per rank in the gather
  auto run = [&](int k) {
    const EnsembleShard& sh = shards[static_cast<size_t>(k)];
    const long b = sh.begin, e = sh.end;
    if (e <= b && comms.empty()) return;
    try {
      // one context per shard (own stream and events): shards on the same device do not share one
      qsg_ctx* ctx = comms.empty() ? nullptr : qsg_comm_ctx(comms[static_cast<size_t>(k)]);
      qsg_ctx* own = nullptr;
      if (!ctx) {
        check(qsg_ctx_create(devs[static_cast<size_t>(k)], &own));
        ctx = own;
      }
      struct CtxGuard {
        qsg_ctx* c;
        ~CtxGuard() {
          if (c) qsg_ctx_destroy(c);
        }
      } ctx_guard{own};
      DeviceGenerator gen(ctx, heff, Complex(0, -1));
      std::vector<int64_t> rlo, rhi;  // leaves as positions in the shard's completed list (valid when none failed)
      for (const auto& lf : sh.leaves) {
        rlo.push_back(lf.first - b);
        rhi.push_back(lf.second - b);
      }
      auto& ls = leaf_sums[static_cast<size_t>(k)];
      ls.assign(static_cast<size_t>(std::max<long>(1, blk)) * sh.leaves.size(), Complex(0, 0));
      qsg_mc_out out{};
      out.per_traj_expect = fetch_per ? reinterpret_cast<double*>(per.data() + b * blk) : nullptr;
      out.block_sum = reinterpret_cast<double*>(bsum.data() + k * std::max<long>(1, blk));
      out.n_ok = &nok[static_cast<size_t>(k)];
      out.failed = failed.data() + b;
      out.fail_time = ftime.data() + b;
      out.traj_stats = tstats.data() + 3 * b;
      out.jump_count = jcount.data() + b;
      out.jump_time = jtime.data() + b * kJumpCap;
      out.jump_channel = jch.data() + b * kJumpCap;
      out.jump_capacity = kJumpCap;
      out.n_ranges = static_cast<int32_t>(sh.leaves.size());
      out.range_lo = rlo.data();
      out.range_hi = rhi.data();
      out.range_sums = reinterpret_cast<double*>(ls.data());
      qsg_timing tm{};
      if (e > b)
        rcs[static_cast<size_t>(k)] =
            qsg_mcsolve(ctx, &gen.g, static_cast<int32_t>(cv.size()), cv.data(), static_cast<int32_t>(ne),
                        ev.data(), psi0.dim(), reinterpret_cast<const double*>(y0.data()), tlist.data(), nt,
                        params.data(), static_cast<int32_t>(params.size()), ens.seed, b, e, &o, &out, &tm);
      if (rcs[static_cast<size_t>(k)] != QSG_OK) errs[static_cast<size_t>(k)] = qsg_last_error();
      dev_ms[static_cast<size_t>(k)] = tm.kernel_ms;
      if (!comms.empty()) {  // NCCL all-gather of [n_ok, n_leaves, leaf sums] from every shard
        std::vector<Complex> send(static_cast<size_t>(gcount / 2), Complex(0, 0));
        send[0] = Complex(static_cast<double>(nok[static_cast<size_t>(k)]), rcs[static_cast<size_t>(k)] == QSG_OK ? 0.0 : 1.0);
        send[1] = Complex(static_cast<double>(sh.leaves.size()), 0.0);
        std::copy(ls.begin(), ls.end(), send.begin() + 2);
        auto& g = gathered[static_cast<size_t>(k)];
        g.resize(static_cast<size_t>(gcount / 2 * nd));
        const qsg_status gs = qsg_comm_allgather(comms[static_cast<size_t>(k)], reinterpret_cast<const double*>(send.data()),
                                                 gcount, reinterpret_cast<double*>(g.data()));
        if (gs != QSG_OK && rcs[static_cast<size_t>(k)] == QSG_OK) {
          rcs[static_cast<size_t>(k)] = gs;
          errs[static_cast<size_t>(k)] = qsg_last_error();
        }
      }
    } catch (const std::exception& ex) {
      rcs[static_cast<size_t>(k)] = QSG_CUDA_ERROR;
      errs[static_cast<size_t>(k)] = ex.what();
    }
  };
  if (nd == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nd; ++k) th.emplace_back(run, k);
    for (auto& t : th) t.join();
  }
  for (int k = 0; k < nd; ++k)
    if (rcs[static_cast<size_t>(k)] != QSG_OK) {
      if (rcs[static_cast<size_t>(k)] >= 1 && rcs[static_cast<size_t>(k)] <= 12)
        throw Error(static_cast<ErrorCode>(rcs[static_cast<size_t>(k)] - 1), errs[static_cast<size_t>(k)]);
      {
        const std::string& m = errs[static_cast<size_t>(k)];
        throw std::runtime_error(m.rfind("qsim device error", 0) == 0 ? m : "qsim device error: " + m);
      }
    }
  TrajectoryEnsembleResult r;  // run_ensemble bookkeeping (trajectories.cpp:60-91)
  r.times.assign(tlist.begin(), tlist.end());
  r.ntraj = static_cast<int>(ntraj);
  r.master_seed = ens.seed;
  for (double ms : dev_ms) r.device_ms = std::max(r.device_ms, ms);
  std::vector<DenseMatrix> mats(fetch_per ? static_cast<size_t>(ntraj) : 0);
  std::vector<const DenseMatrix*> ok;
  long n_ok = 0;
  for (long i = 0; i < ntraj; ++i) {
    if (failed[static_cast<size_t>(i)]) {
      ++r.failed_trajectories;
      r.stats.warnings.push_back("trajectory " + std::to_string(i) + " failed: IntegrationFailure");
      continue;
    }
    ++n_ok;
    if (fetch_per) {
      DenseMatrix m(ne, nt);
      std::copy(per.begin() + i * blk, per.begin() + (i + 1) * blk, m.data());
      mats[static_cast<size_t>(i)] = std::move(m);
      ok.push_back(&mats[static_cast<size_t>(i)]);
    }
    r.traj_indices.push_back(static_cast<int>(i));
    r.stats.steps += tstats[static_cast<size_t>(3 * i)];
    r.stats.rejected += tstats[static_cast<size_t>(3 * i + 1)];
    r.stats.rhs_evals += tstats[static_cast<size_t>(3 * i + 2)];
  }
  require(n_ok > 0, ErrorCode::EnsembleFailure, "every trajectory failed");
  r.mean_expect = DenseMatrix(ne, nt);
  if (blk > 0) {
    std::vector<Complex> mean(static_cast<size_t>(blk));
    if (nd == 1) {
      // the device bracket over the block's completed list is the reference's pairwise_sum
      for (long i = 0; i < blk; ++i) mean[static_cast<size_t>(i)] = bsum[static_cast<size_t>(i)] / Complex(static_cast<double>(n_ok), 0.0);
    } else if (r.failed_trajectories == 0) {
      // every shard's leaves are whole bracket subtrees: combine them (NCCL-gathered when a
      // communicator exists, else straight from the shard threads)
      std::vector<int64_t> lb, le;
      std::vector<Complex> sums;
      for (int k = 0; k < nd; ++k) {
        const EnsembleShard& sh = shards[static_cast<size_t>(k)];
        const Complex* src = leaf_sums[static_cast<size_t>(k)].data();
        if (!comms.empty()) src = gathered[0].data() + static_cast<size_t>(gcount / 2 * k) + 2;
        for (size_t j = 0; j < sh.leaves.size(); ++j) {
          lb.push_back(sh.leaves[j].first);
          le.push_back(sh.leaves[j].second);
          sums.insert(sums.end(), src + j * blk, src + (j + 1) * blk);
        }
      }
      check(qsg_ensemble_combine(static_cast<int32_t>(lb.size()), lb.data(), le.data(),
                                 reinterpret_cast<const double*>(sums.data()), blk, n_ok,
                                 reinterpret_cast<double*>(mean.data())));
    } else {
      // failures shift the bracket over the completed list: the host pairwise over all shards
      DenseMatrix tot = pairwise_sum(ok, 0, ok.size());
      for (long i = 0; i < blk; ++i) mean[static_cast<size_t>(i)] = tot.data()[i] / Complex(static_cast<double>(n_ok), 0.0);
    }
    std::copy(mean.begin(), mean.end(), r.mean_expect.data());
  }
  for (int i : r.traj_indices) {
    std::vector<JumpEvent> jr;
    const int cnt = jcount[static_cast<size_t>(i)];
    if (cnt > kJumpCap) {
      // more jumps than the batch buffers hold: re-run trajectory i alone (it always uses
      // RngStream(seed, i), so the re-run is the same trajectory) with room for every jump, as the
      // reference keeps the whole list (trajectories.cpp:189-200)
      std::vector<double> t1(static_cast<size_t>(cnt));
      std::vector<int32_t> c1(static_cast<size_t>(cnt));
      std::vector<Complex> p1(static_cast<size_t>(std::max<long>(1, blk))), b1(p1.size());
      int32_t f1 = 0, n1 = 0;
      double ft1 = 0.0;
      int64_t ok1 = 0, st1[3] = {0, 0, 0};
      qsg_mc_out out{};
      out.per_traj_expect = reinterpret_cast<double*>(p1.data());
      out.block_sum = reinterpret_cast<double*>(b1.data());
      out.n_ok = &ok1;
      out.failed = &f1;
      out.fail_time = &ft1;
      out.traj_stats = st1;
      out.jump_count = &n1;
      out.jump_time = t1.data();
      out.jump_channel = c1.data();
      out.jump_capacity = cnt;
      qsg_ctx* ctx = device_ctx(devs[0]);
      DeviceGenerator gen(ctx, heff, Complex(0, -1));
      check(qsg_mcsolve(ctx, &gen.g, static_cast<int32_t>(cv.size()), cv.data(), static_cast<int32_t>(ne), ev.data(),
                        psi0.dim(), reinterpret_cast<const double*>(y0.data()), tlist.data(), nt, params.data(),
                        static_cast<int32_t>(params.size()), ens.seed, i, i + 1, &o, &out, nullptr));
      require(n1 == cnt, ErrorCode::EnsembleFailure, "jump log re-run diverged");
      for (int j = 0; j < cnt; ++j) jr.push_back({t1[static_cast<size_t>(j)], c1[static_cast<size_t>(j)]});
    } else {
      for (int j = 0; j < cnt; ++j)
        jr.push_back({jtime[static_cast<size_t>(i * kJumpCap + j)], jch[static_cast<size_t>(i * kJumpCap + j)]});
    }
    r.jump_records.push_back(std::move(jr));
    if (ens.store_per_traj) r.per_traj_expect.push_back(mats[static_cast<size_t>(i)]);
  }
  return r;
}

std::vector<EnsembleShard> ensemble_shards(long ntraj, int nshards) {
  // leaves: the bracket's nodes at depth D (split lo + (hi - lo)/2, trajectories.cpp:17-22), with
  // D = log2(nshards) for a power of two and 3 levels deeper otherwise, so shards stay balanced
  int D = 0;
  while ((1 << D) < nshards) ++D;
  if ((1 << D) != nshards) D += 3;
  std::vector<std::pair<long, long>> leaves;
  std::function<void(long, long, int)> rec = [&](long lo, long hi, int d) {
    if (d == 0 || hi - lo <= 1) {
      leaves.emplace_back(lo, hi);
      return;
    }
    const long mid = lo + (hi - lo) / 2;
    rec(lo, mid, d - 1);
    rec(mid, hi, d - 1);
  };
  rec(0, ntraj, D);
  std::vector<EnsembleShard> out(static_cast<size_t>(nshards));
  size_t j = 0;
  for (int k = 0; k < nshards; ++k) {
    const long target = ntraj * (k + 1) / nshards;  // cumulative trajectories at this shard's end
    EnsembleShard& sh = out[static_cast<size_t>(k)];
    sh.begin = j < leaves.size() ? leaves[j].first : ntraj;
    while (j < leaves.size() && (leaves[j].second <= target || k == nshards - 1)) sh.leaves.push_back(leaves[j++]);
    if (sh.leaves.empty() && j < leaves.size()) sh.leaves.push_back(leaves[j++]);
    sh.end = sh.leaves.empty() ? sh.begin : sh.leaves.back().second;
  }
  return out;
}

namespace {
// shared tail of ssesolve / smesolve: one device call over [0, ntraj), then the run_ensemble
// bookkeeping (trajectories.cpp:60-91) and the measurement records
TrajectoryEnsembleResult run_sde_host(bool sme, qsg_ctx* ctx, const qsg_generator* g, long d,
                                      std::span<const QuantumObject> sc_ops, std::span<const QuantumObject> e_ops,
                                      const DenseMatrix& y0, std::span<const double> tlist, const EnsembleOptions& ens,
                                      const Params& params) {
  require(ens.ntraj >= 1, ErrorCode::InvalidGrid, "ntraj must be >= 1");
  std::vector<SparseMatrix> s_mats, e_mats;
  for (const auto& sop : sc_ops) s_mats.push_back(sop.sparse_matrix());
  for (const auto& e : e_ops) e_mats.push_back(e.sparse_matrix());
  std::vector<qsg_csr> sv, ev;
  for (const auto& m : s_mats) sv.push_back(csr_view(m));
  for (const auto& m : e_mats) ev.push_back(csr_view(m));
  const long ne = static_cast<long>(e_ops.size()), nt = static_cast<long>(tlist.size()), ntraj = ens.ntraj;
  const long blk = ne * nt, nch = static_cast<long>(sc_ops.size());
  // Euler-Maruyama grid size for the record buffers (make_em_grid, trajectories.cpp:261-275)
  const double span = tlist.back() - tlist.front(), spacing = tlist[1] - tlist[0];
  const double dtm = ens.dt_max <= 0.0 ? span / 1e4 : ens.dt_max;
  const long n_steps = std::max(1L, static_cast<long>(std::ceil(spacing / dtm * (1.0 - 1e-12)))) * (nt - 1);
  std::vector<Complex> per(static_cast<size_t>(ntraj * blk)), bsum(static_cast<size_t>(std::max<long>(1, blk)));
  const bool rec = ens.store_measurement && nch > 0;
  std::vector<double> wi, we, wc;
  if (rec) {
    wi.resize(static_cast<size_t>(ntraj * nch * n_steps));
    we.resize(wi.size());
    wc.resize(wi.size());
  }
  qsg_sde_out out{};
  out.per_traj_expect = reinterpret_cast<double*>(per.data());
  out.block_sum = reinterpret_cast<double*>(bsum.data());
  out.w_increments = rec ? wi.data() : nullptr;
  out.w_expectation = rec ? we.data() : nullptr;
  out.w_current = rec ? wc.data() : nullptr;
  qsg_timing tm{};
  auto fn = sme ? qsg_smesolve : qsg_ssesolve;
  check(fn(ctx, g, d, static_cast<int32_t>(nch), sv.data(), static_cast<int32_t>(ne), ev.data(),
           reinterpret_cast<const double*>(y0.data()), tlist.data(), nt, params.data(),
           static_cast<int32_t>(params.size()), ens.seed, 0, ntraj, ens.dt_max, rec ? 1 : 0, &out, &tm));
  TrajectoryEnsembleResult r;
  r.times.assign(tlist.begin(), tlist.end());
  r.ntraj = static_cast<int>(ntraj);
  r.master_seed = ens.seed;
  r.device_ms = tm.kernel_ms;
  std::vector<DenseMatrix> mats(static_cast<size_t>(ntraj));
  std::vector<const DenseMatrix*> ok;
  for (long i = 0; i < ntraj; ++i) {
    DenseMatrix m(ne, nt);
    std::copy(per.begin() + i * blk, per.begin() + (i + 1) * blk, m.data());
    mats[static_cast<size_t>(i)] = std::move(m);
    ok.push_back(&mats[static_cast<size_t>(i)]);
    r.traj_indices.push_back(static_cast<int>(i));
    r.stats.steps += out.n_steps;      // ode_stats.steps = rhs_evals = n_steps (:359-360)
    r.stats.rhs_evals += out.n_steps;
  }
  r.mean_expect = pairwise_sum(ok, 0, ok.size());
  for (long i = 0; i < r.mean_expect.size(); ++i)
    r.mean_expect.data()[i] = r.mean_expect.data()[i] / Complex(static_cast<double>(ok.size()), 0.0);
  for (long i = 0; i < ntraj; ++i) {
    r.jump_records.emplace_back();
    if (ens.store_per_traj) r.per_traj_expect.push_back(mats[static_cast<size_t>(i)]);
    if (rec) {
      WienerRecord w;
      w.dt = out.dt;
      w.n_channels = nch;
      w.n_steps = out.n_steps;
      const size_t o = static_cast<size_t>(i * nch * out.n_steps), len = static_cast<size_t>(nch * out.n_steps);
      w.increments.assign(wi.begin() + o, wi.begin() + o + len);
      w.expectation.assign(we.begin() + o, we.begin() + o + len);
      w.current.assign(wc.begin() + o, wc.begin() + o + len);
      r.measurement.push_back(std::move(w));
    }
  }
  return r;
}
}  // namespace

TrajectoryEnsembleResult ssesolve(const TimeDependentOperator& h, const QuantumObject& psi0,
                                  std::span<const double> tlist, std::span<const QuantumObject> sc_ops,
                                  std::span<const QuantumObject> e_ops, const EnsembleOptions& ens,
                                  const Params& params, const SolveOptions& options) {
  check_tlist(tlist);  // trajectories.cpp:367-393
  require(psi0.is_ket(), ErrorCode::KindMismatch, "ssesolve expects a Ket initial state");
  require(h.kind() == Kind::Operator, ErrorCode::KindMismatch, "ssesolve expects an Operator H");
  require(h.dims() == psi0.dims(), ErrorCode::DimsMismatch, "H and psi0 dims differ");
  for (const auto& s : sc_ops) require(s.dims() == psi0.dims(), ErrorCode::DimsMismatch, "sc_op dims mismatch");
  qsg_ctx* ctx = device_ctx(ens.devices.empty() ? options.device : ens.devices.front());
  DeviceGenerator gen(ctx, h, Complex(0, -1));
  return run_sde_host(false, ctx, &gen.g, psi0.dim(), sc_ops, e_ops, psi0.dense_matrix(), tlist, ens, params);
}

TrajectoryEnsembleResult smesolve(const TimeDependentOperator& h, const QuantumObject& rho0_in,
                                  std::span<const double> tlist, std::span<const QuantumObject> c_ops,
                                  std::span<const QuantumObject> sc_ops, std::span<const QuantumObject> e_ops,
                                  const EnsembleOptions& ens, const Params& params, const SolveOptions& options) {
  check_tlist(tlist);  // trajectories.cpp:474-503
  require(h.kind() == Kind::Operator, ErrorCode::KindMismatch, "smesolve expects an Operator H");
  QuantumObject rho0 = rho0_in.is_ket() ? ket2dm(rho0_in) : rho0_in;
  require(rho0.is_operator(), ErrorCode::KindMismatch, "smesolve expects a Ket or Operator state");
  require(rho0.dims() == h.dims(), ErrorCode::DimsMismatch, "H and rho0 dims differ");
  std::vector<QuantumObject> all_ops(c_ops.begin(), c_ops.end());
  all_ops.insert(all_ops.end(), sc_ops.begin(), sc_ops.end());
  for (const auto& c : all_ops)
    require(c.dims() == h.dims(), ErrorCode::DimsMismatch, "liouvillian: collapse dims mismatch");
  require(all_ops.size() <= 32, ErrorCode::TooLarge, "smesolve supports at most 32 channels");
  qsg_ctx* ctx = device_ctx(ens.devices.empty() ? options.device : ens.devices.front());
  // L = liouvillian(h, c_ops + sc_ops) assembled on the device, td terms as in mesolve
  DeviceGenerator gen;
  const SparseMatrix h0 = h.constant().sparse_matrix();
  const qsg_csr hv = csr_view(h0);
  std::vector<SparseMatrix> cm;
  for (const auto& c : all_ops) cm.push_back(c.sparse_matrix());
  std::vector<qsg_csr> cv;
  for (const auto& m : cm) cv.push_back(csr_view(m));
  qsg_op* op = nullptr;
  check(qsg_liouvillian_create(ctx, h.constant().dim(), &hv, static_cast<int32_t>(cv.size()), cv.data(), &op));
  gen.adopt(op, qsg_coeff{QSG_COEFF_CONST, 0, 0, 1.0, 0.0});
  for (const auto& t : h.terms()) {
    require(t.coeff.kind() != Coeff::Kind::HostOnly, ErrorCode::InvalidGrid,
            "time-dependent coefficient is a host function; the device solvers accept "
            "qsim::Coeff::constant/param/param_cos/param_sin");
    const SparseMatrix tm = t.op.sparse_matrix();
    const qsg_csr tv = csr_view(tm);
    qsg_op* top = nullptr;
    check(qsg_liouvillian_create(ctx, h.constant().dim(), &tv, 0, nullptr, &top));
    gen.adopt(top, qsg_coeff{static_cast<int32_t>(t.coeff.kind()), t.coeff.i(), t.coeff.j(), t.coeff.value().real(),
                             t.coeff.value().imag()});
  }
  return run_sde_host(true, ctx, &gen.g, rho0.dim(), sc_ops, e_ops, rho0.dense_matrix(), tlist, ens, params);
}

std::vector<double> ensemble_stddev(const TrajectoryEnsembleResult& r) {  // trajectories.cpp:94-104
  require(!r.per_traj_expect.empty(), ErrorCode::InvalidGrid, "per-trajectory data was not stored");
  const size_t sz = static_cast<size_t>(r.mean_expect.size());
  const double n = static_cast<double>(r.per_traj_expect.size());
  std::vector<double> acc(sz, 0.0);
  for (const auto& m : r.per_traj_expect)
    for (size_t i = 0; i < sz; ++i) {
      const double dl = m.data()[i].real() - r.mean_expect.data()[i].real();
      acc[i] += dl * dl;
    }
  if (n > 1)
    for (auto& a : acc) a /= (n - 1);
  for (auto& a : acc) a = std::sqrt(a);
  return acc;
}

// ---- RngStream (rng.cpp:14-47) --------------------------------------------------------------------
namespace {
inline std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
std::uint64_t splitmix(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
}  // namespace
RngStream::RngStream(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t z = seed ^ ((stream + 1) * 0x9E3779B97F4A7C15ULL);
  for (auto& w : s_) w = splitmix(z);
  if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = 1;
}
std::uint64_t RngStream::next_u64() {
  const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}
double RngStream::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double RngStream::uniform_pos() {
  double u = uniform();
  while (u == 0.0) u = uniform();
  return u;
}

}  // namespace qsim
