// Model assembly for the BASELINE configurations through the qsim host API, and its C-ABI
// (include/qsg_model.h). Assembly mirrors scenario.cpp:247-395 and the reference test fixtures.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/qsg_model.h"
#include "../../../include/qsim/evolve.hpp"

namespace qsg {
void set_error(const std::string& msg);  // qsg_capi.cu: backs qsg_last_error()
}

struct qsg_model {
  std::string name;
  qsim::TimeDependentOperator h;
  std::vector<qsim::QuantumObject> c_ops, e_ops;
  qsim::QuantumObject psi0;
  qsim::Params params;
};

namespace {

using namespace qsim;

qsg_status fail(const std::exception& e) {
  qsg::set_error(e.what());
  if (auto* qe = dynamic_cast<const Error*>(&e)) return static_cast<qsg_status>(1 + static_cast<int>(qe->code()));
  return QSG_CUDA_ERROR;
}

qsg_model* build(const std::string& name, const double* p, int np) {
  auto P = [&](int i) {
    require(i < np, ErrorCode::InvalidScenario, "model " + name + ": missing parameter");
    return p[i];
  };
  auto m = std::make_unique<qsg_model>();
  m->name = name;
  if (name == "kerr") {
    const int n = static_cast<int>(P(0));
    const double delta = P(1), u = P(2), f = P(3), gamma = P(4);
    QuantumObject a = destroy(n);
    m->h = delta * (dag(a) * a) + u * (dag(a) * dag(a) * a * a) + f * (a + dag(a));
    m->c_ops = {std::sqrt(gamma) * a};
    m->psi0 = fock(n, 0);
    m->e_ops = {dag(a) * a, a};
  } else if (name == "coupled_kerr") {
    const int n = static_cast<int>(P(0));
    const double u = P(1), j = P(2), gamma = P(3);
    QuantumObject a1 = tensor(destroy(n), qeye(n));
    QuantumObject a2 = tensor(qeye(n), destroy(n));
    QuantumObject h0 = u * (dag(a1) * dag(a1) * a1 * a1) + u * (dag(a2) * dag(a2) * a2 * a2) +
                       j * (dag(a1) * a2 + dag(a2) * a1);
    m->h = TimeDependentOperator(h0);
    m->h.add_term(dag(a1) * a1 + dag(a2) * a2, Coeff::param(0));
    m->h.add_term((a1 + dag(a1)) + (a2 + dag(a2)), Coeff::param(1));
    m->c_ops = {std::sqrt(gamma) * a1, std::sqrt(gamma) * a2};
    m->psi0 = tensor(fock(n, 0), fock(n, 0));
    m->e_ops = {dag(a1) * a1, dag(a2) * a2};
    m->params = {0.0, 0.0};
  } else if (name == "ising") {
    const int nx = static_cast<int>(P(0)), ny = static_cast<int>(P(1));
    auto [h, c] = ising_model_uncapped(nx, ny, P(2), P(3), P(4), P(5) != 0.0);
    Dims dims(static_cast<size_t>(nx * ny), 2);
    m->h = h;
    m->c_ops = c;
    QuantumObject up = basis(2, 0);  // scenario.cpp:379-382
    QuantumObject psi = up;
    for (int i = 1; i < nx * ny; ++i) psi = tensor(psi, up);
    m->psi0 = psi;
    auto total = [&](const QuantumObject& op) {  // scenario.cpp:383-392
      QuantumObject sum = embed_site(dims, 0, op);
      for (int i = 1; i < nx * ny; ++i) sum = sum + embed_site(dims, i, op);
      return sum;
    };
    m->e_ops = {total(sigmax()), total(sigmay()), total(sigmaz())};
  } else if (name == "jc") {
    const int n = static_cast<int>(P(0));
    const double wc = P(1), wa = P(2), g = P(3), kappa = P(4), gamma = P(5);
    QuantumObject a = tensor(destroy(n), qeye(2));
    QuantumObject sz = tensor(qeye(n), sigmaz());
    QuantumObject sm = tensor(qeye(n), sigmam());
    QuantumObject sp = tensor(qeye(n), sigmap());
    m->h = wc * (dag(a) * a) + (wa / 2.0) * sz + g * (a * sp + dag(a) * sm);
    m->psi0 = tensor(fock(n, 0), basis(2, 0));
    if (kappa > 0.0 || gamma > 0.0) m->c_ops = {std::sqrt(kappa) * a, std::sqrt(gamma) * sm};
    m->e_ops = {dag(a) * a, sz};
  } else if (name == "jc_sse" || name == "jc_sme") {  // scenario.cpp:252-277 (stochastic solvers)
    const int n = static_cast<int>(P(0));
    const double wc = P(1), wa = P(2), g = P(3), kappa = P(4);
    QuantumObject a = tensor(destroy(n), qeye(2));
    QuantumObject sz = tensor(qeye(n), sigmaz());
    QuantumObject sm = tensor(qeye(n), sigmam());
    QuantumObject sp = tensor(qeye(n), sigmap());
    m->h = wc * (dag(a) * a) + (wa / 2.0) * sz + g * (a * sp + dag(a) * sm);
    m->psi0 = tensor(fock(n, 0), basis(2, 0));
    if (name == "jc_sse") m->c_ops = {std::sqrt(kappa) * a};
    else m->c_ops = {std::sqrt(P(5)) * sm, std::sqrt(P(6)) * (dag(a) * a), std::sqrt(kappa) * a};
    m->e_ops = {dag(a) * a, sz, std::sqrt(kappa) * (a + dag(a))};
  } else if (name == "damped_cavity") {
    const int n = static_cast<int>(P(0));
    QuantumObject a = destroy(n);
    m->h = P(1) * (dag(a) * a);
    m->c_ops = {std::sqrt(P(2)) * a};
    m->psi0 = fock_dm(n, static_cast<int>(P(3)));
    m->e_ops = {dag(a) * a};
  } else if (name == "decay2") {
    m->h = QuantumObject(DenseMatrix::Zero(2, 2), Kind::Operator, Dims{2});
    m->c_ops = {std::sqrt(P(0)) * sigmam()};
    m->psi0 = basis(2, 0);
    m->e_ops = {sigmaz()};
  } else if (name == "driven_cavity_td") {
    const int n = static_cast<int>(P(0));
    QuantumObject a = destroy(n);
    m->h = TimeDependentOperator(0.0 * num(n));
    m->h.add_term(a + dag(a), Coeff::param_cos(0, 1));
    m->c_ops = {std::sqrt(P(1)) * a};
    m->psi0 = fock_dm(n, 0);
    m->e_ops = {a};
    m->params = {0.25, 1.3};
  } else {
    throw_error(ErrorCode::InvalidScenario, "unknown model " + name);
  }
  return m.release();
}

SparseMatrix pick(const qsg_model& m, int which, int k) {
  switch (which) {
    case QSG_SEL_H_CONST: return m.h.constant().sparse_matrix();
    case QSG_SEL_H_TERM: return m.h.terms()[static_cast<size_t>(k)].op.sparse_matrix();
    case QSG_SEL_C_OP: return m.c_ops.at(static_cast<size_t>(k)).sparse_matrix();
    case QSG_SEL_E_OP: return m.e_ops.at(static_cast<size_t>(k)).sparse_matrix();
    case QSG_SEL_L_CONST: return liouvillian(m.h.constant(), m.c_ops).sparse_matrix();
    case QSG_SEL_L_TERM: {
      const QuantumObject& op = m.h.terms()[static_cast<size_t>(k)].op;
      return (Complex(0, -1) * (spre(op) - spost(op))).sparse_matrix();
    }
    case QSG_SEL_MC_GEN: {
      QuantumObject heff = m.h.constant();
      for (const auto& c : m.c_ops) heff = heff + Complex(0, -0.5) * (dag(c) * c);
      return (Complex(0, -1) * heff).sparse_matrix();
    }
    case QSG_SEL_MC_TERM: return (Complex(0, -1) * m.h.terms()[static_cast<size_t>(k)].op).sparse_matrix();
    case QSG_SEL_SE_GEN: return (Complex(0, -1) * m.h.constant()).sparse_matrix();
  }
  throw_error(ErrorCode::InvalidIndex, "bad export selector");
}

SolveOptions from_opts(const qsg_solve_opts* o) {
  SolveOptions s;
  if (!o) return s;
  s.abstol = o->abstol;
  s.reltol = o->reltol;
  s.dt_fixed = o->dt_fixed;
  s.store_states = o->store_states != 0;
  if (o->n_saveat > 0) s.saveat = std::vector<double>(o->saveat, o->saveat + o->n_saveat);
  s.max_steps = static_cast<long>(o->max_steps);
  s.method = o->method == 1 ? SolveOptions::Method::FixedRK4 : SolveOptions::Method::AdaptiveRK45;
  return s;
}

}  // namespace

extern "C" {

qsg_status qsg_model_create(const char* name, const double* p, int32_t n_p, qsg_model** out) {
  try {
    *out = build(name, p, n_p);
    return QSG_OK;
  } catch (const std::exception& e) {
    *out = nullptr;
    return fail(e);
  }
}

void qsg_model_destroy(qsg_model* m) { delete m; }

qsg_status qsg_model_info(const qsg_model* m, int64_t* info) {
  info[0] = m->psi0.dim();
  info[1] = static_cast<int64_t>(m->h.terms().size());
  info[2] = static_cast<int64_t>(m->c_ops.size());
  info[3] = static_cast<int64_t>(m->e_ops.size());
  info[4] = m->psi0.is_ket() ? 1 : 0;
  info[5] = static_cast<int64_t>(m->params.size());
  return QSG_OK;
}

int64_t qsg_model_export(qsg_model* m, int32_t which, int32_t k, int64_t* n_rows, int32_t* rowptr, int32_t* col,
                         double* val) {
  try {
    SparseMatrix s = pick(*m, which, k);
    if (n_rows) *n_rows = s.rows;
    if (rowptr) {
      std::memcpy(rowptr, s.rowptr.data(), s.rowptr.size() * sizeof(int32_t));
      std::memcpy(col, s.col.data(), s.col.size() * sizeof(int32_t));
      std::memcpy(val, s.val.data(), s.val.size() * sizeof(Complex));
    }
    return s.nonZeros();
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

qsg_status qsg_model_psi0(const qsg_model* m, double* out) {
  const DenseMatrix d = m->psi0.dense_matrix();
  std::memcpy(out, d.data(), static_cast<size_t>(d.size()) * sizeof(Complex));
  return QSG_OK;
}

qsg_status qsg_model_default_params(const qsg_model* m, double* out) {
  for (size_t i = 0; i < m->params.size(); ++i) out[i] = m->params[i];
  return QSG_OK;
}

static qsg_status model_solve(bool me, qsg_model* m, int32_t device, const double* tlist, int64_t n_t,
                              const double* params, int32_t n_params, const qsg_solve_opts* opts, double* expect,
                              int64_t* stats, double* device_ms) {
  try {
    SolveOptions o = from_opts(opts);
    o.device = device;
    Params prm = n_params > 0 ? Params(params, params + n_params) : m->params;
    std::span<const double> tl(tlist, static_cast<size_t>(n_t));
    SolveResult r = me ? mesolve(m->h, m->psi0, tl, m->c_ops, m->e_ops, prm, o)
                       : sesolve(m->h, m->psi0, tl, m->e_ops, prm, o);
    if (expect) std::memcpy(expect, r.expect.data(), static_cast<size_t>(r.expect.size()) * sizeof(Complex));
    if (stats) {
      stats[0] = r.stats.steps;
      stats[1] = r.stats.rejected;
      stats[2] = r.stats.rhs_evals;
    }
    if (device_ms) *device_ms = r.device_ms;
    return QSG_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

qsg_status qsg_model_mesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t, const double* params,
                             int32_t n_params, const qsg_solve_opts* opts, double* expect, int64_t* stats,
                             double* device_ms) {
  return model_solve(true, m, device, tlist, n_t, params, n_params, opts, expect, stats, device_ms);
}

qsg_status qsg_model_sesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t, const double* params,
                             int32_t n_params, const qsg_solve_opts* opts, double* expect, int64_t* stats,
                             double* device_ms) {
  return model_solve(false, m, device, tlist, n_t, params, n_params, opts, expect, stats, device_ms);
}

qsg_status qsg_model_mcsolve(qsg_model* m, int32_t n_devices, const int32_t* devices, const double* tlist,
                             int64_t n_t, const double* params, int32_t n_params, uint64_t seed, int32_t ntraj,
                             const qsg_solve_opts* opts, double* mean, double* per_traj, int64_t* traj_stats,
                             int32_t* n_jumps, double* jump_time, int32_t* jump_channel, int32_t jump_cap,
                             int32_t* n_failed, double* device_ms, double* stddev) {
  try {
    SolveOptions o = from_opts(opts);
    EnsembleOptions ens;
    ens.ntraj = ntraj;
    ens.seed = seed;
    ens.store_per_traj = true;
    if (n_devices > 0) ens.devices.assign(devices, devices + n_devices);
    Params prm = n_params > 0 ? Params(params, params + n_params) : m->params;
    TrajectoryEnsembleResult r = mcsolve(m->h, m->psi0, std::span<const double>(tlist, static_cast<size_t>(n_t)),
                                         m->c_ops, m->e_ops, ens, prm, o);
    if (mean) std::memcpy(mean, r.mean_expect.data(), static_cast<size_t>(r.mean_expect.size()) * sizeof(Complex));
    const size_t blk = static_cast<size_t>(r.mean_expect.size());
    for (size_t q = 0; q < r.traj_indices.size(); ++q) {
      const int i = r.traj_indices[q];
      if (per_traj) std::memcpy(per_traj + 2 * blk * static_cast<size_t>(i), r.per_traj_expect[q].data(), blk * sizeof(Complex));
      if (n_jumps) n_jumps[i] = static_cast<int32_t>(r.jump_records[q].size());
      for (size_t j = 0; j < r.jump_records[q].size() && static_cast<int>(j) < jump_cap; ++j) {
        if (jump_time) jump_time[static_cast<size_t>(i) * jump_cap + j] = r.jump_records[q][j].time;
        if (jump_channel) jump_channel[static_cast<size_t>(i) * jump_cap + j] = r.jump_records[q][j].channel;
      }
    }
    if (traj_stats) {
      traj_stats[0] = r.stats.steps;
      traj_stats[1] = r.stats.rejected;
      traj_stats[2] = r.stats.rhs_evals;
    }
    if (n_failed) *n_failed = r.failed_trajectories;
    if (device_ms) *device_ms = r.device_ms;
    if (stddev) {  // trajectories.cpp:94-104
      const std::vector<double> sd = ensemble_stddev(r);
      std::memcpy(stddev, sd.data(), sd.size() * sizeof(double));
    }
    return QSG_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static qsg_status model_sde(qsg_model* m, bool sme, int32_t device, int32_t n_det, const double* tlist, int64_t n_t,
                            const double* params, int32_t n_params, uint64_t seed, int32_t ntraj, double dt_max,
                            int32_t store, double* mean, double* per_traj, double* wi, double* we, double* wc,
                            int64_t* n_steps, double* dt, double* device_ms) {
  try {
    SolveOptions o;
    o.device = device;
    EnsembleOptions ens;
    ens.ntraj = ntraj;
    ens.seed = seed;
    ens.dt_max = dt_max;
    ens.store_measurement = store != 0;
    Params prm = n_params > 0 ? Params(params, params + n_params) : m->params;
    std::span<const double> tl(tlist, static_cast<size_t>(n_t));
    TrajectoryEnsembleResult r;
    if (!sme) {
      r = ssesolve(m->h, m->psi0, tl, m->c_ops, m->e_ops, ens, prm, o);
    } else {
      const size_t nd = static_cast<size_t>(std::clamp<int32_t>(n_det, 0, static_cast<int32_t>(m->c_ops.size())));
      std::span<const QuantumObject> all(m->c_ops);
      r = smesolve(m->h, m->psi0, tl, all.subspan(0, nd), all.subspan(nd), m->e_ops, ens, prm, o);
    }
    if (mean) std::memcpy(mean, r.mean_expect.data(), static_cast<size_t>(r.mean_expect.size()) * sizeof(Complex));
    const size_t blk = static_cast<size_t>(r.mean_expect.size());
    for (size_t i = 0; i < r.per_traj_expect.size(); ++i)
      if (per_traj) std::memcpy(per_traj + 2 * blk * i, r.per_traj_expect[i].data(), blk * sizeof(Complex));
    for (size_t i = 0; i < r.measurement.size(); ++i) {
      const auto& w = r.measurement[i];
      const size_t len = w.increments.size();
      if (wi) std::memcpy(wi + len * i, w.increments.data(), len * sizeof(double));
      if (we) std::memcpy(we + len * i, w.expectation.data(), len * sizeof(double));
      if (wc) std::memcpy(wc + len * i, w.current.data(), len * sizeof(double));
      if (n_steps) *n_steps = w.n_steps;
      if (dt) *dt = w.dt;
    }
    if (device_ms) *device_ms = r.device_ms;
    return QSG_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

qsg_status qsg_model_ssesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t, const double* params,
                              int32_t n_params, uint64_t seed, int32_t ntraj, double dt_max, int32_t store,
                              double* mean, double* per_traj, double* wi, double* we, double* wc, int64_t* n_steps,
                              double* dt, double* device_ms) {
  return model_sde(m, false, device, 0, tlist, n_t, params, n_params, seed, ntraj, dt_max, store, mean, per_traj, wi,
                   we, wc, n_steps, dt, device_ms);
}

qsg_status qsg_model_smesolve(qsg_model* m, int32_t device, int32_t n_det, const double* tlist, int64_t n_t,
                              const double* params, int32_t n_params, uint64_t seed, int32_t ntraj, double dt_max,
                              int32_t store, double* mean, double* per_traj, double* wi, double* we, double* wc,
                              int64_t* n_steps, double* dt, double* device_ms) {
  return model_sde(m, true, device, n_det, tlist, n_t, params, n_params, seed, ntraj, dt_max, store, mean, per_traj,
                   wi, we, wc, n_steps, dt, device_ms);
}

}  // extern "C"
