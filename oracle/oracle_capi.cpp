// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle for tests/ and bench.py's
// cpu_baseline leg (ctypes). Never linked by the product.
#include <cstring>
#include <memory>
#include <string>

#include "qsim_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

struct Handle {
  Model m;
  std::unique_ptr<TdOp> L;  // prebuilt Liouvillian (SuperOperator input path, evolve.cpp:244-252)
};

int fail(const std::exception& e) {
  g_err = e.what();
  if (auto* qe = dynamic_cast<const Error*>(&e)) return 1 + static_cast<int>(qe->code());
  return 100;
}

Csc pick(const Handle& h, int which, int k) {
  const Model& m = h.m;
  switch (which) {
    case 0: return m.h.constant.sparse();
    case 1: return m.h.terms.at(static_cast<size_t>(k)).op.sparse();
    case 2: return m.c_ops.at(static_cast<size_t>(k)).sparse();
    case 3: return m.e_ops.at(static_cast<size_t>(k)).sparse();
    case 4: return liouvillian(m.h.constant, m.c_ops).sparse();
    case 5: {
      const QObj& op = m.h.terms.at(static_cast<size_t>(k)).op;
      return (cd(0, -1) * (spre(op) - spost(op))).sparse();
    }
    case 6: {  // mcsolve generator: -i * H_eff (trajectories.cpp:229-237)
      QObj heff = m.h.constant;
      for (const auto& c : m.c_ops) heff = heff + cd(0, -0.5) * (dag(c) * c);
      return (cd(0, -1) * heff).sparse();
    }
    case 7: return (cd(0, -1) * m.h.terms.at(static_cast<size_t>(k)).op).sparse();
    case 8: return (cd(0, -1) * m.h.constant).sparse();  // sesolve generator
  }
  throw_error(ErrorCode::InvalidIndex, "bad export selector");
}

SolveOptions to_opts(const double* o, int n_saveat, const double* saveat) {
  SolveOptions s;
  if (o) {
    s.abstol = o[0];
    s.reltol = o[1];
    s.max_steps = static_cast<long>(o[2]);
    s.store_states = o[3] != 0.0;
  }
  if (n_saveat > 0) s.saveat = std::vector<double>(saveat, saveat + n_saveat);
  return s;
}

void write_dense(const Dense& d, double* out) {
  std::memcpy(out, d.v.data(), d.v.size() * sizeof(cd));
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

/// Worker threads for single-solve loops (bit-identical results; see qsim_oracle.hpp).
void orc_set_threads(int n) { set_threads(n); }
int orc_threads(void) { return threads(); }

void* orc_model_new(const char* name, const double* p, int np) {
  try {
    auto h = std::make_unique<Handle>();
    h->m = build_model(name, std::span<const double>(p, static_cast<size_t>(np)));
    return h.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void orc_model_free(void* h) { delete static_cast<Handle*>(h); }

long orc_model_dim(void* h) { return static_cast<Handle*>(h)->m.psi0.dim; }

int orc_model_count(void* hp, int what) {
  const Model& m = static_cast<Handle*>(hp)->m;
  switch (what) {
    case 0: return static_cast<int>(m.h.terms.size());
    case 1: return static_cast<int>(m.c_ops.size());
    case 2: return static_cast<int>(m.e_ops.size());
    case 3: return m.psi0.is_ket() ? 1 : 0;
    case 4: return static_cast<int>(m.params.size());
  }
  return -1;
}

int orc_model_default_params(void* hp, double* out) {
  const Model& m = static_cast<Handle*>(hp)->m;
  for (size_t i = 0; i < m.params.size(); ++i) out[i] = m.params[i];
  return static_cast<int>(m.params.size());
}

/// CSR export (row-major, columns sorted) of the selected operator. Returns nnz, -1 on error.
/// Call with rowptr == nullptr to query nnz / rows only.
long orc_model_export(void* hp, int which, int k, long* nrows, int* rowptr, int* col, double* val) {
  try {
    Csc c = pick(*static_cast<Handle*>(hp), which, k);
    if (nrows) *nrows = c.rows;
    if (!rowptr) return c.nnz();
    Csc t = sp_transpose(c);  // CSC of A^T == CSR of A
    std::memcpy(rowptr, t.outer.data(), t.outer.size() * sizeof(int));
    std::memcpy(col, t.inner.data(), t.inner.size() * sizeof(int));
    std::memcpy(val, t.val.data(), t.val.size() * sizeof(cd));
    return c.nnz();
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int orc_model_psi0(void* hp, double* out) {
  write_dense(static_cast<Handle*>(hp)->m.psi0.dense(), out);
  return 0;
}

/// opts = {abstol, reltol, max_steps, store_states}. expect: n_e x n_t complex col-major.
/// stats: steps, rejected, rhs_evals. states (optional): n_save x state size complex.
int orc_mesolve(void* hp, const double* tlist, int nt, const double* params, int np,
                const double* opts, int n_saveat, const double* saveat, double* expect,
                long* stats, double* states) {
  try {
    const Model& m = static_cast<Handle*>(hp)->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    SolveResult r = mesolve(m.h, m.psi0, std::span<const double>(tlist, static_cast<size_t>(nt)),
                            m.c_ops, m.e_ops, prm, to_opts(opts, n_saveat, saveat));
    write_dense(r.expect, expect);
    stats[0] = r.stats.steps;
    stats[1] = r.stats.rejected;
    stats[2] = r.stats.rhs_evals;
    if (states) {
      size_t off = 0;
      for (const auto& s : r.states) {
        Dense d = s.dense();
        std::memcpy(states + 2 * off, d.v.data(), d.v.size() * sizeof(cd));
        off += d.v.size();
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_sesolve(void* hp, const double* tlist, int nt, const double* params, int np,
                const double* opts, int n_saveat, const double* saveat, double* expect,
                long* stats, double* states) {
  try {
    const Model& m = static_cast<Handle*>(hp)->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    SolveResult r = sesolve(m.h, m.psi0, std::span<const double>(tlist, static_cast<size_t>(nt)),
                            m.e_ops, prm, to_opts(opts, n_saveat, saveat));
    write_dense(r.expect, expect);
    stats[0] = r.stats.steps;
    stats[1] = r.stats.rejected;
    stats[2] = r.stats.rhs_evals;
    if (states) {
      size_t off = 0;
      for (const auto& s : r.states) {
        Dense d = s.dense();
        std::memcpy(states + 2 * off, d.v.data(), d.v.size() * sizeof(cd));
        off += d.v.size();
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// Build and cache L = liouvillian(H, c_ops) (td terms kept) for orc_mesolve_prepared.
int orc_model_prepare_liouvillian(void* hp) {
  try {
    auto* h = static_cast<Handle*>(hp);
    h->L = std::make_unique<TdOp>(liouvillian_td(h->m.h, h->m.c_ops));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// mesolve on the cached SuperOperator (c_ops empty), i.e. the reference's solve loop without the
/// Liouvillian assembly — what the CPU baseline times.
int orc_mesolve_prepared(void* hp, const double* tlist, int nt, const double* params, int np,
                         const double* opts, double* expect, long* stats) {
  try {
    auto* h = static_cast<Handle*>(hp);
    if (!h->L) throw_error(ErrorCode::InvalidGrid, "call orc_model_prepare_liouvillian first");
    const Model& m = h->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    SolveResult r = mesolve(*h->L, m.psi0, std::span<const double>(tlist, static_cast<size_t>(nt)), {},
                            m.e_ops, prm, to_opts(opts, 0, nullptr));
    write_dense(r.expect, expect);
    stats[0] = r.stats.steps;
    stats[1] = r.stats.rejected;
    stats[2] = r.stats.rhs_evals;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// Runs trajectories 0..ntraj-1 of mcsolve (trajectory i uses RngStream(seed, i)).
/// mean: n_e x n_t complex (pairwise mean over completed trajectories).
/// per_traj (optional): ntraj x (n_e x n_t) complex; stats: ntraj x 3; njumps: ntraj;
/// jt/jc: ntraj x jcap jump times / channels; failed: ntraj flags.
int orc_mcsolve(void* hp, const double* tlist, int nt, const double* params, int np,
                const double* opts, unsigned long long seed, int ntraj, int nthreads,
                double* mean, double* per_traj, long* stats, int* njumps, double* jt, int* jc,
                int jcap, int* failed) {
  try {
    const Model& m = static_cast<Handle*>(hp)->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    EnsembleOptions ens;
    ens.ntraj = ntraj;
    ens.seed = seed;
    ens.n_threads = nthreads;
    EnsembleResult r = mcsolve(m.h, m.psi0, std::span<const double>(tlist, static_cast<size_t>(nt)),
                               m.c_ops, m.e_ops, ens, prm, to_opts(opts, 0, nullptr));
    write_dense(r.mean_expect, mean);
    const size_t blk = static_cast<size_t>(m.e_ops.size()) * static_cast<size_t>(nt);
    for (int i = 0; i < ntraj; ++i) {
      const auto& s = r.raw[static_cast<size_t>(i)];
      if (failed) failed[i] = s.failed ? 1 : 0;
      if (per_traj && !s.failed) std::memcpy(per_traj + 2 * blk * static_cast<size_t>(i), s.expect.v.data(), blk * sizeof(cd));
      if (stats) {
        stats[3 * i] = s.steps;
        stats[3 * i + 1] = s.rejected;
        stats[3 * i + 2] = s.rhs_evals;
      }
      if (njumps) njumps[i] = static_cast<int>(s.jumps.size());
      for (int j = 0; j < static_cast<int>(s.jumps.size()) && j < jcap; ++j) {
        if (jt) jt[static_cast<size_t>(i) * static_cast<size_t>(jcap) + static_cast<size_t>(j)] = s.jumps[static_cast<size_t>(j)].time;
        if (jc) jc[static_cast<size_t>(i) * static_cast<size_t>(jcap) + static_cast<size_t>(j)] = s.jumps[static_cast<size_t>(j)].channel;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// Stochastic solvers (trajectories.cpp:251-503) on a zoo model. ssesolve: every model c_op is a
/// measurement channel (sc_op). smesolve: the first n_det model c_ops are deterministic c_ops, the
/// rest sc_ops. mean: n_e x n_t; per_traj (optional): ntraj x (n_e x n_t) complex;
/// winc/wexp/wcur (optional, store_measurement): ntraj x (n_ch x n_steps) doubles;
/// *n_steps_out / *dt_out: the Euler-Maruyama grid.
static int sde_common(void* hp, int sme, int n_det, const double* tlist, int nt, const double* params, int np,
                      unsigned long long seed, int ntraj, int nthreads, double dt_max, int store_meas,
                      double* mean, double* per_traj, double* winc, double* wexp, double* wcur, long* n_steps_out,
                      double* dt_out) {
  try {
    const Model& m = static_cast<Handle*>(hp)->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    EnsembleOptions ens;
    ens.ntraj = ntraj;
    ens.seed = seed;
    ens.n_threads = nthreads;
    ens.dt_max = dt_max;
    ens.store_measurement = store_meas != 0;
    std::span<const double> tl(tlist, static_cast<size_t>(nt));
    EnsembleResult r;
    if (!sme) {
      r = ssesolve(m.h, m.psi0, tl, m.c_ops, m.e_ops, ens, prm);
    } else {
      const size_t nd = static_cast<size_t>(std::max(0, std::min<int>(n_det, static_cast<int>(m.c_ops.size()))));
      std::span<const QObj> cops(m.c_ops.data(), nd), scops(m.c_ops.data() + nd, m.c_ops.size() - nd);
      r = smesolve(m.h, m.psi0, tl, cops, scops, m.e_ops, ens, prm);
    }
    write_dense(r.mean_expect, mean);
    const EmGrid g = make_em_grid(tl, dt_max);
    if (n_steps_out) *n_steps_out = g.n_steps;
    if (dt_out) *dt_out = g.dt;
    const size_t blk = static_cast<size_t>(m.e_ops.size()) * static_cast<size_t>(nt);
    for (int i = 0; i < ntraj; ++i) {
      const auto& s = r.raw[static_cast<size_t>(i)];
      if (per_traj) std::memcpy(per_traj + 2 * blk * static_cast<size_t>(i), s.expect.v.data(), blk * sizeof(cd));
      if (s.has_wiener) {
        const size_t w = s.wiener.increments.size();
        if (winc) std::memcpy(winc + w * static_cast<size_t>(i), s.wiener.increments.data(), w * sizeof(double));
        if (wexp) std::memcpy(wexp + w * static_cast<size_t>(i), s.wiener.expectation.data(), w * sizeof(double));
        if (wcur) std::memcpy(wcur + w * static_cast<size_t>(i), s.wiener.current.data(), w * sizeof(double));
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_ssesolve(void* hp, const double* tlist, int nt, const double* params, int np, unsigned long long seed,
                 int ntraj, int nthreads, double dt_max, int store_meas, double* mean, double* per_traj,
                 double* winc, double* wexp, double* wcur, long* n_steps_out, double* dt_out) {
  return sde_common(hp, 0, 0, tlist, nt, params, np, seed, ntraj, nthreads, dt_max, store_meas, mean, per_traj,
                    winc, wexp, wcur, n_steps_out, dt_out);
}

int orc_smesolve(void* hp, int n_det, const double* tlist, int nt, const double* params, int np,
                 unsigned long long seed, int ntraj, int nthreads, double dt_max, int store_meas, double* mean,
                 double* per_traj, double* winc, double* wexp, double* wcur, long* n_steps_out, double* dt_out) {
  return sde_common(hp, 1, n_det, tlist, nt, params, np, seed, ntraj, nthreads, dt_max, store_meas, mean, per_traj,
                    winc, wexp, wcur, n_steps_out, dt_out);
}

/// out = G y for the selected generator (which = 4 Liouvillian / 6 mcsolve -iH_eff /
/// 8 sesolve -iH), including parameter terms at time t.
int orc_generator_apply(void* hp, int which, double t, const double* params, int np,
                        const double* y, double* out) {
  try {
    const Model& m = static_cast<Handle*>(hp)->m;
    Params prm = np > 0 ? Params(params, params + np) : m.params;
    TdOp op;
    cd pref(1, 0);
    if (which == 4) {
      op = liouvillian_td(m.h, m.c_ops);
    } else if (which == 6) {
      QObj heff = m.h.constant;
      for (const auto& c : m.c_ops) heff = heff + cd(0, -0.5) * (dag(c) * c);
      op = TdOp{heff, m.h.terms};
      pref = cd(0, -1);
    } else {
      op = m.h;
      pref = cd(0, -1);
    }
    SparseGenerator gen(op, pref, prm);
    const size_t n = static_cast<size_t>(gen.size());
    std::vector<cd> yy(reinterpret_cast<const cd*>(y), reinterpret_cast<const cd*>(y) + n), oo(n);
    gen.apply(t, yy, oo);
    std::memcpy(out, oo.data(), n * sizeof(cd));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// kind 0: next_u64 (out_u), 1: uniform, 2: uniform_pos, 3: normal (out_d).
void orc_rng(unsigned long long seed, unsigned long long stream, int kind, int n, double* out_d,
             unsigned long long* out_u) {
  RngStream r(seed, stream);
  for (int i = 0; i < n; ++i) {
    switch (kind) {
      case 0: out_u[i] = r.next_u64(); break;
      case 1: out_d[i] = r.uniform(); break;
      case 2: out_d[i] = r.uniform_pos(); break;
      default: out_d[i] = r.normal(); break;
    }
  }
}

unsigned long long orc_splitmix64(unsigned long long* state) {
  std::uint64_t s = *state;
  std::uint64_t r = splitmix64_next(s);
  *state = s;
  return r;
}

/// Reference ising_model with its 12-site cap (factories.cpp:208); returns error code.
int orc_ising_capped(int nx, int ny) {
  try {
    ising_model(nx, ny, 1.0, 0.2, 1.0, true, true);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
