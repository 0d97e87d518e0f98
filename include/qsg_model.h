/*
 * qsg_model.h — C-ABI over the qsim C++ host API (include/qsim/ headers) for the model
 * configurations of BASELINE.json, assembled the way the reference's scenario runner does
 * (scenario.cpp:247-395): H, c_ops, e_ops and the initial state are built with the factory /
 * tensor / dag / arithmetic functions, Liouvillians with liouvillian() (superop.cpp:78-91).
 *
 * Models (parameters in order):
 *   "kerr"             N, Delta, U, F, gamma        H = D a^+a + U a^+a^+aa + F(a + a^+), c = sqrt(g) a
 *   "coupled_kerr"     N, U, J, gamma ; params (Delta, F) as PARAM terms (sweep configuration)
 *   "ising"            nx, ny, Jz, hx, gamma, periodic   (factories.cpp:204-246, no 12-site cap)
 *   "jc"               N, wc, wa, g, kappa, gamma   (test_evolve.cpp:16-28)
 *   "damped_cavity"    N, omega, gamma, n0          (test_evolve.cpp:124-140)
 *   "decay2"           gamma                        (test_trajectories.cpp:40-88)
 *   "driven_cavity_td" N, gamma ; params (F, wd) as PARAM_COS term (test_evolve.cpp:203-237)
 */
#ifndef QSG_MODEL_H_
#define QSG_MODEL_H_

#include <stdint.h>

#include "qsg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsg_model qsg_model;

enum {
  QSG_SEL_H_CONST = 0,  /* H constant part                                   */
  QSG_SEL_H_TERM = 1,   /* H term k                                          */
  QSG_SEL_C_OP = 2,     /* collapse operator k                               */
  QSG_SEL_E_OP = 3,     /* expectation operator k                            */
  QSG_SEL_L_CONST = 4,  /* liouvillian(H const, c_ops)                       */
  QSG_SEL_L_TERM = 5,   /* -i(spre(H_k) - spost(H_k))                        */
  QSG_SEL_MC_GEN = 6,   /* -i * H_eff, H_eff = H - i/2 sum c^+c               */
  QSG_SEL_MC_TERM = 7,  /* -i * H_k                                          */
  QSG_SEL_SE_GEN = 8    /* -i * H                                            */
};

qsg_status qsg_model_create(const char* name, const double* p, int32_t n_p, qsg_model** out);
void qsg_model_destroy(qsg_model* m);
/* info: [dim, n_terms, n_cops, n_eops, psi0_is_ket, n_params] */
qsg_status qsg_model_info(const qsg_model* m, int64_t* info);
/* CSR export; call with rowptr == NULL to query nnz / rows. Returns nnz, or -1 on error. */
int64_t qsg_model_export(qsg_model* m, int32_t which, int32_t k, int64_t* n_rows, int32_t* rowptr,
                         int32_t* col, double* val);
qsg_status qsg_model_psi0(const qsg_model* m, double* out);
qsg_status qsg_model_default_params(const qsg_model* m, double* out);

/* Full reference-API solves (qsim::mesolve / sesolve / mcsolve) on device `device`.
 * stats: steps, rejected, rhs_evals. expect: n_e x n_t col-major complex. */
qsg_status qsg_model_mesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t,
                             const double* params, int32_t n_params, const qsg_solve_opts* opts,
                             double* expect, int64_t* stats, double* device_ms);
qsg_status qsg_model_sesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t,
                             const double* params, int32_t n_params, const qsg_solve_opts* opts,
                             double* expect, int64_t* stats, double* device_ms);
/* mean: n_e x n_t; per_traj (optional): ntraj x n_e x n_t; traj_stats: ensemble totals
 * (steps, rejected, rhs_evals over completed trajectories); jump arrays
 * ntraj x jump_cap. n_devices/devices shard trajectories over several GPUs in-process (NCCL
 * all-gather of bracket-subtree sums between distinct devices). stddev (optional): n_e x n_t
 * sample standard deviation of Re over the trajectories (ensemble_stddev, trajectories.cpp:94-104). */
qsg_status qsg_model_mcsolve(qsg_model* m, int32_t n_devices, const int32_t* devices, const double* tlist,
                             int64_t n_t, const double* params, int32_t n_params, uint64_t seed,
                             int32_t ntraj, const qsg_solve_opts* opts, double* mean, double* per_traj,
                             int64_t* traj_stats, int32_t* n_jumps, double* jump_time, int32_t* jump_channel,
                             int32_t jump_cap, int32_t* n_failed, double* device_ms, double* stddev);
/* qsim::ssesolve (every model c_op is a measurement channel, as the reference scenario's
 * "ssesolve" jc assembly) / qsim::smesolve (model c_ops[0:n_det) unmonitored, the rest measured).
 * mean: n_e x n_t; per_traj (optional): ntraj x n_e x n_t; w_* (optional, store_measurement):
 * ntraj x (n_ch x n_steps); *n_steps / *dt: the Euler-Maruyama grid. */
qsg_status qsg_model_ssesolve(qsg_model* m, int32_t device, const double* tlist, int64_t n_t,
                              const double* params, int32_t n_params, uint64_t seed, int32_t ntraj,
                              double dt_max, int32_t store_measurement, double* mean, double* per_traj,
                              double* w_increments, double* w_expectation, double* w_current,
                              int64_t* n_steps, double* dt, double* device_ms);
qsg_status qsg_model_smesolve(qsg_model* m, int32_t device, int32_t n_det, const double* tlist,
                              int64_t n_t, const double* params, int32_t n_params, uint64_t seed,
                              int32_t ntraj, double dt_max, int32_t store_measurement, double* mean,
                              double* per_traj, double* w_increments, double* w_expectation,
                              double* w_current, int64_t* n_steps, double* dt, double* device_ms);

#ifdef __cplusplus
}
#endif

#endif /* QSG_MODEL_H_ */
