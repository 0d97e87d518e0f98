/*
 * qsg.h — C-ABI drop-in boundary of the B200 time-evolution engine (paper_2504_21440_b200).
 *
 * The reference (QuantumToolbox.jl desk-scale C++ core, /root/reference/proj/core) has no FFI:
 * its hot path is the in-process C++ API
 *   - detail::SparseGenerator{ctor, apply}          evolve.hpp:96-111, evolve.cpp:53-69
 *   - Dopri5<Rhs>{start, step, dense}               integrator.hpp:23-195
 *   - sesolve / mesolve                             evolve.hpp:81-91, evolve.cpp:191-299
 *   - mcsolve / run_ensemble / ensemble_stddev      trajectories.hpp:49-95, trajectories.cpp:11-249
 * Each entry point below replaces one of those seams with plain pointers and sizes; the C++
 * host library (include/qsim/ headers) builds operators exactly as the reference does and calls
 * these functions, so a reference user keeps the same solver API.
 *
 * Conventions (Eigen-compatible, qobj.hpp:15-19):
 *   complex values are interleaved (re, im) doubles (std::complex<double>);
 *   matrices handed back are column-major; operators are handed in as CSR with int32 indices
 *   (Eigen's default StorageIndex) and columns sorted within each row;
 *   every pointer may be host or device memory (detected through UVA); host arrays are only
 *   borrowed for the duration of the call.
 * There is no CPU fallback: without a usable sm_100 device every call returns QSG_CUDA_ERROR.
 */
#ifndef QSG_H_
#define QSG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1..12 are qsim::ErrorCode + 1 (errors.hpp:8-21); the host C++ wrapper throws
 * qsim::Error(code - 1, qsg_last_error()). */
typedef enum {
  QSG_OK = 0,
  QSG_KIND_MISMATCH = 1,
  QSG_DIMS_MISMATCH = 2,
  QSG_INVALID_SUBSYSTEM = 3,
  QSG_INVALID_DIMENSION = 4,
  QSG_INVALID_INDEX = 5,
  QSG_TOO_LARGE = 6,
  QSG_INTEGRATION_FAILURE = 7,
  QSG_ENSEMBLE_FAILURE = 8,
  QSG_STEADYSTATE_FAILURE = 9,
  QSG_DFD_OVERFLOW = 10,
  QSG_INVALID_GRID = 11,
  QSG_INVALID_SCENARIO = 12,
  QSG_CUDA_ERROR = 100,
  QSG_NCCL_ERROR = 101,
  QSG_OUT_OF_MEMORY = 102,
  QSG_UNSUPPORTED = 103
} qsg_status;

typedef struct qsg_ctx qsg_ctx; /* one device + stream + workspace cache */
typedef struct qsg_op qsg_op;   /* HBM-resident CSR operator (the operator store) */

/* Device coefficient library for TimeDependentOperator terms (evolve.hpp:13-43). A host
 * std::function CoeffFn cannot run on the GPU; these forms cover the reference's uses
 * (scenario.cpp:289-291, test_evolve.cpp:203-237) and parameter sweeps. */
typedef enum {
  QSG_COEFF_CONST = 0,     /* re + i*im                         */
  QSG_COEFF_PARAM = 1,     /* params[i]                         */
  QSG_COEFF_PARAM_COS = 2, /* params[i] * cos(params[j] * t)    */
  QSG_COEFF_PARAM_SIN = 3  /* params[i] * sin(params[j] * t)    */
} qsg_coeff_kind;

typedef struct {
  int32_t kind;
  int32_t i, j;
  double re, im;
} qsg_coeff;

/* Host CSR view (row-major, int32 indices, sorted columns; val interleaved complex). */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const int32_t* rowptr;
  const int32_t* col;
  const double* val;
} qsg_csr;

/* G(t) = A_0 + sum_{k>=1} c_k(params, t) A_k with the prefactor already folded into the
 * matrices (SparseGenerator ctor, evolve.cpp:53-61). coeffs[0] is ignored. */
typedef struct {
  int32_t n_terms;
  const qsg_op* const* ops;
  const qsg_coeff* coeffs;
} qsg_generator;

/* SolveOptions (evolve.hpp:55-64). method: 0 AdaptiveRK45 (Dormand-Prince 5(4)). */
typedef struct {
  int32_t method;
  double abstol, reltol, dt_fixed;
  int32_t store_states;
  int64_t n_saveat;
  const double* saveat;
  int64_t max_steps;
} qsg_solve_opts;

/* IntegratorStats / SolveStats counters (integrator.hpp:12-16, evolve.hpp:66-71). */
typedef struct {
  int64_t steps, rejected, rhs_evals;
} qsg_stats;

/* Per-launch device timing of the last solve (CUDA events on the solve stream). */
typedef struct {
  double kernel_ms;   /* the persistent solver kernel(s) */
  double total_ms;    /* including host<->device copies done by the call */
  int64_t attempts;   /* DP5 attempts (accepted + rejected) executed on device */
  int32_t grid_ctas;  /* CTAs cooperating on one system */
  int32_t lanes;      /* lanes per CSR row in the SpMV */
  int32_t store;      /* operator store the solver streamed: 0 plain, 1 coded, 2 key-aligned */
  int32_t engine;     /* deterministic solves: 0 cooperative grid, 1 grid launched as one cluster,
                         2 cluster-resident (state and operator in distributed shared memory) */
} qsg_timing;

/* ---- context / operator store ------------------------------------------------------- */
qsg_status qsg_ctx_create(int device, qsg_ctx** out);
void qsg_ctx_destroy(qsg_ctx* ctx);
const char* qsg_last_error(void);
/* SM count, L2 bytes and name of the context's device. */
qsg_status qsg_device_info(qsg_ctx* ctx, int* sm_count, int64_t* l2_bytes, char* name, int name_len);

/* Upload a CSR operator into HBM (evolve.cpp:53-61 materialises P*A once per solve). */
qsg_status qsg_op_create(qsg_ctx* ctx, const qsg_csr* a, qsg_op** out);
/* Frees the store stream-ordered on its context's stream. A context stays alive until its last
 * operator is destroyed, so the two may be destroyed in either order. */
void qsg_op_destroy(qsg_op* op);
int64_t qsg_op_nnz(const qsg_op* op);
int64_t qsg_op_rows(const qsg_op* op);
/* Storage of the operator store: 0 = plain SELL-32 (int32 column + complex128 value per entry),
 * 1 / 2 = dictionary-coded SELL-32 (uint8 / uint16 code into the operator's distinct
 * (column - row, value) pairs; lossless). qsg_op_dict_size: distinct pairs (0 when plain).
 * Set QSG_NO_COMPRESS=1 to force the plain store. */
int32_t qsg_op_code_bytes(const qsg_op* op);
int32_t qsg_op_dict_size(const qsg_op* op);
/* The stores an operator carries and the bytes one SpMV reads from each.
 * info[0] = store the grid engine streams (0 plain, 1/2 coded, 3 key-aligned); info[1] plain
 * bytes; info[2] coded bytes (0 if absent); info[3] key-aligned bytes (0 if absent); info[4]
 * key-aligned distinct values; info[5] key-aligned positions; info[6] coded pairs; info[7]
 * largest key-aligned slice block (bytes). The key-aligned store is built next to the coded one
 * on request (QSG_KA_STORE=1, or QSG_KA_SOLVE=1 which also makes the grid solver stream it). */
qsg_status qsg_op_store_info(const qsg_op* op, int64_t* info);

/* On-device Liouvillian assembly (superop.cpp:78-91 liouvillian, :51-76 spre/spost/sprepost/
 * lindblad_dissipator): L = -i(I(x)H - H^T(x)I) + sum_k D(c_k) for d x d CSR operators H (may be
 * NULL) and c_ops, column-stacked vectorization (superop.hpp:9-10). Values and sparsity pattern
 * (explicit zeros included) equal the reference's entry for entry. At most 32 collapse operators.
 * qsg_liouvillian_create builds the operator store from it directly; qsg_liouvillian_export copies
 * the CSR (n = d*d rows) into caller buffers (host or device; pass rowptr == NULL to query nnz). */
qsg_status qsg_liouvillian_create(qsg_ctx* ctx, int64_t d, const qsg_csr* H, int32_t n_c,
                                  const qsg_csr* c_ops, qsg_op** out);
qsg_status qsg_liouvillian_export(qsg_ctx* ctx, int64_t d, const qsg_csr* H, int32_t n_c,
                                  const qsg_csr* c_ops, int64_t* nnz, int32_t* rowptr,
                                  int32_t* col, double* val);

/* out = G(t) y  — SparseGenerator::apply (evolve.cpp:63-69). y/out: n complex. */
qsg_status qsg_generator_apply(qsg_ctx* ctx, const qsg_generator* g, const double* params,
                               int32_t n_params, double t, const double* y, double* out);
/* Same, timed: runs `reps` back-to-back launches on device buffers, returns mean ms. */
qsg_status qsg_generator_apply_timed(qsg_ctx* ctx, const qsg_generator* g, const double* params,
                                     int32_t n_params, double t, const double* y_dev,
                                     double* out_dev, int32_t reps, double* mean_ms);

/* ---- deterministic solvers ----------------------------------------------------------- */
/* mesolve on a ready Liouvillian generator L (evolve.cpp:237-299 after line 262):
 *   rho0: d x d complex column-major (ket inputs are promoted by the caller, :254);
 *   e_ops: n_e CSR operators (d x d); expect: n_e x n_t complex column-major;
 *   states: optional n_save x (d*d) hermitized states (:286, :296) — n_save is the number of
 *   save events (saveat, or tlist when store_states or n_e == 0). */
qsg_status qsg_mesolve(qsg_ctx* ctx, const qsg_generator* L, int64_t d, const double* rho0,
                       const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                       const double* params, int32_t n_params, const qsg_solve_opts* opts,
                       double* expect, double* states, qsg_stats* stats, qsg_timing* timing);

/* sesolve with generator -i*H (evolve.cpp:191-233); expect = <psi|E|psi>. */
qsg_status qsg_sesolve(qsg_ctx* ctx, const qsg_generator* G, int64_t d, const double* psi0,
                       const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                       const double* params, int32_t n_params, const qsg_solve_opts* opts,
                       double* expect, double* states, qsg_stats* stats, qsg_timing* timing);

/* ---- stochastic Schroedinger / master equations (trajectories.cpp:251-503) ------------- */
typedef struct {
  double* per_traj_expect; /* optional: n_blk x (n_e x n_t) complex, col-major blocks      */
  double* block_sum;       /* required: n_e x n_t complex, pairwise sum over the block     */
  int64_t n_ok;            /* out: trajectories in block_sum                               */
  double* w_increments;    /* optional (store_measurement): n_blk x (n_ch x n_steps) dW    */
  double* w_expectation;   /*   e_c per step                                              */
  double* w_current;       /*   J = e_c + dW / dt (trajectories.hpp:18-24)                */
  int64_t n_steps;         /* out: Euler-Maruyama steps per trajectory (make_em_grid)    */
  double dt;               /* out: step size                                              */
} qsg_sde_out;

/* ssesolve (trajectories.cpp:367-393) for trajectories [traj_begin, traj_end): G = -i H(t),
 * sc_ops d x d (S^dag S and S + S^dag are formed here in the reference's arithmetic), psi0 is
 * normalised; tlist must be uniform. Trajectory i uses RngStream(seed, i). At most 8 channels. */
qsg_status qsg_ssesolve(qsg_ctx* ctx, const qsg_generator* G, int64_t d, int32_t n_sc,
                        const qsg_csr* sc_ops, int32_t n_e, const qsg_csr* e_ops, const double* psi0,
                        const double* tlist, int64_t n_t, const double* params, int32_t n_params,
                        uint64_t seed, int64_t traj_begin, int64_t traj_end, double dt_max,
                        int32_t store_measurement, qsg_sde_out* out, qsg_timing* timing);
/* smesolve (trajectories.cpp:474-503): L = the full Liouvillian including the sc_op
 * dissipators (qsg_liouvillian_create over c_ops followed by sc_ops), rho0 d x d col-major. */
qsg_status qsg_smesolve(qsg_ctx* ctx, const qsg_generator* L, int64_t d, int32_t n_sc,
                        const qsg_csr* sc_ops, int32_t n_e, const qsg_csr* e_ops, const double* rho0,
                        const double* tlist, int64_t n_t, const double* params, int32_t n_params,
                        uint64_t seed, int64_t traj_begin, int64_t traj_end, double dt_max,
                        int32_t store_measurement, qsg_sde_out* out, qsg_timing* timing);

/* ---- Monte-Carlo trajectories (trajectories.cpp:106-249) ------------------------------ */
typedef struct {
  /* outputs, all optional (NULL to skip) except block_sum / n_ok */
  double* per_traj_expect;   /* n_blk x (n_e x n_t) complex, col-major blocks        */
  double* block_sum;         /* n_e x n_t: pairwise_sum (trajectories.cpp:17-22) over the
                                completed trajectories of [traj_begin, traj_end)      */
  int64_t* n_ok;             /* completed trajectories in the block                  */
  int32_t* failed;           /* n_blk flags (status code of the failure, 0 = ok)     */
  double* fail_time;         /* n_blk: t at failure                                  */
  int64_t* traj_stats;       /* n_blk x 3: steps, rejected, rhs_evals                */
  int32_t* jump_count;       /* n_blk                                                */
  double* jump_time;         /* n_blk x jump_capacity                                */
  int32_t* jump_channel;     /* n_blk x jump_capacity                                */
  int64_t jump_capacity;
  /* optional: pairwise_sum of each of n_ranges sub-ranges [range_lo[r], range_hi[r]) of the
   * block's completed-trajectory list (positions in that list, ascending), computed on the device;
   * range_sums: n_ranges x (n_e x n_t) complex. A rank whose trajectories are several subtrees of
   * the global bracket returns one sum per subtree (paper_2504_21440_b200/dist.py). */
  int32_t n_ranges;
  const int64_t* range_lo;
  const int64_t* range_hi;
  double* range_sums;
} qsg_mc_out;

/* Runs trajectories traj_begin..traj_end-1; trajectory i draws from RngStream(seed, i)
 * (trajectories.cpp:42), so any partition of the index range gives identical per-trajectory
 * results. G = -i*H_eff generator (trajectories.cpp:229-237), c_ops / e_ops as CSR. The ensemble
 * sums are accumulated on the device (the pairwise bracket of trajectories.cpp:17-22 over the
 * completed trajectories, bit-identical to the host recursion); per-trajectory expectations are
 * copied back only when per_traj_expect is non-NULL. */
qsg_status qsg_mcsolve(qsg_ctx* ctx, const qsg_generator* G, int32_t n_c, const qsg_csr* c_ops,
                       int32_t n_e, const qsg_csr* e_ops, int64_t d, const double* psi0,
                       const double* tlist, int64_t n_t, const double* params, int32_t n_params,
                       uint64_t seed, int64_t traj_begin, int64_t traj_end,
                       const qsg_solve_opts* opts, qsg_mc_out* out, qsg_timing* timing);

/* Deterministic ensemble combine of per-block pairwise sums whose blocks tile [0, ntraj)
 * at the top levels of the pairwise_sum bracket (trajectories.cpp:17-22,82-83):
 * mean = bracket(block_sums) / Complex(n_ok_total, 0). Host or device buffers. */
qsg_status qsg_ensemble_combine(int32_t n_blocks, const int64_t* block_begin,
                                const int64_t* block_end, const double* block_sums,
                                int64_t n_vals, int64_t n_ok_total, double* mean);

/* ---- NCCL communicators: the one exchange step of sharded ensembles ----------
 * Replaces run_ensemble's in-process combine (trajectories.cpp:31-58,82-83) when trajectories are
 * spread over GPUs. qsg_comm_init_rank: one rank per process (ncclCommInitRank; rank 0 makes the
 * id with qsg_comm_unique_id and the caller broadcasts it); qsg_comm_init_all: every device of
 * one process (ncclCommInitAll; each comm gets its own context, distinct devices only).
 * qsg_comm_allgather: recv[r*count ..] = rank r's `count` doubles (host or device buffers),
 * synchronous on the comm's context stream. NCCL is loaded at run time (the process's own copy
 * if one is already loaded); without it these return QSG_NCCL_ERROR. */
typedef struct qsg_comm qsg_comm;
int32_t qsg_nccl_version(void);
qsg_status qsg_comm_unique_id(uint8_t* id128);
qsg_status qsg_comm_init_rank(qsg_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id128,
                              qsg_comm** out);
qsg_status qsg_comm_init_all(int32_t n_dev, const int32_t* devices, qsg_comm** out);
qsg_ctx* qsg_comm_ctx(qsg_comm* comm);
void qsg_comm_destroy(qsg_comm* comm);
qsg_status qsg_comm_allgather(qsg_comm* comm, const double* send, int64_t count, double* recv);

/* ---- parameter sweeps (a14: one mesolve per parameter point) ---------------------------- */
/* n_points independent mesolve runs of the same td Liouvillian with per-point params
 * (point p uses params[p*n_params .. ]); expect: n_points x (n_e x n_t). */
qsg_status qsg_mesolve_batch(qsg_ctx* ctx, const qsg_generator* L, int64_t d, const double* rho0,
                             const double* tlist, int64_t n_t, int32_t n_e, const qsg_csr* e_ops,
                             int64_t n_points, const double* params, int32_t n_params,
                             const qsg_solve_opts* opts, double* expect, qsg_stats* stats,
                             int32_t* status, qsg_timing* timing);

/* ---- RNG (rng.cpp) on device, for parity checks ------------------------------------------ */
/* kind 0: next_u64, 1: uniform, 2: uniform_pos; n draws of stream (seed, stream). */
qsg_status qsg_rng_draw(qsg_ctx* ctx, uint64_t seed, uint64_t stream, int32_t kind, int32_t n,
                        double* out_d, uint64_t* out_u);

#ifdef __cplusplus
}
#endif

#endif /* QSG_H_ */
