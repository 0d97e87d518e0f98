// Host <-> device contract of the persistent grid DP5 engine (grid_engine.cu).
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace qsg {

constexpr int kMaxPending = 32;
constexpr int kObsSlots = 128;  // doubles per observation slot bank (2 banks)
enum : int { kSlotErr = 0, kSlotD0 = 1, kSlotD1 = 2, kSlotD2 = 3, kSlotObs0 = 4 };
constexpr int kNumSlots = kSlotObs0 + 2 * kObsSlots;

struct GridCtl {
  double t, h, fail_t;
  long long steps, rejected, rhs_evals, attempts;
  int status;
  int final_buf;
};

constexpr int kGridMaxSeOps = 8;  // sesolve e_ops kept as operator stores

struct GridProblem {
  int cluster;    // 1: the whole grid is one thread-block cluster (hardware cluster barriers)
  int smem_dict;  // > 0: the single-term coded generator's dictionary (entries) staged in shared memory
  int x2;         // materialise the stage-2 input (one extra pass + barrier, half the stage-2 gathers)
  int k1g;        // autonomous single-term generator: stage 2 as k1 + (h a21) G k1 (no x2 pass)
  int n;     // vector length (d*d for mesolve, d for sesolve)
  int d;     // Hilbert dimension
  DevGen gen;
  const double* params;
  double2* buf[11];
  double atol, rtol;
  long long max_steps;
  double t0, tf, eps_t;
  int n_ev;
  const double* ev_t;
  const int* ev_grid;
  const int* ev_save;
  int n_e;
  // mesolve observation: e_op entries in CSC order, concatenated (evolve.cpp:288-295)
  const int* eo_off;
  const int* eo_i;
  const int* eo_j;
  const double2* eo_v;
  // sesolve observation: e_ops as CSR, rowptr blocks of n+1 per op, col/val at se_off[e]
  const int* se_rowptr;
  const int* se_col;
  const double2* se_val;
  const long long* se_off;
  // sesolve observation through operator stores (plain or dictionary-coded, like the generator's)
  // instead of the CSR above when n_se_ops == n_e
  int n_se_ops;
  DevSell se_ops[kGridMaxSeOps];
  double2* expect;  // n_e x n_grid, column-major
  double2* states;  // n_save x n
  GridCtl* ctl;
  double* red;       // kNumSlots x G partials
  unsigned* bar;     // grid barrier: one 64-bit arrival counter
};

// K-cluster (cluster-resident solve, grid_engine.cu): dynamic shared-memory layout of one CTA.
struct ClLayout {
  int R;  // rows per CTA (multiple of 32)
  int S;  // slices per CTA = R / 32
  int E;  // entry capacity (32 * the widest CTA's summed slice widths)
  int n_eo;  // mesolve e_op entries staged in shared memory (0: read from global)
  unsigned rmagic;  // ceil(2^32 / R): owner CTA of a row by multiply-high
  int obs_ow;  // stage-2 observation by one otherwise idle warp beside the pass
  unsigned vec, rowlen, soff, tgt, val, red, eo, bytes;
};
// true (and the cluster size / layout) when a single-term plain-store generator fits one cluster;
// n_eo: mesolve e_op entries (staged in shared memory when they fit too)
bool plan_cluster_solve(const GridProblem& P, const long long* slice_off_host, int n_obs_slots, int n_eo, int* C_out,
                        ClLayout* plan);
cudaError_t launch_cluster_dp5(const GridProblem& P, int mode, const ClLayout& L, int C, cudaStream_t s);

int grid_threads();
// st: 0 generic rows, 1 dictionary-coded store (pipelined), 2 key-aligned store (TMA ring)
size_t grid_smem_bytes(const GridProblem& P, int st);
int grid_max_blocks_per_sm(int mode, int st, size_t dyn_smem = 0);
cudaError_t launch_grid_dp5(const GridProblem& P, int mode, int st, int grid, cudaStream_t s);
// largest grid that runs as ONE thread-block cluster (<= 16 CTAs, one per SM), 0 if none
int grid_max_cluster(int mode, int st, size_t dyn_smem);

}  // namespace qsg
