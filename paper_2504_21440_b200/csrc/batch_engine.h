// Host <-> device contract of the batched trajectory / sweep engine (batch_engine.cu).
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace qsg {

constexpr int kBatchMaxPend = 6;   // observation events a slot can carry into one round
constexpr int kBatchMaxCops = 24;  // collapse operators (mcsolve)
constexpr int kBatchMaxEops = 8;   // expectation operators

struct BatchProblem {
  int mode;  // 0: mcsolve trajectories, 1: mesolve parameter points
  int autonomous;  // every generator term's coefficient is time-independent (stage-2 identity)
  int lean;  // every operator is a plain SELL store: launch the plain-only kernel instantiation
  int n;     // vector length (d for mcsolve, d*d for mesolve)
  int d;
  DevGen gen;  // terms shared by every system
  const double* params;  // n_systems x n_params (mode 1) or n_params (mode 0)
  int n_params;
  long long n_systems;   // trajectories (mode 0) or parameter points (mode 1)
  long long sys_begin;   // first trajectory index (RNG stream) / point index
  unsigned long long seed;
  const double2* y0;     // initial vector (n)
  double atol, rtol;
  long long max_steps;
  const double* tlist;
  int n_t;
  double t0, tf, eps_t;
  // observation operators: mcsolve <y|E y>/|y|^2 (SELL, trajectories.cpp:133-139);
  // mesolve hermitized trace over entries (evolve.cpp:286-295)
  int n_e;
  DevSell e_ops[kBatchMaxEops];
  const int* eo_off;
  const int* eo_i;
  const int* eo_j;
  const double2* eo_v;
  int n_c;
  DevSell c_ops[kBatchMaxCops];
  // workspace: per CTA 14 buffers of n x B complex
  double2* work;
  long long work_stride;  // doubles2 per CTA
  unsigned long long* queue;  // next system counter
  // outputs (indexed by system - sys_begin)
  double2* expect;           // n_sys x (n_e x n_t)
  int* status;               // n_sys
  double* fail_t;            // n_sys
  long long* stats;          // n_sys x 3
  int* jump_count;           // n_sys
  double* jump_time;         // n_sys x jump_cap
  int* jump_channel;
  int jump_cap;
  long long* attempts_total;  // accumulated device attempts (perf accounting)
  // grid mode: deterministic cross-CTA slot reductions and pass barriers
  double* gpart;  // (32 slots x 15 values) x G partials
  double* gfin;   // 32 x 15 totals
  unsigned* bar;  // {count, generation}
  // layout 7 (state resident in the cluster's distributed shared memory): each CTA of a cluster
  // owns 1 << dsm_shift rows of every state array, in its shared memory
  int dsm_shift;
};

int batch_slots(int layout);
// layout 7: dynamic shared memory per CTA for 1 << shift rows of the 12 state arrays
size_t batch_dsm_smem(int shift);
// cs: CTAs per cluster (cluster layouts 5/6 only); grid must then be a multiple of cs
cudaError_t launch_batch(const BatchProblem& P, int layout, int grid, int cs, cudaStream_t s);
int batch_max_clusters(int layout, int cs);  // co-resident clusters of cs CTAs
int batch_max_blocks_per_sm(int layout);
size_t batch_work_stride(int n, int layout);  // double2 elements per batch

}  // namespace qsg
