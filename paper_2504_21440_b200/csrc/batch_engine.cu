// Layout dispatch of the batched DP5 engine (kernels in batch_kernel.cuh, one instantiation per
// translation unit: batch_layout_*.cu).
#include "batch_engine.h"

namespace qsg {

#define QSG_DECL_LAYOUT(ID)                                                       \
  int batch_layout_occ_##ID();                                                    \
  int batch_layout_clusters_##ID(int cs);                                         \
  cudaError_t batch_layout_launch_##ID(const BatchProblem& P, int grid, int cs, cudaStream_t s);
QSG_DECL_LAYOUT(0)
QSG_DECL_LAYOUT(1)
QSG_DECL_LAYOUT(2)
QSG_DECL_LAYOUT(3)
QSG_DECL_LAYOUT(4)
QSG_DECL_LAYOUT(5)
QSG_DECL_LAYOUT(6)
QSG_DECL_LAYOUT(7)
#define QSG_DECL_LEAN(ID) \
  cudaError_t batch_layout_lean_launch_##ID(const BatchProblem& P, int grid, int cs, cudaStream_t s);
QSG_DECL_LEAN(0)
QSG_DECL_LEAN(1)
QSG_DECL_LEAN(2)
QSG_DECL_LEAN(3)
QSG_DECL_LEAN(4)
QSG_DECL_LEAN(5)
QSG_DECL_LEAN(6)
QSG_DECL_LEAN(7)
cudaError_t batch_layout_lean1_launch_1(const BatchProblem& P, int grid, int cs, cudaStream_t s);
cudaError_t batch_layout_lean1_launch_4(const BatchProblem& P, int grid, int cs, cudaStream_t s);

constexpr int kNbuf = 12;  // state arrays per batch (batch_kernel.cuh NBUF)

// layouts: 0/2/3/4 = per-CTA batches of 8/4/2/1 slots, 1 = grid-wide batch of 32 slots,
// 5/6 = per-cluster batches of 1/2 slots, 7 = 1 slot per cluster with its state in DSMEM
int batch_slots(int layout) {
  switch (layout) {
    case 1: return 32;
    case 2: return 4;
    case 3: return 2;
    case 4: return 1;
    case 5: return 1;
    case 6: return 2;
    case 7: return 1;
    default: return 8;
  }
}

size_t batch_work_stride(int n, int layout) {
  if (layout == 7) return 2;  // state in shared memory; a token global workspace
  return static_cast<size_t>(kNbuf) * static_cast<size_t>(n) * batch_slots(layout);
}

size_t batch_dsm_smem(int shift) {
  return static_cast<size_t>(16 * 15 * 8 + 15) / 16 * 16 + static_cast<size_t>(kNbuf) * (size_t(1) << shift) * 16;
}

int batch_max_blocks_per_sm(int layout) {
  switch (layout) {
    case 1: return batch_layout_occ_1();
    case 2: return batch_layout_occ_2();
    case 3: return batch_layout_occ_3();
    case 4: return batch_layout_occ_4();
    case 5: return batch_layout_occ_5();
    case 6: return batch_layout_occ_6();
    case 7: return batch_layout_occ_7();
    default: return batch_layout_occ_0();
  }
}

int batch_max_clusters(int layout, int cs) {
  return layout == 5 ? batch_layout_clusters_5(cs) : layout == 6 ? batch_layout_clusters_6(cs)
         : layout == 7 ? batch_layout_clusters_7(cs) : 0;
}

cudaError_t launch_batch(const BatchProblem& P, int layout, int grid, int cs, cudaStream_t s) {
  if (P.lean && P.gen.n_terms == 1 && (layout == 1 || layout == 4))
    return layout == 1 ? batch_layout_lean1_launch_1(P, grid, cs, s) : batch_layout_lean1_launch_4(P, grid, cs, s);
  if (P.lean) switch (layout) {
      case 1: return batch_layout_lean_launch_1(P, grid, cs, s);
      case 2: return batch_layout_lean_launch_2(P, grid, cs, s);
      case 3: return batch_layout_lean_launch_3(P, grid, cs, s);
      case 4: return batch_layout_lean_launch_4(P, grid, cs, s);
      case 5: return batch_layout_lean_launch_5(P, grid, cs, s);
      case 6: return batch_layout_lean_launch_6(P, grid, cs, s);
      case 7: return batch_layout_lean_launch_7(P, grid, cs, s);
      default: return batch_layout_lean_launch_0(P, grid, cs, s);
    }
  switch (layout) {
    case 1: return batch_layout_launch_1(P, grid, cs, s);
    case 2: return batch_layout_launch_2(P, grid, cs, s);
    case 3: return batch_layout_launch_3(P, grid, cs, s);
    case 4: return batch_layout_launch_4(P, grid, cs, s);
    case 5: return batch_layout_launch_5(P, grid, cs, s);
    case 6: return batch_layout_launch_6(P, grid, cs, s);
    case 7: return batch_layout_launch_7(P, grid, cs, s);
    default: return batch_layout_launch_0(P, grid, cs, s);
  }
}

}  // namespace qsg
