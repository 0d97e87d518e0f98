// Batch engine layout 1, plain-store single-term instantiation (batch_kernel.cuh QSG_BATCH_LEAN 2):
// the mcsolve layouts, whose generator is one H_eff term.
#define QSG_BATCH_LEAN 2
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(1, 32, GM_GRID)
