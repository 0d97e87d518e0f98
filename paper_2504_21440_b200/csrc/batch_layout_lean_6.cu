// Batch engine layout 6, plain-store-only instantiation (batch_kernel.cuh QSG_BATCH_LEAN).
#define QSG_BATCH_LEAN 1
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(6, 2, GM_CLUSTER)
