// Batch engine layout 2, plain-store-only instantiation (batch_kernel.cuh QSG_BATCH_LEAN).
#define QSG_BATCH_LEAN 1
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(2, 4, GM_CTA)
