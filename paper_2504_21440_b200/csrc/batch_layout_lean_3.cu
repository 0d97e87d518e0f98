// Batch engine layout 3, plain-store-only instantiation (batch_kernel.cuh QSG_BATCH_LEAN).
#define QSG_BATCH_LEAN 1
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(3, 2, GM_CTA)
