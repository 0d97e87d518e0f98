// Batch engine layout 4, plain-store-only instantiation (batch_kernel.cuh QSG_BATCH_LEAN).
#define QSG_BATCH_LEAN 1
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(4, 1, GM_CTA)
