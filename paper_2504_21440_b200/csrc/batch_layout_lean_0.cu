// Batch engine layout 0, plain-store-only instantiation (batch_kernel.cuh QSG_BATCH_LEAN).
#define QSG_BATCH_LEAN 1
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(0, 8, GM_CTA)
