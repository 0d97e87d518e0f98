// Batch engine layout 4, plain-store single-term instantiation (batch_kernel.cuh QSG_BATCH_LEAN 2):
// the mcsolve layouts, whose generator is one H_eff term.
#define QSG_BATCH_LEAN 2
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(4, 1, GM_CTA)
