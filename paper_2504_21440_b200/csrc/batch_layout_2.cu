// Batch engine layout 2: 4 slots per CTA.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(2, 4, GM_CTA)
