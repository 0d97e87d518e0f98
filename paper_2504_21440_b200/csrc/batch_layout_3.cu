// Batch engine layout 3: 2 slots per CTA.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(3, 2, GM_CTA)
