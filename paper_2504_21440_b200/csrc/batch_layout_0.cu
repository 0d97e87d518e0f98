// Batch engine layout 0: 8 slots per CTA.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(0, 8, GM_CTA)
