// Batch engine layout 4: 1 slot per CTA (default).
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(4, 1, GM_CTA)
