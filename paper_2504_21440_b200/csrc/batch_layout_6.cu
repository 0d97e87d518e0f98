// Batch engine layout 6: 2 slots per thread-block cluster.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(6, 2, GM_CLUSTER)
