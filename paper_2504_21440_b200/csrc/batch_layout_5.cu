// Batch engine layout 5: 1 slot per thread-block cluster.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(5, 1, GM_CLUSTER)
