// Batch engine layout 7: 1 slot per thread-block cluster, its state resident in the cluster's
// distributed shared memory.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(7, 1, GM_DSM)
