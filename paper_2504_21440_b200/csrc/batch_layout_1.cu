// Batch engine layout 1: one 32-slot batch over the cooperative grid.
#include "batch_kernel.cuh"

QSG_BATCH_LAYOUT(1, 32, GM_GRID)
