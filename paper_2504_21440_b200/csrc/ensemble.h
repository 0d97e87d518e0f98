// Device-side ensemble accumulation (ensemble.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace qsg {

// Pairwise-bracket sums (trajectories.cpp:17-22) of per-trajectory matrices per (n_sys x nv,
// device) over the completed trajectories (status == kDone), computed on the device. With
// n_ranges == 0 one sum over the whole completed list; otherwise one per [range_lo, range_hi) of
// completed-list positions (range_hi < 0: to the end of the list). n_ok: completed trajectories; sums: nr x nv.
cudaError_t device_bracket_sums(const double2* per, const int* status, long long n_sys, long long nv,
                                int n_ranges, const long long* range_lo, const long long* range_hi,
                                cudaStream_t s, long long& n_ok, std::vector<double2>& sums);

}  // namespace qsg
