// Internal host-side structures shared by the C-ABI translation units.
#pragma once

#include <atomic>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <string>
#include <vector>

#include "../../include/qsg.h"
#include "engine.cuh"

struct qsg_ctx {
  int device = 0;
  int sm_count = 0;
  long long l2_bytes = 0;
  char name[256] = {0};
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // cached solver workspace
  void* work = nullptr;
  size_t work_bytes = 0;
  // lifetime: one reference held by the creator (dropped by qsg_ctx_destroy) plus one per live
  // operator, so an operator destroyed after its context can still free on the context's stream
  std::atomic<int> refs{1};
};

// HBM operator store: SELL-32 layout (engine.cuh DevSell) built on device from the CSR input.
struct qsg_op {
  qsg_ctx* ctx = nullptr;
  long long n_rows = 0, n_cols = 0, nnz = 0;
  long long n_slices = 0, padded_cols = 0;  // padded_cols = slice_off[n_slices]
  long long* slice_off = nullptr;
  int* rowlen = nullptr;
  int* col = nullptr;
  double2* val = nullptr;
  int max_rowlen = 0;
  // dictionary-coded entries (engine.cuh DevSell): 0 = plain, 1 = uint8, 2 = uint16 codes
  int code_bytes = 0;
  long long* code_off = nullptr;  // per slice, in entries (row-contiguous code blocks)
  void* code = nullptr;
  int* dict_off = nullptr;
  double2* dict_val = nullptr;
  int dict_n = 0;
  // key-aligned store (engine.cuh DevSell::ka_*): per-slice blocks of (key, lane mask, value id)
  // positions + the distinct-value table; built alongside the other stores when it pays
  unsigned* ka_off = nullptr;  // n_slices + 1, in 16-byte units
  uint4* ka_blk = nullptr;
  double2* ka_val = nullptr;
  int ka_nval = 0;
  int ka_slot = 0;            // largest block, bytes
  long long ka_bytes = 0;     // whole store, bytes
  long long ka_positions = 0; // sum over slices of the key-union width
};

namespace qsg {
DevSell sell_view(const qsg_op* op, bool use_codes = true);
}

namespace qsg {

void set_error(const std::string& msg);
qsg_status cuda_fail(cudaError_t e, const char* where);
bool is_device_ptr(const void* p);

// RAII device buffer on the context stream (stream-ordered allocator).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(&p, bytes ? bytes : 16, st);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Upload host-or-device array into a fresh device buffer.
cudaError_t upload(DevBuf& b, const void* src, size_t bytes, cudaStream_t s);

DevGen make_devgen(const qsg_generator* g, bool use_codes = true);
qsg_status check_generator(const qsg_generator* g, long long n);
qsg_status check_tlist(const double* tlist, long long n_t);

// evolve.cpp:89-118 build_events: tlist points (+ merged saveat) -> (t, grid index, save slot)
struct Events {
  std::vector<double> t;
  std::vector<int> grid;
  std::vector<int> save;
  int n_save = 0;
};
qsg_status build_events(const double* tlist, long long n_t, const qsg_solve_opts* o,
                        bool keep_states, Events& ev);

qsg_status status_from_device(int st, double t);

}  // namespace qsg

// NVTX range over a C-ABI entry point (named in nsys timelines and `ncu --nvtx` filters); NVTX v3 is
// header-only and costs nothing unless a tool is attached.
struct QsgRange {
  explicit QsgRange(const char* name) { nvtxRangePushA(name); }
  ~QsgRange() { nvtxRangePop(); }
  QsgRange(const QsgRange&) = delete;
  QsgRange& operator=(const QsgRange&) = delete;
};
#define QSG_RANGE(name) QsgRange qsg_nvtx_range_(name)
