// NCCL communicators behind the C-ABI: the exchange step of sharded ensembles and
// sweeps. Block sums of the pairwise bracket (trajectories.cpp:17-22) are all-gathered over
// NVLink and combined in the reference bracket (qsg_ensemble_combine), so the mean is bitwise the
// single-device one. Replaces run_ensemble's in-process thread pool combine (trajectories.cpp:
// 31-58, 82-83) when the ensemble spans several GPUs.
//
// NCCL is resolved at run time (dlopen): a process that already loaded an NCCL (torch's) shares
// it, so two different libnccl.so.2 never meet in one address space. Missing NCCL is reported as
// QSG_NCCL_ERROR, never silently replaced.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "qsg_internal.h"

using namespace qsg;

namespace {

// the slice of nccl.h this file uses (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0, ncclFloat64 = 8, ncclDouble = 8 };

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  bool ok = false;
  std::string why;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("NCCL library not found: ") + (dlerror() ? dlerror() : "");
      return;
    }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(sym("ncclGetVersion"));
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommInitAll && n.CommDestroy && n.AllGather && n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
    if (!n.ok) n.why = "NCCL library lacks a required symbol";
  });
  return n;
}

qsg_status nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string("NcclError: ") + where + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
  return QSG_NCCL_ERROR;
}

qsg_status need_nccl() {
  if (!nccl().ok) {
    set_error("NcclError: " + nccl().why);
    return QSG_NCCL_ERROR;
  }
  return QSG_OK;
}

}  // namespace

struct qsg_comm {
  ncclComm_t comm = nullptr;
  qsg_ctx* ctx = nullptr;  // device + stream the collectives run on
  int nranks = 0, rank = 0;
  bool own_ctx = false;
};

extern "C" {

int32_t qsg_nccl_version(void) {
  int v = 0;
  if (nccl().ok && nccl().GetVersion) nccl().GetVersion(&v);
  return v;
}

qsg_status qsg_comm_unique_id(uint8_t* id128) {
  if (qsg_status s = need_nccl()) return s;
  ncclUniqueId id;
  if (ncclResult_t r = nccl().GetUniqueId(&id)) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id128, id.internal, 128);
  return QSG_OK;
}

qsg_status qsg_comm_init_rank(qsg_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id128, qsg_comm** out) {
  QSG_RANGE("qsg_comm_init_rank");
  if (!ctx || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("InvalidGrid: bad communicator arguments");
    return QSG_INVALID_GRID;
  }
  if (qsg_status s = need_nccl()) return s;
  cudaSetDevice(ctx->device);
  ncclUniqueId id;
  std::memcpy(id.internal, id128, 128);
  auto* c = new qsg_comm;
  if (ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank)) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return QSG_OK;
}

qsg_status qsg_comm_init_all(int32_t n_dev, const int32_t* devices, qsg_comm** out) {
  QSG_RANGE("qsg_comm_init_all");
  if (n_dev < 1 || !devices || !out) {
    set_error("InvalidGrid: bad communicator arguments");
    return QSG_INVALID_GRID;
  }
  if (qsg_status s = need_nccl()) return s;
  for (int i = 0; i < n_dev; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j]) {
        set_error("InvalidGrid: one communicator rank per device (duplicate device id)");
        return QSG_INVALID_GRID;
      }
  std::vector<ncclComm_t> cs(static_cast<size_t>(n_dev));
  std::vector<int> dv(devices, devices + n_dev);
  if (ncclResult_t r = nccl().CommInitAll(cs.data(), n_dev, dv.data())) return nccl_fail(r, "ncclCommInitAll");
  for (int i = 0; i < n_dev; ++i) {
    auto* c = new qsg_comm;
    c->comm = cs[static_cast<size_t>(i)];
    if (qsg_status s = qsg_ctx_create(devices[i], &c->ctx)) {
      delete c;
      return s;
    }
    c->own_ctx = true;
    c->nranks = n_dev;
    c->rank = i;
    out[i] = c;
  }
  return QSG_OK;
}

qsg_ctx* qsg_comm_ctx(qsg_comm* c) { return c ? c->ctx : nullptr; }

void qsg_comm_destroy(qsg_comm* c) {
  if (!c) return;
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  if (c->own_ctx) qsg_ctx_destroy(c->ctx);
  delete c;
}

// recv[r*count .. (r+1)*count) = rank r's send (doubles); host or device buffers.
qsg_status qsg_comm_allgather(qsg_comm* c, const double* send, int64_t count, double* recv) {
  QSG_RANGE("qsg_comm_allgather");
  if (!c || !send || !recv || count < 0) {
    set_error("InvalidGrid: bad all-gather arguments");
    return QSG_INVALID_GRID;
  }
  cudaSetDevice(c->ctx->device);
  cudaStream_t s = c->ctx->stream;
  const size_t bytes = sizeof(double) * static_cast<size_t>(count);
  DevBuf ds, dr;
  cudaError_t e;
  if ((e = ds.alloc(bytes, s)) || (e = dr.alloc(bytes * c->nranks, s)) ||
      (e = cudaMemcpyAsync(ds.p, send, bytes, cudaMemcpyDefault, s)))
    return cuda_fail(e, "all-gather staging");
  if (ncclResult_t r = nccl().AllGather(ds.p, dr.p, static_cast<size_t>(count), ncclFloat64, c->comm, s))
    return nccl_fail(r, "ncclAllGather");
  if ((e = cudaMemcpyAsync(recv, dr.p, bytes * c->nranks, cudaMemcpyDefault, s)) || (e = cudaStreamSynchronize(s)))
    return cuda_fail(e, "all-gather");
  return QSG_OK;
}

}  // extern "C"
