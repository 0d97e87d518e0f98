// Batched trajectory / sweep engine — entry points (implementation in progress).
#include "qsg_internal.h"

using namespace qsg;

extern "C" qsg_status qsg_mcsolve(qsg_ctx*, const qsg_generator*, int32_t, const qsg_csr*, int32_t,
                                  const qsg_csr*, int64_t, const double*, const double*, int64_t,
                                  const double*, int32_t, uint64_t, int64_t, int64_t,
                                  const qsg_solve_opts*, qsg_mc_out*, qsg_timing*) {
  set_error("mcsolve engine not built yet");
  return QSG_UNSUPPORTED;
}

extern "C" qsg_status qsg_mesolve_batch(qsg_ctx*, const qsg_generator*, int64_t, const double*,
                                        const double*, int64_t, int32_t, const qsg_csr*, int64_t,
                                        const double*, int32_t, const qsg_solve_opts*, double*,
                                        qsg_stats*, int32_t*, qsg_timing*) {
  set_error("batched mesolve engine not built yet");
  return QSG_UNSUPPORTED;
}
