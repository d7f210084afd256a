// Multi-GPU communication of librk: z-slab decomposition
// with one ghost plane per neighbour, exchanged by grouped NCCL send/recv,
// and in-place fp64 sum all-reduce of the batched dot-product vectors.
// With one rank both are no-ops (a single-rank periodic z wraps in-kernel).
#include "rk_internal.h"

namespace rk {

#ifdef RK_WITH_NCCL
#define RK_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw ::rk::Error(RK_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));  \
  } while (0)
#endif

// Fill the ghost planes v[-P..-1] and v[N..N+P-1] of a padded vector from
// the z-neighbours.  Ordering: first every rank sends its TOP plane up and
// receives its lower ghost from below, then sends its BOTTOM plane down and
// receives its upper ghost from above; sends/recvs between one pair of ranks
// are matched in issue order, so this is also correct for a 2-rank ring.
void halo(rk_op* op, const double* v) {
  rk_ctx* ctx = op->ctx;
  if (ctx->nranks == 1) return;
#ifdef RK_WITH_NCCL
  const bool pz = (op->g.periodic_mask & 4) != 0;
  const int R = ctx->nranks, me = ctx->rank;
  int up = me + 1, dn = me - 1;
  if (pz) {
    up %= R;
    dn = (dn + R) % R;
  } else {
    if (up >= R) up = -1;
  }
  const size_t P = (size_t)op->P;
  const double* top = v + (op->g.nz_local - 1) * op->P;
  double* ghost_lo = const_cast<double*>(v) - op->P;
  double* ghost_hi = const_cast<double*>(v) + op->N;
  RK_NCCL(ncclGroupStart());
  if (up >= 0) RK_NCCL(ncclSend(top, P, ncclDouble, up, ctx->comm, ctx->stream));
  if (dn >= 0) RK_NCCL(ncclRecv(ghost_lo, P, ncclDouble, dn, ctx->comm, ctx->stream));
  if (dn >= 0) RK_NCCL(ncclSend(v, P, ncclDouble, dn, ctx->comm, ctx->stream));
  if (up >= 0) RK_NCCL(ncclRecv(ghost_hi, P, ncclDouble, up, ctx->comm, ctx->stream));
  RK_NCCL(ncclGroupEnd());
#else
  throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
}

void allreduce(rk_ctx* ctx, double* buf, int n) {
  if (ctx->nranks == 1 || n == 0) return;
#ifdef RK_WITH_NCCL
  RK_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
#else
  throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
}

}  // namespace rk
