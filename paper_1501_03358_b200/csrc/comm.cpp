// Multi-GPU communication of librk: z-slab decomposition
// with one ghost plane per neighbour, exchanged by grouped NCCL send/recv,
// and in-place fp64 sum all-reduce of the batched dot-product vectors.
// With one rank both are no-ops (a single-rank periodic z wraps in-kernel).
#include <condition_variable>
#include <memory>
#include <mutex>

#include "rk_internal.h"

// ------------------------------------------------------------------ local
// In-process rank group: contexts whose uid is "RKLOCAL:<name>" (the rest of
// the 128 bytes zero) join the group <name>; each rank is driven by its own
// host thread and stream.  It exists so that librk's own multi-rank
// schedule -- every halo() and allreduce() call of the solvers, in the order
// the solvers issue them -- runs, and is tested, on a box with one GPU: the
// kernels of one rank never wait on another rank's kernels (a halo is a
// device copy of a neighbour's planes after that neighbour's producer event;
// an all-reduce is host-mediated), so nothing can deadlock on the device.
struct LocalGroup {
  int n = 0, members = 0;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  int64_t gen = 0;
  std::vector<const double*> lo, hi;
  std::vector<cudaEvent_t> eva, evb;
  std::vector<std::vector<double>> hbuf;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {
std::mutex g_reg_mu;
std::map<std::string, std::shared_ptr<LocalGroup>> g_reg;
const char kLocal[] = "RKLOCAL:";
}  // namespace

namespace rk {

bool local_uid(const uint8_t* uid) {
  return uid && std::memcmp(uid, kLocal, sizeof(kLocal) - 1) == 0;
}

void local_join(rk_ctx* ctx, const uint8_t* uid) {
  std::string name(reinterpret_cast<const char*>(uid) + sizeof(kLocal) - 1,
                   strnlen(reinterpret_cast<const char*>(uid) + sizeof(kLocal) - 1, 128 - sizeof(kLocal) + 1));
  std::shared_ptr<LocalGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto& e = g_reg[name];
    if (!e) {
      e = std::make_shared<LocalGroup>();
      e->n = ctx->nranks;
      e->lo.assign(e->n, nullptr);
      e->hi.assign(e->n, nullptr);
      e->eva.assign(e->n, nullptr);
      e->evb.assign(e->n, nullptr);
      e->hbuf.assign(e->n, {});
    }
    RK_REQUIRE(e->n == ctx->nranks, RK_EINVAL, "local group size mismatch");
    ++e->members;
    g = e;
  }
  for (auto& ev : ctx->lev) RK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  ctx->lgrp = g.get();
}

void local_leave(rk_ctx* ctx) {
  if (!ctx->lgrp) return;
  for (auto& ev : ctx->lev)
    if (ev) cudaEventDestroy(ev);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (auto it = g_reg.begin(); it != g_reg.end(); ++it)
    if (it->second.get() == ctx->lgrp) {
      if (--it->second->members == 0) g_reg.erase(it);
      break;
    }
  ctx->lgrp = nullptr;
}

namespace {
// z-neighbours of this rank (-1: none), as halo() below
void neighbours(const rk_op* op, int& up, int& dn) {
  const rk_ctx* ctx = op->ctx;
  const bool pz = (op->g.periodic_mask & 4) != 0;
  const int R = ctx->nranks, me = ctx->rank;
  up = me + 1;
  dn = me - 1;
  if (pz) {
    up %= R;
    dn = (dn + R) % R;
  } else if (up >= R) {
    up = -1;
  }
}

// Neighbour exchange: publish (source pointers, a producer event), copy the
// neighbours' sources after their events, publish a copies-done event that
// the neighbours wait for before they may overwrite what was just read.
void exchange_local(rk_op* op, const double* lo_src, const double* hi_src, double* lo_dst,
                    double* hi_dst, size_t count) {
  rk_ctx* ctx = op->ctx;
  LocalGroup* g = ctx->lgrp;
  const int me = ctx->rank;
  int up, dn;
  neighbours(op, up, dn);
  const size_t bytes = sizeof(double) * count;
  RK_CUDA(cudaEventRecord(ctx->lev[0], ctx->stream));
  g->lo[me] = lo_src;
  g->hi[me] = hi_src;
  g->eva[me] = ctx->lev[0];
  g->barrier();
  if (dn >= 0) {   // lo_dst <- the lower neighbour's hi_src
    RK_CUDA(cudaStreamWaitEvent(ctx->stream, g->eva[dn], 0));
    RK_CUDA(cudaMemcpyAsync(lo_dst, g->hi[dn], bytes, cudaMemcpyDefault, ctx->stream));
  }
  if (up >= 0) {   // hi_dst <- the upper neighbour's lo_src
    RK_CUDA(cudaStreamWaitEvent(ctx->stream, g->eva[up], 0));
    RK_CUDA(cudaMemcpyAsync(hi_dst, g->lo[up], bytes, cudaMemcpyDefault, ctx->stream));
  }
  RK_CUDA(cudaEventRecord(ctx->lev[1], ctx->stream));
  g->evb[me] = ctx->lev[1];
  g->barrier();
  if (dn >= 0) RK_CUDA(cudaStreamWaitEvent(ctx->stream, g->evb[dn], 0));
  if (up >= 0) RK_CUDA(cudaStreamWaitEvent(ctx->stream, g->evb[up], 0));
  g->barrier();
}

// Sum over the ranks in rank order (every rank gets the same bits).
void allreduce_local(rk_ctx* ctx, double* buf, int n) {
  LocalGroup* g = ctx->lgrp;
  const int me = ctx->rank;
  g->hbuf[me].resize(n);
  RK_CUDA(cudaMemcpyAsync(g->hbuf[me].data(), buf, sizeof(double) * n, cudaMemcpyDeviceToHost,
                          ctx->stream));
  RK_CUDA(cudaStreamSynchronize(ctx->stream));
  g->barrier();
  std::vector<double> sum(g->hbuf[0]);
  for (int r = 1; r < g->n; ++r)
    for (int i = 0; i < n; ++i) sum[i] += g->hbuf[r][i];
  g->barrier();
  RK_CUDA(cudaMemcpyAsync(buf, sum.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  RK_CUDA(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

#ifdef RK_WITH_NCCL
#define RK_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw ::rk::Error(RK_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));  \
  } while (0)
#endif

// Collective-launch accounting (rk_comm_count): what NCCL would launch --
// one per all-reduce or halo exchange issued outside a group, one per
// outermost group (a group holding a halo counts as a halo launch).  The
// in-process rank group counts the same way, so the schedule's collective
// count per Krylov step is testable on one GPU.
static void note_collective(rk_ctx* ctx, bool is_halo) {
  if (ctx->comm_depth > 0) {
    (is_halo ? ctx->comm_pend_halo : ctx->comm_pend_ar) = true;
  } else {
    ++(is_halo ? ctx->n_halo : ctx->n_allreduce);
  }
}
static void note_group(rk_ctx* ctx, int delta) {
  ctx->comm_depth += delta;
  if (ctx->comm_depth == 0) {
    if (ctx->comm_pend_halo) ++ctx->n_halo;
    else if (ctx->comm_pend_ar) ++ctx->n_allreduce;
    ctx->comm_pend_halo = ctx->comm_pend_ar = false;
  }
}

// Ordering (NCCL): first every rank sends its hi_src up and receives its
// lo_dst from below, then sends its lo_src down and receives its hi_dst from
// above; sends/recvs between one pair of ranks are matched in issue order,
// so this is also correct for a 2-rank ring.
void exchange(rk_op* op, const double* lo_src, const double* hi_src, double* lo_dst, double* hi_dst,
              size_t count) {
  rk_ctx* ctx = op->ctx;
  if (ctx->nranks == 1) return;
  note_collective(ctx, true);
  if (ctx->lgrp) return exchange_local(op, lo_src, hi_src, lo_dst, hi_dst, count);
#ifdef RK_WITH_NCCL
  int up, dn;
  neighbours(op, up, dn);
  RK_NCCL(ncclGroupStart());
  if (up >= 0) RK_NCCL(ncclSend(hi_src, count, ncclDouble, up, ctx->comm, ctx->stream));
  if (dn >= 0) RK_NCCL(ncclRecv(lo_dst, count, ncclDouble, dn, ctx->comm, ctx->stream));
  if (dn >= 0) RK_NCCL(ncclSend(lo_src, count, ncclDouble, dn, ctx->comm, ctx->stream));
  if (up >= 0) RK_NCCL(ncclRecv(hi_dst, count, ncclDouble, up, ctx->comm, ctx->stream));
  RK_NCCL(ncclGroupEnd());
#else
  throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
}

// Collectives issued between comm_group_begin / comm_group_end go out as one
// NCCL launch (NCCL groups nest; the outermost end issues them); the
// in-process rank group runs them one by one as issued.
void comm_group_begin(rk_ctx* ctx) {
  if (ctx->nranks > 1) note_group(ctx, +1);
#ifdef RK_WITH_NCCL
  if (ctx->nranks > 1 && !ctx->lgrp) RK_NCCL(ncclGroupStart());
#else
  (void)ctx;
#endif
}
void comm_group_end(rk_ctx* ctx) {
#ifdef RK_WITH_NCCL
  if (ctx->nranks > 1 && !ctx->lgrp) RK_NCCL(ncclGroupEnd());
#endif
  if (ctx->nranks > 1) note_group(ctx, -1);
}

// Fill `depth` ghost planes below and above the padded vector v (local
// planes [0, nz_local)) from the z-neighbours' boundary planes.
void halo(rk_op* op, const double* v, int depth) {
  if (op->ctx->nranks == 1) return;
  RK_REQUIRE(depth >= 1 && depth <= GHOST && depth <= op->g.nz_local, RK_EINVAL, "bad halo depth");
  const int64_t P = op->P;
  exchange(op, v, v + (op->g.nz_local - depth) * P, const_cast<double*>(v) - depth * P,
           const_cast<double*>(v) + op->N, (size_t)(depth * P));
}

// Several reduction outputs in ONE collective launch: NCCL aggregates the
// all-reduces of a group (batch each reduction's values).
void allreduce2(rk_ctx* ctx, double* a, int na, double* b, int nb) {
  if (ctx->nranks == 1 || na + nb == 0) return;
  note_collective(ctx, false);
  if (ctx->lgrp) {
    if (na) allreduce_local(ctx, a, na);
    if (nb) allreduce_local(ctx, b, nb);
    return;
  }
#ifdef RK_WITH_NCCL
  RK_NCCL(ncclGroupStart());
  if (na) RK_NCCL(ncclAllReduce(a, a, (size_t)na, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  if (nb) RK_NCCL(ncclAllReduce(b, b, (size_t)nb, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  RK_NCCL(ncclGroupEnd());
#else
  throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
}

void allreduce(rk_ctx* ctx, double* buf, int n) {
  if (ctx->nranks == 1 || n == 0) return;
  note_collective(ctx, false);
  if (ctx->lgrp) return allreduce_local(ctx, buf, n);
#ifdef RK_WITH_NCCL
  RK_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
#else
  throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
}

}  // namespace rk
