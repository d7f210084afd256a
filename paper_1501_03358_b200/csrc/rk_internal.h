// Internal declarations of librk (not part of the ABI; see include/rk.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <unordered_map>
#include <string>
#include <vector>

#include "rk.h"

#ifdef RK_WITH_NCCL
#include <nccl.h>
#endif

namespace rk {

constexpr int MAXCOL = 80;      // columns of one block product ([C V_j w] <= k_max + m + 1)
// Ghost planes below and above every padded vector: one per stencil stage
// of a fused chain launch (at most 3), so a chain launch on a z-slab reads
// its input NST planes beyond the slab after one NST-deep halo exchange.
constexpr int GHOST = 3;
// Ghost planes of the bands kept from each z-neighbour on several ranks
// (the chains recompute NST - 1 <= 2 halo planes of stage 0).
constexpr int BGHOST = 2;
constexpr int MAXOUT = 5;       // outputs of one lincomb (dx, u1, c1, u2, c2)

struct Error : std::runtime_error {
  rk_status st;
  Error(rk_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define RK_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::rk::Error(RK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define RK_REQUIRE(cond, st, msg)                    \
  do {                                               \
    if (!(cond)) throw ::rk::Error((st), (msg));     \
  } while (0)

// ---------------------------------------------------------------- kernels
struct ColPtrs {
  const double* p[MAXCOL];
};

struct RedArgs {
  double* partials;     // [nval][gridDim.x]
  unsigned* counter;    // last-block ticket (reset by the last block)
  double* out;          // nval results (value q -> out[q] ...
  double* out2 = nullptr;   // ... or, for q >= split, out2[q - split])
  int split = 1 << 30;
  int valid = 1 << 30;  // only values with (q mod split) < valid are stored
  const double* gate = nullptr;   // kernel is a no-op when *gate != 0 (rBiCGStab lookahead)
  int defer = 0;                  // 1: store the per-CTA partials only (the consumer sums them)
};

// Block-update coefficients still as per-CTA partials of a deferred block dot
// (part[c * G + b], b < G); every CTA of the consumer sums them in the same
// fixed order and CTA 0 stores the sums to `store`.
struct CoefIn {
  const double* part = nullptr;
  int G = 0;
  double* store = nullptr;
};

// Stencil kernel modes (K1/K2 of SURVEY §2.4)
enum StencilMode {
  SM_SPMV = 0,          // out0 = A x
  SM_SPMV_SWEEP1 = 1,   // out0 = t = A x ; out1 = w t / D            (first Jacobi sweep fused)
  SM_SWEEP = 2,         // out0 = x + w (r - A x) / D                 (Jacobi sweep, x = z_in)
  SM_SWEEP_NORM = 3,    // SM_SWEEP + red ||out0||^2
  SM_RESID = 4,         // out0 = r - A x ; red ||out0||^2            (true residual, r = b)
  SM_RESID_SWEEP1 = 5,  // SM_RESID + out1 = w out0 / D
  SM_SCALE = 6,         // out0 = w r / D   (first sweep from z = 0; no stencil)
};

struct StencilParams {
  const double* bands;  // [S][N] canonical order, band 0 = diagonal
  const double* invd;   // [N] 1 / D
  int64_t N, P;
  int nx, ny, nzl;
  int px, py, wrapz;
  const double* x;      // padded stencil input (ghost planes at -P and N)
  const double* r;
  double* out0;
  double* out1;
  double omega;
  RedArgs red;
  int zb, zg0;          // local (block-Jacobi) sweep: z-block size in planes (0 = global), global z of plane 0
  const double* gate;   // no-op when *gate != 0 (rBiCGStab lookahead)
};

struct LcOut {
  double* out[MAXOUT];
  double scale[MAXOUT];
  int acc[MAXOUT];
};

// Stage kinds of the fused preconditioned-operator chain (chain.cu)
enum ChainKind {
  CK_SPMV1 = 0,   // t = A x (kept as the sweeps' right-hand side); z = w t / D
  CK_SWEEP = 1,   // z' = z + w (r - A z) / D
  CK_SPMV = 2,    // y = A z
};

struct ChainParams {
  const double* bands;  // [S + 1][N]: bands, then 1 / D
  int64_t N, P;
  int nx, ny, nz;
  int px, py, pz;
  const double* xin;    // stage-0 input (padded vector)
  const double* r;      // sweep right-hand side (unused when stage 0 is CK_SPMV1)
  double* out_t;        // CK_SPMV1: t (nullable)
  double* out_mid;      // output of stage NST-2 (nullable)
  double* out;          // output of the last stage
  double omega[3];
  int zc;               // z planes per CTA
  int zb, zg0;          // z-block size (0 = none) and global z of plane 0 (block-Jacobi)
  int local[3];         // stage s is a local sweep (no coupling across z-blocks)
  const double* gate;   // no-op when *gate != 0 (rBiCGStab lookahead)
  int ghost;            // several ranks: bands of planes outside [0, nz) from the ghost-band map
  int rz;               // z coordinate of plane 0 in the rhs tensor map (GHOST: padded rhs)
  // Arnoldi line 10 folded into the next line 6 (19-point chain, stage 0 =
  // CK_SPMV1 only): when xs_n2 != nullptr the input is the unnormalised w and
  // every input value is taken as w * (1 / h), h = sqrt(*xs_n2) (0 on the
  // happy breakdown h <= 1e-14 sqrt(*xs_in2)) -- normalize_kernel's
  // arithmetic; v_{j+1} of the interior cells goes to xs_out, the breakdown
  // flag to *xs_flag.
  const double* xs_n2;
  const double* xs_in2;
  double* xs_out;
  double* xs_flag;
};

// The normalisation a chain launch applies to its input (ChainParams::xs_*).
struct XScale {
  const double* n2;
  const double* in2;
  double* out;
  double* flag;
};

// Per-iteration device scalars of rBiCGStab (one 64-byte record per iteration).
struct BiIter {
  double rho;    // r~^T r_i            (written by iteration i-1 or the setup)
  double rr;     // ||r_i||^2
  double sigma;  // r~^T v_i            (v projected)
  double ss;     // ||s_i||^2
  double ts;     // t_i^T s_i           (t projected)
  double tt;     // ||t_i||^2
  double flag;   // 0 normal, 1 exact exit (s = 0), 2 breakdown
  double stop;   // 1: this iteration is not run (set by its bicg_p; gates the rest)
};

}  // namespace rk

// ----------------------------------------------------------------- objects
struct ProfAgg {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
};

struct rk_ctx {
  int device = 0, rank = 0, nranks = 1, sms = 148;
  int64_t l2_bytes = 0;         // L2 capacity (chain policy)
  bool pdl = true;              // programmatic dependent launch (env RK_NO_PDL: off)
  int pdl_mode = 3;             // RK_PDL_MODE (chain.cu): default 3 = the chain overlaps its predecessor, its successor does not
  bool pdl_skip_next = false;   // set by a chain launch (mode 2)
  const double* gate = nullptr; // copied into the kernels launched while set (rBiCGStab lookahead)
  bool defer_coef = true;        // bproject: deferred block-dot finalisation (RK_DEFER_COEF=0: off)
  int bupd_bulk = 1;             // bulk-copy-fed Gram-corrected update: 0 off, 1 large N, 2 always (RK_BUPD_BULK)
  int bdot_bulk = 1;             // bulk-copy-fed bdot: 0 off, 1 large N, 2 always (RK_BDOT_BULK)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double* partials = nullptr;
  double* dpartials = nullptr;  // deferred block-dot partials (read by the next kernel)
  size_t partials_cap = 0;      // doubles
  unsigned* counter = nullptr;
  int64_t launches = 0;
  // collective launches issued on several ranks (comm.cpp; rk_comm_count): a
  // group (comm_group_begin/end, allreduce2) counts once, as NCCL launches it
  int64_t n_allreduce = 0, n_halo = 0;
  int comm_depth = 0;
  bool comm_pend_ar = false, comm_pend_halo = false;
  // profiling
  bool prof_on = false;
  std::string prof_filter;
  int prof_every = 1;           // bracket every n-th matching launch
  int64_t prof_seen = 0;
  struct Pending {
    std::string cls;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, ProfAgg> agg;
#ifdef RK_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  // in-process rank group (comm.cpp, "RKLOCAL:" uids): ranks are contexts of
  // one process driven by separate host threads; halos are device copies
  // ordered by events, all-reduces sum the ranks' partials in rank order
  struct LocalGroup* lgrp = nullptr;
  cudaEvent_t lev[2] = {nullptr, nullptr};
  // resident CTAs per SM of each kernel instantiation (grid = SMs x occupancy)
  std::unordered_map<const void*, int> occ_cache;
};

struct rk_op {
  rk_ctx* ctx = nullptr;
  rk_grid g{};
  int S = 7;                    // 7, 19 or 27 (canonical layout)
  int64_t N = 0, P = 0;
  double* bands = nullptr;      // [S][N] canonical bands, then [N] 1/D (invd())
  double* gbands = nullptr;     // several ranks: [S + 1][2 BGHOST][P] neighbours' band planes
                                //   (lower BGHOST planes from below, then upper from above; 0 at
                                //   a non-periodic global boundary), for the fused chains
  double* rscratch_base = nullptr;   // padded copy of a caller's rhs (rk_precond_apply, ranks > 1)
  const double* invd() const { return bands + (int64_t)S * N; }
  int64_t epoch = 0;
  // scratch (padded) for rk_op_apply / rk_precond_apply
  double* scratch_base[2] = {nullptr, nullptr};
  double* scratch[2] = {nullptr, nullptr};
  int wrapz = 0;
  std::vector<int8_t> user_offsets;   // caller's band order (for rk_op_update_bands)
  bool no_chain = false;              // env RK_NO_CHAIN: disable the fused TMA chain
  bool force_chain = false;           // env RK_FORCE_CHAIN: use it below the L2 threshold (tests)
};

namespace rk {

// Every librk launch goes through a Launch: it counts the launch and, with
// profiling on, brackets it with CUDA events on the context stream.
struct Launch {
  rk_ctx* ctx;
  bool on = false;
  size_t idx = 0;
  Launch(rk_ctx* c, const char* cls, double bytes) : ctx(c) {
    ++ctx->launches;
    if (ctx->prof_on && (ctx->prof_filter.empty() || strstr(cls, ctx->prof_filter.c_str())) &&
        (ctx->prof_seen++ % ctx->prof_every) == 0) {
      on = true;
      rk_ctx::Pending p;
      p.cls = cls;
      p.bytes = bytes;
      if (ctx->pool.size() < 2) {
        cudaEvent_t e;
        for (int q = 0; q < 64; ++q) {
          RK_CUDA(cudaEventCreate(&e));
          ctx->pool.push_back(e);
        }
      }
      p.a = ctx->pool.back();
      ctx->pool.pop_back();
      p.b = ctx->pool.back();
      ctx->pool.pop_back();
      RK_CUDA(cudaEventRecord(p.a, ctx->stream));
      ctx->pending.push_back(p);
      idx = ctx->pending.size() - 1;
    }
  }
  void done() {
    RK_CUDA(cudaGetLastError());
    if (on) RK_CUDA(cudaEventRecord(ctx->pending[idx].b, ctx->stream));
  }
};

// Every librk kernel is launched with programmatic stream serialization
// (PDL): the next kernel's CTAs may become resident while this kernel's last
// CTAs still run; each kernel begins with RK_PDL_ENTRY (griddepcontrol.wait:
// the predecessor grid has completed and its memory is visible; then
// launch_dependents), so the overlap hides launch latency and tails without
// changing any result.
template <typename... KArgs, typename... Args>
void launch_pdl_if(rk_ctx* ctx, bool allow, void (*kern)(KArgs...), dim3 grid, dim3 blk,
                   size_t smem, Args&&... args);

#define RK_PDL_ENTRY()                                         \
  do {                                                         \
    asm volatile("griddepcontrol.wait;" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)
// a gated kernel (the speculative next rBiCGStab iteration) returns at once
#define RK_GATE(g)                        \
  do {                                    \
    if ((g) != nullptr && *(g) != 0.0) return; \
  } while (0)

template <typename... KArgs, typename... Args>
void launch_pdl_if(rk_ctx* ctx, bool allow, void (*kern)(KArgs...), dim3 grid, dim3 blk,
                   size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = blk;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = allow ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

template <typename... KArgs, typename... Args>
void launch_pdl(rk_ctx* ctx, void (*kern)(KArgs...), dim3 grid, dim3 blk, size_t smem,
                Args&&... args) {
  const bool allow = ctx->pdl && !ctx->pdl_skip_next;
  ctx->pdl_skip_next = false;
  launch_pdl_if(ctx, allow, kern, grid, blk, smem, std::forward<Args>(args)...);
}

// fused chain (chain.cu): max stages per launch for this operator (0 = unavailable)
int chain_max_stages(const rk_op* op);
void chain_launch(rk_op* op, int nst, const int* kinds, const double* omegas, const double* xin,
                  const double* r, double* out_t, double* out_mid, double* out,
                  const int* local = nullptr, int zb = 0, const XScale* xs = nullptr);
// true when chain_run can take an XScale (the first launch is a fused 19-point
// chain launch with stage 0 = CK_SPMV1)
bool chain_scales_input(const rk_op* op);
// Runs n chained stencil stages; fused (TMA) launches of up to chain_max_stages()
// stages when available, else one stencil launch per stage.  za/zb: padded scratch.
// local[q] != 0: stage q is a local sweep of the block-Jacobi preconditioner
// (couplings across z-blocks of zbs planes dropped; reading R17).
void chain_run(rk_op* op, const std::vector<int>& kinds, const std::vector<double>& om,
               const double* xin, const double* r, double* out_t, double* out_mid, double* out,
               double* za, double* zb, const std::vector<int>& local = {}, int zbs = 0,
               const XScale* xs = nullptr);

// ------------------------------------------------------------ launch layer
// All kernels are launched through these wrappers (stencil.cu, blockops.cu, bicg.cu).  Each
// increments ctx->launches and, when profiling, is bracketed by events.
void init_ctx_kernels(rk_ctx* ctx);
// zb > 0: local sweep of the block-Jacobi preconditioner (z-blocks of zb planes)
void stencil(rk_op* op, int mode, const double* x, const double* r, double* out0,
             double* out1, double omega, double* red_out, int zb = 0);
void bdot(rk_ctx* ctx, const std::vector<const double*>& cols, const double* w, int64_t N,
          double* out);
// reduce = false: the dots stay rank-local (the caller all-reduces them with
// other values in one collective)
void bupd(rk_ctx* ctx, const std::vector<const double*>& cols, const double* g, double gscale,
          double* w, int64_t N, const std::vector<const double*>& dots, double* red_out,
          CoefIn cin = CoefIn{}, bool reduce = true);
// Recycle projection w <- w - C (C^T w) (+ dots of the new w, as bupd);
// eta <- C^T w.  One rank: the block dot leaves per-CTA partials and the
// update kernel sums them (no last-CTA finalisation between the two);
// otherwise bdot + allreduce + bupd.
void bproject(rk_ctx* ctx, const std::vector<const double*>& cols, double* w, int64_t N,
              double* eta, const std::vector<const double*>& dots, double* red_out,
              bool reduce = true);
// [Q^T w, Q^T v] in one read of Q (Gram-corrected CGS2, R19)
void bdot2(rk_ctx* ctx, const std::vector<const double*>& cols, const double* w, const double* v,
           int64_t N, double* out_w, double* out_v);
// w <- w - Q h with h = 2 g - G g (G from the lagged Gram rows), ||w||^2 -> red_out
void bupd_gram(rk_ctx* ctx, const std::vector<const double*>& cols, int k, const double* g,
               const double* grow, double* hout, double* w, int64_t N, double* red_out);
void normalize(rk_ctx* ctx, double* w, int64_t N, const double* nrm2, const double* nin2,
               double* flag);
void lincomb(rk_ctx* ctx, const std::vector<const double*>& cols, const double* coef, int nout,
             const LcOut& lo, int64_t N);
void proj(rk_ctx* ctx, const std::vector<const double*>& C, const std::vector<const double*>& U,
          const double* xi, double* r, double* x, int64_t N, double* red_out);
// [q_0 .. q_{k-1}] <- [q_0 .. q_{k-1}] T in place, T k x kout (column-major),
// outputs into the first kout columns (kout = -1: square).
// T: DEVICE k x k column-major; T_host (same matrix on the host), when given,
// is passed in the kernel's parameter space instead (rotate_cb_kernel)
void rotate(rk_ctx* ctx, const std::vector<double*>& cols, const double* T, int64_t N, int kout = -1,
            const double* T_host = nullptr);
// also decides whether iteration `cur` runs at all (lookahead): it stops when
// the previous iteration ended the loop (flag / sigma), converged
// (||r|| <= thr_conv), diverged (||r|| > thr_div) or rho == 0; cur->stop gates
// the rest of the iteration's kernels
void bicg_p(rk_op* op, const double* r, double* p, const double* v, double* z, double wl,
            bool jacobi, BiIter* cur, const BiIter* prev, int first, double thr_conv, double thr_div);
// rBiCGStab lines 7a + 8 in two launches (reading R20): the block dot of
// [C, r~] with v, then one kernel for sigma, v -= C eta, alpha, s, the first
// sweep of s_hat (z) and ||s||^2.  ctr = C^T r~ (k values, per solve).  On
// several ranks the block dot is finalised into `stage` (k + 1 values) and
// all-reduced once between the two kernels; ||s||^2 stays rank-local (the
// caller all-reduces it with t^T s, t^T t).  Returns false (nothing
// launched) where it does not apply.
bool bicg_proj_s(rk_op* op, const std::vector<const double*>& C, double* v, const double* rtl,
                 const double* ctr, double* eta, const double* r, double* s, double* z, double wl,
                 bool jacobi, BiIter* cur, double* stage);
void bicg_s(rk_op* op, const double* r, const double* v, double* s, double* z, double wl,
            bool jacobi, BiIter* cur);
void bicg_xr(rk_ctx* ctx, double* x, double* r, const double* s, const double* t, const double* ph,
             const double* sh, const double* rt, int64_t N, BiIter* cur, BiIter* next, double* xi,
             const double* eta1, const double* eta2, int k);
void bicg_setup(rk_ctx* ctx, double* xi, const double* eta0, int k, BiIter* it0);
int validate_bands(rk_op* op);
// band S := 1 / D (the Jacobi sweeps' reciprocal, computed once per matrix
// epoch; 1.0 / D is correctly rounded, so every kernel sees the same bits)
void compute_invdiag(rk_op* op);
// one multicolour SOR pass over the cells of `colour` (0..7), in place on the
// padded vector z (SSOR preconditioner, reading R18)
void colour_sweep(rk_op* op, double* z, const double* r, double omega, int colour);

// communication (comm.cpp): no-ops for one rank
// Ghost planes of the padded vector v from the z-neighbours, `depth` planes
// per side (<= GHOST).
void halo(rk_op* op, const double* v, int depth = 1);
// General neighbour exchange of `count` doubles: this rank's lo_src goes to
// the lower neighbour's hi_dst, its hi_src to the upper neighbour's lo_dst.
void exchange(rk_op* op, const double* lo_src, const double* hi_src, double* lo_dst, double* hi_dst,
              size_t count);
void allreduce(rk_ctx* ctx, double* buf, int n);
// one NCCL launch for the collectives issued in between (no-op on one rank
// and for in-process rank groups)
void comm_group_begin(rk_ctx* ctx);
void comm_group_end(rk_ctx* ctx);
// two reduction outputs (not adjacent in memory) in one collective launch
void allreduce2(rk_ctx* ctx, double* a, int na, double* b, int nb);
// in-process rank groups (tests of the multi-rank schedule on one device)
bool local_uid(const uint8_t* uid);
void local_join(rk_ctx* ctx, const uint8_t* uid);
void local_leave(rk_ctx* ctx);

}  // namespace rk
