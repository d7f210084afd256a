/*
 * rk.h -- C-ABI of librk, the B200 (sm_100a) hot path of the recycling
 * Krylov solvers of arXiv:1501.03358 (Amritkar, de Sturler, Swirydowicz,
 * Tafti, Ahuja): rGCROT(m,k) (Alg. 3), rBiCGStab with
 * one recycle space (Alg. 4), their k = 0 special cases GMRES(m)
 * (Alg. 1) and BiCGStab (Alg. 2), and the hybrid
 * rGCROT -> rBiCGStab sequence strategy.
 *
 * Conventions (apply to every entry point unless stated otherwise)
 *  - Vectors are fp64, the caller's LOCAL z-slab of the grid in x-fastest
 *    order n = i + nx*(j + ny*k), nz_local planes, no ghosts.
 *    "device" pointers are CUDA device memory on the context's device;
 *    "host" pointers are ordinary host memory.
 *  - Ownership: the caller owns every pointer it passes.  librk copies
 *    bands and recycle spaces into memory it owns; export copies out.
 *  - Streams: all work is enqueued on the context stream.  Functions that
 *    return results (rk_solve*, rk_op_apply, rk_precond_apply, exports)
 *    return after that stream has synchronised.
 *  - Errors: API/runtime failures return an rk_status != RK_OK and set a
 *    thread-local message readable with rk_last_error().  No C++ exception
 *    crosses the ABI.  Numerical outcomes (breakdown, no convergence,
 *    instability) are NOT errors: they are rk_report.outcome.
 *  - Threading: one context per host thread and stream.
 *  - Multi-GPU: one process per GPU; every rank calls every function
 *    collectively with identical arguments except the slab data.
 */
#ifndef RK_H
#define RK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rk_ctx rk_ctx;
typedef struct rk_op rk_op;
typedef struct rk_solver rk_solver;

typedef enum {
  RK_OK = 0,
  RK_EINVAL = 1,       /* bad argument (sizes, offsets, truncation violated, NULL) */
  RK_ECUDA = 2,        /* CUDA runtime error */
  RK_ENCCL = 3,        /* NCCL error */
  RK_ENOMEM = 4,       /* device allocation failed */
  RK_ESTATE = 5,       /* call not valid in the object's current state */
  RK_EUNSUPPORTED = 6  /* option not implemented */
} rk_status;

/* Solve outcome (SURVEY.md §5 failure detection). */
typedef enum {
  RK_CONVERGED = 0,    /* ||b - A x||_2 <= tol ||b||_2 (true residual)            */
  RK_MAX_MATVECS = 1,  /* Krylov matvec budget exhausted                           */
  RK_BREAKDOWN = 2,    /* rho, sigma, tau or omega exactly 0 (Alg. 2/4 line 5)     */
  RK_STAGNATION = 3,   /* reserved                                                 */
  RK_UNSTABLE = 4,     /* ||r_i|| > divergence_factor ||r_0|| ("unstable") */
  RK_DRIFT = 5         /* rBiCGStab updated residual converged, certified did not  */
} rk_outcome;

/* GMRES == rGCROT with k_max = 0; BICGSTAB == rBiCGStab with k = 0. */
typedef enum { RK_GMRES = 0, RK_RGCROT = 1, RK_BICGSTAB = 2, RK_RBICGSTAB = 3 } rk_method;

/* Grid of the operator.  Global nx x ny x nz_global; this rank owns planes
 * [z0, z0 + nz_local).  periodic_mask: bit0 x, bit1 y, bit2 z. */
typedef struct {
  int64_t nx, ny, nz_global, z0, nz_local;
  uint32_t periodic_mask;
} rk_grid;

/* Jacobi(5+1) preconditioner: z = w_l D^-1 r; (sweeps-1) x
 * z += w_l D^-1 (r - A_l z); then z += w_g D^-1 (r - A z).  kind 0 = none.
 * zblocks <= 1: A_l = A (every sweep global, reading D9).  zblocks = P > 1:
 * the paper's "sweeps ... on the local sub-domains" -- A_l drops every
 * coupling between the P equal z-blocks (R17); requires P | nz and,
 * on several ranks, that every rank owns whole blocks (those sweeps then
 * exchange no halo).  RK_EINVAL otherwise.
 * kind 2 = SSOR (R18): from z = 0, `sweeps` x
 * (forward then backward multicolour SOR pass, colour = (i&1) + 2(j&1) +
 * 4(k&1), relaxation omega_local) and one global point-Jacobi sweep with
 * omega_global; periodic axes need even extents (RK_EINVAL otherwise). */
typedef struct {
  int kind;            /* 0 none, 1 jacobi, 2 ssor                  */
  int sweeps;          /* local relaxed sweeps (paper: 5)           */
  double omega_local;  /* 0.8 (reading D9)                          */
  double omega_global; /* 1.0 (reading D9)                          */
  int zblocks;         /* block-Jacobi z-blocks (0/1 = global)      */
} rk_precond;

typedef struct {
  rk_method method;
  int m;               /* inner cycle length (rGCROT/GMRES)                 */
  int k_max;           /* max recycle dimension                             */
  int k_keep;          /* k_t: dimension after truncation       */
  int select_count;    /* p1: candidates added per cycle, 0..2  */
  int ortho;           /* 0 = CGS2 (block classical Gram-Schmidt, twice);   
                        * 1 = Gram-corrected CGS2: coefficients (2I - G) Q^T w
                        * with G = Q^T Q from lagged dots, one update pass  
                        * (R19; falls back to 0 for odd N)        */
  int trunc;           /* 0 = T1 (drop the oldest columns);     
                        * 1 = T2 (keep the directions of range(C) with the 
                        * smallest principal angles to the cycle's image  
                        * space A_hat V_m; R13)       */
  rk_precond pc;
  double tol;          /* default tolerance (rk_solve's tol overrides)      */
  int64_t max_matvecs; /* Krylov matvec budget per solve (paper: 2000)      */
  double divergence_factor; /* UNSTABLE threshold (1e4)         */
} rk_config;

typedef struct {
  int32_t outcome;               /* rk_outcome                                   */
  int32_t k_after;               /* recycle dimension after the solve            */
  int64_t krylov_matvecs;        /* preconditioned operator applications in the Krylov loop */
  int64_t operator_applications; /* other applications of A: true residuals, refresh, certification */
  int64_t cycles_or_iters;       /* rGCROT cycles or rBiCGStab iterations        */
  double bnorm;                  /* ||b||_2                                      */
  double final_true_res;         /* ||b - A x||_2 at exit                        */
  double final_updated_res;      /* preconditioned LS residual (rGCROT) / updated ||r|| (rBiCGStab) */
  double seconds;                /* host wall time of the solve                  */
  int64_t history_len;
} rk_report;

/* Thread-local message describing the last non-OK status. */
const char* rk_last_error(void);

/* Library build/version string. */
const char* rk_version(void);

/* NCCL unique id for multi-GPU bootstrap (rank 0 calls it and broadcasts
 * the 128 bytes through torch.distributed).  RK_EUNSUPPORTED if librk was
 * built without NCCL. */
rk_status rk_nccl_unique_id(uint8_t out[128]);

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t
 * (e.g. torch.cuda.current_stream().cuda_stream) or NULL for a library-
 * owned non-blocking stream.  uid must be NULL iff nranks == 1; it is the
 * 128-byte NCCL unique id (one process per GPU, the product path), or the
 * bytes "RKLOCAL:<name>" zero-padded: an in-process rank group <name> whose
 * nranks contexts (one per host thread, any devices) exchange halos by
 * device copies and sum all-reduces on the host in rank order -- the same
 * multi-rank schedule without NCCL, for tests on a one-GPU box. */
rk_status rk_ctx_create(int device, int rank, int nranks, const uint8_t* uid,
                        void* cuda_stream, rk_ctx** out);
void rk_ctx_destroy(rk_ctx* ctx);

/* Create a grid operator A in banded storage.
 * offsets: nbands x 3 int8 (dx, dy, dz), each in {-1, 0, 1}, exactly one
 * (0,0,0) (the diagonal, nonzero everywhere).  bands: DEVICE pointer,
 * [nbands][nz_local][ny][nx] fp64, band d multiplies x at offset d.
 * A coefficient reaching outside a non-periodic axis must be exactly 0
 * (SPEC S:39): checked on the device, RK_EINVAL otherwise.  librk copies the
 * bands (reordered into its canonical 7-, 19- or 27-point layout). */
rk_status rk_op_create(rk_ctx* ctx, const rk_grid* grid, int nbands,
                       const int8_t* offsets, const double* bands, rk_op** out);
/* New matrix epoch (same offsets): copies new bands, invalidates every
 * solver's C (it is rebuilt by QR of A U on the next solve, Alg. 3 l.1a). */
rk_status rk_op_update_bands(rk_op* op, const double* bands);
void rk_op_destroy(rk_op* op);

/* y = A x (O1 / kernel K1).  DEVICE pointers, no ghosts. */
rk_status rk_op_apply(rk_op* op, const double* x, double* y);
/* z = M^-1 r (O2 / kernel K2 chain).  DEVICE pointers. */
rk_status rk_precond_apply(rk_op* op, const rk_precond* pc, const double* r, double* z);

/* Solver bound to an operator.  Allocates the workspace for (m, k_max). */
rk_status rk_solver_create(rk_op* op, const rk_config* cfg, rk_solver** out);
void rk_solver_destroy(rk_solver* s);
/* Hybrid switch: keeps U, invalidates C (reading D3). */
rk_status rk_solver_set_method(rk_solver* s, rk_method method);
/* Recycle space.  U (and optionally C) are DEVICE pointers to k
 * column-major local columns with leading dimension ld >= N_local.  C == NULL
 * -> QR refresh C R = op(U) on the next solve, op = M^-1 A for rGCROT and A
 * for rBiCGStab (reading D3).  R is a HOST k x k column-major upper
 * triangular matrix or NULL (= I); it is absorbed into U (U <- U R^-1,
 * reading D14).  A given C must satisfy op(U) = C R for the solver's current
 * method.  k = 0 empties the space.  k <= k_max. */
rk_status rk_recycle_set(rk_solver* s, int k, const double* U, const double* C,
                         const double* R, int64_t ld);
/* Current recycle dimension k (query before rk_recycle_export). */
rk_status rk_recycle_dim(rk_solver* s, int* k);
/* Copies U, C (DEVICE, ld) and R (HOST k x k, always I after absorption):
 * the RecycleSpace dump of SPEC S:293-294 ("so hybrid runs can be
 * checkpointed"); rk_recycle_set with the exported U and C (and R = NULL)
 * restores it bit for bit.  Any of U, C, R may be NULL. */
rk_status rk_recycle_export(rk_solver* s, double* U, double* C, double* R, int64_t ld);

/* Solve A x = b (rGCROT/GMRES: Alg. 3/1 left-preconditioned; rBiCGStab/
 * BiCGStab: Alg. 4/2 right-preconditioned).  b, x DEVICE; x holds x0 on
 * entry (the paper always uses x0 = 0) and the solution on exit.
 * tol <= 0 uses cfg.tol.  rep may be NULL. */
rk_status rk_solve(rk_solver* s, const double* b, double* x, double tol, rk_report* rep);
/* Same with HOST b and x: the host<->device copies are part of the call. */
rk_status rk_solve_host(rk_solver* s, const double* b_host, double* x_host, double tol,
                        rk_report* rep);
/* HOST b, HOST initial guess x0_host (NULL: x0 = 0, the paper's x_hat = 0,
 * nothing is uploaded or cleared for it), HOST solution x_host
 * (written on exit; may alias x0_host).  Copies are part of the call. */
rk_status rk_solve_host_ex(rk_solver* s, const double* b_host, const double* x0_host,
                           double* x_host, double tol, rk_report* rep);
/* Pipelined host-buffer solves for a sequence of systems (x0 = 0):
 * the upload of the next right-hand side and the download of the previous
 * solution run on the context's copy engine while the current system solves.
 *   rk_stage_rhs    queues the copy of b_host (N_local doubles, pinned for
 *                   overlap) into the solver's staging slot `slot` (0 or 1)
 *                   and returns at once.  A slot may be restaged once the
 *                   rk_solve_staged call that used it has returned.
 *   rk_solve_staged solves with the right-hand side staged in `slot` (it
 *                   waits for that copy on the device), then queues the copy
 *                   of x to x_host and returns without waiting for it.
 *   rk_host_sync    waits for every queued copy; afterwards the x_host
 *                   buffers hold the solutions, and work queued later on the
 *                   library stream is ordered after the copies.
 * b_host and x_host must stay valid, and x_host unread, until rk_host_sync.
 * Errors: RK_EINVAL (NULL, slot not 0/1, slot never staged). */
rk_status rk_stage_rhs(rk_solver* s, int slot, const double* b_host);
rk_status rk_solve_staged(rk_solver* s, int slot, double* x_host, double tol, rk_report* rep);
rk_status rk_host_sync(rk_solver* s);
/* Residual history of the last solve (SolveReport
 * residual_history): rows (krylov_matvecs, ||b-Ax|| or NaN,
 * preconditioned / updated ||r||).  out is HOST [cap][3]; *len = rows. */
rk_status rk_history(rk_solver* s, double* out, int64_t cap, int64_t* len);
/* Per-step trace of the last solve, for per-kernel parity against a CPU
 * reference (the values librk's kernels produced, as read by the host).
 * what = 0: one record per rGCROT/GMRES cycle (Alg. 3 lines 4-12):
 *   k, m_eff, rho = ||r|| (line 4), |g_{m+1}| (LS residual), then
 *   H_ ((m_eff+1) x m_eff, column-major; lines 7-10), B (k x m_eff,
 *   column-major; line 6b: B(:,j) = C^T w_j), y (m_eff; line 12).
 * what = 1: six doubles per rBiCGStab/BiCGStab iteration (Alg. 4 lines
 *   4-15): rho_i = r~^T r_i, sigma_i = r~^T v_i (v projected, line 7a),
 *   ||s_i||^2, t_i^T s_i, t_i^T t_i (t projected, line 12a; omega_i =
 *   t^T s / t^T t), ||r_{i+1}||^2.
 * out: HOST [cap] doubles (NULL to query); *len = doubles available. */
rk_status rk_trace(rk_solver* s, int what, double* out, int64_t cap, int64_t* len);
/* Workspace audit: number of N_local-length vectors allocated. */
rk_status rk_solver_workspace(rk_solver* s, int64_t* nvec);

/* ---------------------------------------------------------------------
 * Per-kernel entry points (operations "exported for
 * per-kernel parity", as rk_op_apply / rk_precond_apply are).  Each runs one
 * family of the solvers' block or rBiCGStab kernels -- through the same
 * host launch path, size thresholds and kernel variants the solvers use --
 * on the context stream, and synchronises before returning.
 *   Q: HOST array of ncol DEVICE pointers, each to n fp64 values (one
 *      column of [C V_j], U or C); 1 <= ncol <= 80 (RK_EINVAL otherwise).
 *   Every other vector or coefficient pointer is DEVICE, fp64.
 *   Single-rank contexts only (RK_EUNSUPPORTED otherwise): the multi-rank
 *   all-reduces of the same kernels are exercised through rk_solve.
 *   Ownership: nothing is retained after the call.
 * --------------------------------------------------------------------- */
/* Block dot (kernel K3; Alg. 3 lines 6a and 6b-9 "[C V_j]^T w", Alg. 4
 * lines 7a / 12a "C^T v"): out_w[c] = Q_c^T w;
 * with v != NULL also out_v[c] = Q_c^T v in the same read of Q (the
 * two-right-hand-side form of DESIGN.md reading R19). */
rk_status rk_block_dot(rk_ctx* ctx, int ncol, const double* const* Q, const double* w,
                       const double* v, int64_t n, double* out_w, double* out_v);
/* Block update (kernel K4; Alg. 3 lines 6c / 9, Alg. 4 line 7a):
 * w <- w - sum_c Q_c g[c]; then red[q] = w_new^T dots[q] for q < ndots
 * (ndots <= 3; dots: HOST array of DEVICE pointers, a NULL entry means
 * w_new itself; red may be NULL iff ndots == 0). */
rk_status rk_block_update(rk_ctx* ctx, int ncol, const double* const* Q, const double* g,
                          double* w, int64_t n, int ndots, const double* const* dots,
                          double* red);
/* Recycle projection (K3 + K4; Alg. 3 lines 1b, 6a-6c, Alg. 4 lines 1c,
 * 7a, 12a): eta = Q^T w; w <- w - Q eta; nrm2 (nullable) =
 * ||w_new||^2.  The update kernel sums the block dot's per-CTA partials
 * itself (deferred finalisation). ncol <= 40. */
rk_status rk_block_project(rk_ctx* ctx, int ncol, const double* const* Q, double* w, int64_t n,
                           double* eta, double* nrm2);
/* Gram-corrected CGS2 update (reading R19, replacing Alg. 3
 * lines 6a-9): h = 2 g - G g with G the Gram matrix of Q = [C, v_0 ..]
 * whose leading k x k block (C^T C) is taken as I and whose other entries
 * are G[i][l] = G[l][i] = grow[i * 80 + l] for rows i >= k, l <= i (row
 * stride 80); then w <- w - Q h, h_out[c] = h[c], nrm2 = ||w_new||^2.
 * 0 <= k <= ncol; n even and every pointer 16-byte aligned. */
rk_status rk_gram_update(rk_ctx* ctx, int ncol, int k, const double* const* Q, const double* g,
                         const double* grow, double* h_out, double* w, int64_t n, double* nrm2);
/* Recycle-space correction (Alg. 3 line 1b, Alg. 4 line 1c, reading D20):
 * r <- r - sum_c C_c xi[c]; if x != NULL (then U != NULL), x <- x + sum_c
 * U_c xi[c]; nrm2 = ||r_new||^2.  C, U: HOST arrays of k (1 <= k <= 48)
 * DEVICE pointers. */
rk_status rk_project_update(rk_ctx* ctx, int k, const double* const* C, const double* const* U,
                            const double* xi, double* r, double* x, int64_t n, double* nrm2);
/* Arnoldi normalisation (Alg. 3 line 10, reading D18): h = sqrt(nrm2[0]);
 * if nin2 != NULL and !(h > 1e-14 sqrt(nin2[0])) (happy breakdown) then
 * w <- 0 and flag[0] = 1, else w <- w / h and flag[0] = 0 (flag nullable). */
rk_status rk_normalize(rk_ctx* ctx, double* w, int64_t n, const double* nrm2, const double* nin2,
                       double* flag);
/* Linear combinations (kernel K5; Alg. 3 lines 13-13a (eq. (6)) and the
 * line-14a extension): for o < nout (<= 5): out[o] = scale[o] *
 * sum_c Q_c coef[o * ncol + c], plus the old out[o] when acc[o] != 0.
 * out: HOST array of nout DEVICE pointers; scale, acc: HOST arrays. */
rk_status rk_lincomb(rk_ctx* ctx, int ncol, const double* const* Q, const double* coef, int nout,
                     double* const* out, const double* scale, const int* acc, int64_t n);
/* Recycle-space rotation (kernel K8; line 1a U <- U R^-1, C <- C~ R^-1 and
 * the line-14a truncation): in place [q_0 .. q_{k-1}] <- [q_0 .. q_{k-1}] T
 * (T: DEVICE k x k column-major); only the first kout (1 <= kout <= k)
 * columns are written.  Q: HOST array of k (1 <= k <= 48) DEVICE pointers. */
rk_status rk_rotate(rk_ctx* ctx, int k, double* const* Q, const double* T, int kout, int64_t n);

/* rBiCGStab per-iteration device scalars (one record per iteration). */
typedef struct {
  double rho;    /* r~^T r_i                                              */
  double rr;     /* ||r_i||^2                                             */
  double sigma;  /* r~^T v_i (v projected, line 7a)                       */
  double ss;     /* ||s_i||^2                                             */
  double ts;     /* t_i^T s_i (t projected, line 12a)                     */
  double tt;     /* ||t_i||^2                                             */
  double flag;   /* 0 normal, 1 exact exit (s = 0), 2 breakdown           */
  double stop;   /* 1: iteration not run (set by its rk_bicg_p)           */
} rk_bicg_iter;
/* Alg. 4 line 6 fused with the first Jacobi sweep of p_hat = M^-1 p
 * (right preconditioning, reading D2): first != 0: p = r;
 * else, unless the stop test below holds, p = r + beta (p - omega v) with
 * alpha = prev->rho / prev->sigma, omega = prev->ts / prev->tt,
 * beta = (cur->rho / prev->rho)(alpha / omega).  z = omega_l p / D
 * (jacobi != 0; D the operator's diagonal band) or z = p.  Stop test (the
 * lookahead decision): prev->flag != 0, prev->sigma == 0,
 * !(sqrt(cur->rr) > thr_conv), cur->rho == 0 or !(sqrt(cur->rr) <= thr_div);
 * cur->stop receives it (p, z untouched when it holds).  cur, prev: DEVICE
 * records (prev ignored when first != 0). */
rk_status rk_bicg_p(rk_op* op, int first, const double* r, double* p, const double* v, double* z,
                    double omega_l, int jacobi, rk_bicg_iter* cur, const rk_bicg_iter* prev,
                    double thr_conv, double thr_div);
/* Alg. 4 line 8 fused with the first sweep of s_hat = M^-1 s: alpha =
 * cur->rho / cur->sigma; s = r - alpha v; z = omega_l s / D (or s);
 * cur->ss = ||s||^2. */
rk_status rk_bicg_s(rk_op* op, const double* r, const double* v, double* s, double* z,
                    double omega_l, int jacobi, rk_bicg_iter* cur);
/* Alg. 4 lines 7a + 8 fused (reading R20): eta = C^T v, sigma = r~^T v -
 * ctr^T eta (ctr = C^T r~), v <- v - C eta, alpha = cur->rho / sigma, then
 * s = r - alpha v, z = omega_l s / D (or s), cur->sigma = sigma,
 * cur->ss = ||s||^2.  C: HOST array of k (1 <= k <= 39) DEVICE pointers;
 * n even and every pointer 16-byte aligned (RK_EUNSUPPORTED otherwise). */
rk_status rk_bicg_project_s(rk_op* op, int k, const double* const* C, double* v, const double* rt,
                            const double* ctr, double* eta, const double* r, double* s, double* z,
                            double omega_l, int jacobi, rk_bicg_iter* cur);
/* Alg. 4 lines 13-15 (+ 10-10a exact exit, breakdown guards of reading
 * D17): alpha = rho / sigma, omega = ts / tt from *cur; mode 2 (no update)
 * if sigma == 0, or tt == 0 or omega == 0 with ss != 0; mode 1 (exact
 * exit) if ss == 0: x += alpha p_hat, r = s; mode 0: x += alpha p_hat +
 * omega s_hat, r = s - omega t.  xi[c] += alpha eta1[c] (+ omega eta2[c])
 * for c < k; cur->flag = mode; next->rho = r~^T r, next->rr = ||r||^2. */
rk_status rk_bicg_xr(rk_op* op, double* x, double* r, const double* s, const double* t,
                     const double* p_hat, const double* s_hat, const double* rt,
                     rk_bicg_iter* cur, rk_bicg_iter* next, double* xi, const double* eta1,
                     const double* eta2, int k);

/* Instrumentation.  Every kernel launch increments a per-context counter.
 * With profiling on, launches of the kernel classes whose names contain
 * `filter` (NULL = all) are bracketed by CUDA events on the context stream;
 * rk_profile_read returns, per class, launches, summed device ms and summed
 * algorithmic bytes. */
rk_status rk_launch_count(rk_ctx* ctx, int64_t* count);
/* Collective launches this context has issued so far on several ranks
 * (the paper's parallel runs are MPI domain decompositions, P:117-118 and
 * P:728 "16 CPU cores ... with MPI parallelism"; "batched so each iteration issues as few collectives as
 * the algorithm allows"; BASELINE north_star): *allreduces = all-reduce
 * launches (a group of all-reduces counts once, as NCCL launches it),
 * *halos = neighbour-exchange launches (one grouped send/recv set; the two
 * halos of one fused chain launch count once).  Both stay 0 on one rank.
 * HOST pointers; either may be NULL. */
rk_status rk_comm_count(rk_ctx* ctx, int64_t* allreduces, int64_t* halos);
rk_status rk_profile_enable(rk_ctx* ctx, int on, const char* filter);
/* Bracket only every `every`-th matching launch (>= 1; default 1): a live
 * sample of a kernel class with less event traffic in a timed region. */
rk_status rk_profile_every(rk_ctx* ctx, int every);
/* names: HOST buffer of cap x 32 chars; launches, ms, bytes: HOST [cap]. */
rk_status rk_profile_read(rk_ctx* ctx, int cap, char* names, int64_t* launches,
                          double* ms, double* bytes, int* n);

#ifdef __cplusplus
}
#endif

#endif /* RK_H */
