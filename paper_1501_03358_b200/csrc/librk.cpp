// librk host engine: contexts, grid operators, and the solver state machines
// of rGCROT(m,k) (Alg. 3), rBiCGStab with one recycle space
// (Alg. 4) and their k = 0 cases GMRES(m) / BiCGStab (Alg. 1 / 2).
//
// All N-length work runs in the sm_100a kernels (stencil.cu, chain.cu, blockops.cu, bicg.cu); this file
// only sequences them, keeps the tiny dense algebra (Hessenberg least
// squares, line-14a coefficient-space algebra, k x k Cholesky) on the host
// and reads back a handful of scalars per rGCROT cycle / rBiCGStab
// iteration.  Readings of the paper are tagged [Dn].
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <limits>
#include <numeric>

#include "rk_internal.h"

using namespace rk;

namespace {

thread_local std::string g_err;

rk_status fail(rk_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

template <class F>
rk_status guarded(F&& f) {
  try {
    f();
    return RK_OK;
  } catch (const Error& e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc&) {
    return fail(RK_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(RK_EINVAL, e.what());
  }
}

// Padded vector: GHOST zero ghost planes below and above the owned planes.
double* alloc_padded(rk_op* op, double** base, int* nvec) {
  const size_t n = (size_t)(op->N + 2 * GHOST * op->P);
  cudaError_t e = cudaMalloc(base, n * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(RK_ENOMEM, "cudaMalloc of a work vector failed");
  }
  RK_CUDA(cudaMemsetAsync(*base, 0, n * sizeof(double), op->ctx->stream));
  if (nvec) ++*nvec;
  return *base + GHOST * op->P;
}

// Several ranks: the BGHOST band planes (all S + 1 arrays, 1/D included)
// next to this slab, from the z-neighbours, for the fused chains' halo
// planes (zero at a non-periodic global boundary).  Once per matrix epoch.
void exchange_ghost_bands(rk_op* op) {
  if (op->ctx->nranks == 1) return;
  const int64_t P = op->P, nzl = op->g.nz_local;
  RK_REQUIRE(nzl >= BGHOST, RK_EINVAL, "slab thinner than the band halo");
  const size_t per = (size_t)(2 * BGHOST) * P;
  if (!op->gbands) {
    cudaError_t e = cudaMalloc(&op->gbands, sizeof(double) * per * (op->S + 1));
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(RK_ENOMEM, "cudaMalloc of the ghost bands failed");
    }
  }
  RK_CUDA(cudaMemsetAsync(op->gbands, 0, sizeof(double) * per * (op->S + 1), op->ctx->stream));
  for (int d = 0; d <= op->S; ++d) {
    const double* b = op->bands + (int64_t)d * op->N;
    double* g = op->gbands + per * d;
    exchange(op, b, b + (nzl - BGHOST) * P, g, g + BGHOST * P, (size_t)(BGHOST * P));
  }
}

int canonical_slot(int S, int dx, int dy, int dz) {
  static const int DX[19] = {0, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1};
  static const int DY[19] = {0, 0, 0, -1, 1, 0, 0, -1, -1, 1, 1, -1, 1, -1, 1, 0, 0, 0, 0};
  static const int DZ[19] = {0, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, -1, 1, 1, -1, -1, 1, 1};
  if (S == 27) {
    int e = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
    return e == 13 ? 0 : (e < 13 ? e + 1 : e);
  }
  for (int d = 0; d < S; ++d)
    if (DX[d] == dx && DY[d] == dy && DZ[d] == dz) return d;
  return -1;
}

void copy_bands(rk_op* op, const int8_t* offs, int nb, const double* src) {
  RK_CUDA(cudaMemsetAsync(op->bands, 0, sizeof(double) * op->S * op->N, op->ctx->stream));
  for (int d = 0; d < nb; ++d) {
    const int c = canonical_slot(op->S, offs[3 * d], offs[3 * d + 1], offs[3 * d + 2]);
    RK_CUDA(cudaMemcpyAsync(op->bands + (int64_t)c * op->N, src + (int64_t)d * op->N,
                            sizeof(double) * op->N, cudaMemcpyDeviceToDevice, op->ctx->stream));
  }
}

// Hessenberg least squares  min ||rho e1 - H y||  by Givens rotations
// (Alg. 1/3 line 12).  H column-major (m+1) x m.  Returns y and |g_{m+1}|.
double ls_givens(const std::vector<double>& H, int m, double rho, std::vector<double>& y) {
  const int ld = m + 1;
  std::vector<double> R(H), g(m + 1, 0.0);
  g[0] = rho;
  for (int j = 0; j < m; ++j) {
    const double a = R[j + j * ld], b = R[j + 1 + j * ld];
    const double r = std::hypot(a, b);
    const double c = r == 0.0 ? 1.0 : a / r, s = r == 0.0 ? 0.0 : b / r;
    for (int l = j; l < m; ++l) {
      const double t1 = R[j + l * ld], t2 = R[j + 1 + l * ld];
      R[j + l * ld] = c * t1 + s * t2;
      R[j + 1 + l * ld] = -s * t1 + c * t2;
    }
    const double t1 = g[j], t2 = g[j + 1];
    g[j] = c * t1 + s * t2;
    g[j + 1] = -s * t1 + c * t2;
  }
  y.assign(m, 0.0);
  for (int j = m - 1; j >= 0; --j) {
    double v = g[j];
    for (int l = j + 1; l < m; ++l) v -= R[j + l * ld] * y[l];
    y[j] = R[j + j * ld] != 0.0 ? v / R[j + j * ld] : 0.0;
  }
  return std::fabs(g[m]);
}

// Truncation T2 (reading R13).  The cycle's image
// space is A_hat V_m = [C V_{m+1}] M with M = [B; H_] ((k+m+1) x m, eq. (5)).
// With M = Q R (Householder), the cosines of the principal angles between
// range(C) and the image are the singular values of Q1 = Q(1:k, :); the left
// singular vectors are the eigenvectors of Q1 Q1^T (cyclic Jacobi).  Returns
// W (k x keep, column-major): the `keep` leading directions, each column
// sign-normalised so that its largest-|.| entry is positive.
std::vector<double> t2_directions(int k, int m, const std::vector<double>& B,
                                  const std::vector<double>& H, int keep) {
  const int n = k + m + 1;
  std::vector<double> A((size_t)n * m, 0.0);  // column-major [B; H]
  for (int j = 0; j < m; ++j) {
    for (int i = 0; i < k; ++i) A[i + (size_t)j * n] = B[i + (size_t)j * k];
    for (int i = 0; i <= m; ++i) A[k + i + (size_t)j * n] = H[i + (size_t)j * (m + 1)];
  }
  // Householder QR: reflectors v_j (stored below the diagonal, v_j[j] = 1)
  std::vector<double> tau(m, 0.0);
  for (int j = 0; j < m; ++j) {
    double nrm = 0.0;
    for (int i = j; i < n; ++i) nrm += A[i + (size_t)j * n] * A[i + (size_t)j * n];
    nrm = std::sqrt(nrm);
    const double a = A[j + (size_t)j * n];
    if (nrm == 0.0) continue;
    const double beta = a >= 0 ? -nrm : nrm;
    const double v0 = a - beta;
    for (int i = j + 1; i < n; ++i) A[i + (size_t)j * n] /= v0;
    tau[j] = (beta - a) / beta;
    A[j + (size_t)j * n] = beta;
    for (int l = j + 1; l < m; ++l) {
      double d = A[j + (size_t)l * n];
      for (int i = j + 1; i < n; ++i) d += A[i + (size_t)j * n] * A[i + (size_t)l * n];
      d *= tau[j];
      A[j + (size_t)l * n] -= d;
      for (int i = j + 1; i < n; ++i) A[i + (size_t)l * n] -= d * A[i + (size_t)j * n];
    }
  }
  // Q (n x m) = H_0 H_1 ... H_{m-1} [I; 0]
  std::vector<double> Q((size_t)n * m, 0.0);
  for (int j = 0; j < m; ++j) Q[j + (size_t)j * n] = 1.0;
  for (int j = m - 1; j >= 0; --j)
    for (int l = 0; l < m; ++l) {
      double d = Q[j + (size_t)l * n];
      for (int i = j + 1; i < n; ++i) d += A[i + (size_t)j * n] * Q[i + (size_t)l * n];
      d *= tau[j];
      Q[j + (size_t)l * n] -= d;
      for (int i = j + 1; i < n; ++i) Q[i + (size_t)l * n] -= d * A[i + (size_t)j * n];
    }
  // K = Q1 Q1^T (k x k), cyclic Jacobi eigen-decomposition K = V diag(e) V^T
  std::vector<double> K((size_t)k * k, 0.0), V((size_t)k * k, 0.0);
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b) {
      double d = 0.0;
      for (int l = 0; l < m; ++l) d += Q[a + (size_t)l * n] * Q[b + (size_t)l * n];
      K[a + (size_t)b * k] = d;
    }
  for (int a = 0; a < k; ++a) V[a + (size_t)a * k] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        const double v = K[a + (size_t)b * k] * K[a + (size_t)b * k];
        tot += v;
        if (a != b) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = K[p + (size_t)q * k];
        if (apq == 0.0) continue;
        const double app = K[p + (size_t)p * k], aqq = K[q + (size_t)q * k];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int r = 0; r < k; ++r) {  // K <- K J
          const double kp = K[r + (size_t)p * k], kq = K[r + (size_t)q * k];
          K[r + (size_t)p * k] = c * kp - sn * kq;
          K[r + (size_t)q * k] = sn * kp + c * kq;
        }
        for (int r = 0; r < k; ++r) {  // K <- J^T K
          const double kp = K[p + (size_t)r * k], kq = K[q + (size_t)r * k];
          K[p + (size_t)r * k] = c * kp - sn * kq;
          K[q + (size_t)r * k] = sn * kp + c * kq;
        }
        for (int r = 0; r < k; ++r) {  // V <- V J
          const double vp = V[r + (size_t)p * k], vq = V[r + (size_t)q * k];
          V[r + (size_t)p * k] = c * vp - sn * vq;
          V[r + (size_t)q * k] = sn * vp + c * vq;
        }
      }
  }
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int a, int b) { return K[a + (size_t)a * k] > K[b + (size_t)b * k]; });
  std::vector<double> W((size_t)k * keep, 0.0);
  for (int j = 0; j < keep; ++j) {
    const int e = idx[j];
    int im = 0;
    for (int i = 1; i < k; ++i)
      if (std::fabs(V[i + (size_t)e * k]) > std::fabs(V[im + (size_t)e * k])) im = i;
    const double sg = V[im + (size_t)e * k] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < k; ++i) W[i + (size_t)j * k] = sg * V[i + (size_t)e * k];
  }
  return W;
}

// SSOR(sweeps) + 1 preconditioner (reading R18): from z = 0, `sweeps` x
// (forward colour passes 0..7, backward 7..0) of in-place multicolour SOR
// with omega_local, then the global point-Jacobi sweep (omega_global) into
// dst (+ ||dst||^2 into red).  zbuf: padded scratch.
void ssor_apply(rk_op* op, const rk_precond& pc, const double* r, double* dst, double* zbuf,
                double* red) {
  RK_CUDA(cudaMemsetAsync(zbuf, 0, sizeof(double) * op->N, op->ctx->stream));
  for (int s = 0; s < pc.sweeps; ++s) {
    for (int c = 0; c < 8; ++c) colour_sweep(op, zbuf, r, pc.omega_local, c);
    for (int c = 7; c >= 0; --c) colour_sweep(op, zbuf, r, pc.omega_local, c);
  }
  stencil(op, red ? SM_SWEEP_NORM : SM_SWEEP, zbuf, r, dst, nullptr, pc.omega_global, red);
}

// SSOR's colouring needs even extents on periodic axes (a wrap would couple
// two cells of one colour)
void check_ssor(const rk_op* op, const rk_precond& pc) {
  if (pc.kind != 2) return;
  const uint32_t pm = op->g.periodic_mask;
  RK_REQUIRE(!(pm & 1) || op->g.nx % 2 == 0, RK_EINVAL, "SSOR: periodic x needs an even nx");
  RK_REQUIRE(!(pm & 2) || op->g.ny % 2 == 0, RK_EINVAL, "SSOR: periodic y needs an even ny");
  RK_REQUIRE(!(pm & 4) || op->g.nz_global % 2 == 0, RK_EINVAL, "SSOR: periodic z needs an even nz");
}

// Block-Jacobi z-blocks [R17]: equal blocks, and on several ranks every rank
// owns whole blocks (its local sweeps then need no halo exchange).
void check_zblocks(const rk_op* op, const rk_precond& pc) {
  if (pc.zblocks <= 1) return;
  RK_REQUIRE(op->g.nz_global % pc.zblocks == 0, RK_EINVAL, "zblocks must divide nz");
  const int64_t zb = op->g.nz_global / pc.zblocks;
  RK_REQUIRE(op->g.z0 % zb == 0 && op->g.nz_local % zb == 0, RK_EINVAL,
             "every rank must own whole z-blocks (zblocks a multiple of the rank count)");
}

}  // namespace

// --------------------------------------------------------------- solver
struct rk_solver {
  rk_op* op = nullptr;
  rk_ctx* ctx = nullptr;
  rk_config cfg{};
  rk_method method = RK_RGCROT;
  int64_t N = 0;
  int nvec = 0;
  std::vector<double*> bases;                 // for cudaFree
  std::vector<double*> V;                     // max(m+1, 8) padded vectors
  std::vector<double*> Us, Cs;                // k_max + 2 slots each
  std::vector<int> order;                     // recycle space: slot ids, oldest first
  double *x = nullptr, *t = nullptr, *za = nullptr, *zb = nullptr, *rt = nullptr;
  // Arnoldi line 10 folded into the next step's chain (19-point fused chain):
  // the normalised v_{j+1} is written here and swapped into V[j+1]
  double* vspare = nullptr;
  bool nfuse = true;                          // RK_NFUSE=0 keeps normalize_kernel
  double* bdev = nullptr;                     // for rk_solve_host
  // recycle-space validity: C matches the operator of `c_kind` at `c_epoch`
  bool c_valid = true;
  int c_kind = 0;                             // 0: A_hat = M^-1 A (rGCROT), 1: A (rBiCGStab)
  int64_t c_epoch = 0;
  // device scalar arena + pinned host mirror
  double* dsc = nullptr;
  double* hsc = nullptr;
  size_t nsc = 0;
  size_t o_arn = 0, o_misc = 0, o_coef = 0, o_gram = 0, o_T = 0, o_bi = 0, o_eta = 0, o_grow = 0;
  int max_it = 0;
  std::vector<std::array<double, 3>> history;
  // per-step trace of the last solve (rk_trace): every rGCROT cycle's
  // [k, m_eff, rho, LS residual, H_ (m_eff+1 x m_eff), B (k x m_eff), y] and
  // every rBiCGStab iteration's [rho, sigma, ||s||^2, t^T s, t^T t, ||r_next||^2]
  std::vector<double> tr_cyc, tr_bi;
  rk_report last{};
  cudaEvent_t bev[2] = {nullptr, nullptr};    // rBiCGStab lookahead: iteration records landed
  // pipelined host solves (rk_stage_rhs / rk_solve_staged / rk_host_sync)
  cudaStream_t cstream = nullptr;             // copy stream
  double* bstage[2] = {nullptr, nullptr};     // staged right-hand sides
  cudaEvent_t staged_ev[2] = {nullptr, nullptr};
  bool staged_ok[2] = {false, false};
  double* xstage = nullptr;                   // x snapshot being downloaded
  cudaEvent_t xready = nullptr, xcopied = nullptr;
  bool xcopy_pending = false;
  void ensure_pipeline() {
    if (cstream) return;
    RK_CUDA(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      RK_CUDA(cudaMalloc(&bstage[q], sizeof(double) * N));
      RK_CUDA(cudaEventCreateWithFlags(&staged_ev[q], cudaEventDisableTiming));
    }
    RK_CUDA(cudaMalloc(&xstage, sizeof(double) * N));
    RK_CUDA(cudaEventCreateWithFlags(&xready, cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&xcopied, cudaEventDisableTiming));
  }
  void free_pipeline() {
    if (!cstream) return;
    cudaStreamSynchronize(cstream);
    for (int q = 0; q < 2; ++q) {
      cudaFree(bstage[q]);
      cudaEventDestroy(staged_ev[q]);
    }
    cudaFree(xstage);
    cudaEventDestroy(xready);
    cudaEventDestroy(xcopied);
    cudaStreamDestroy(cstream);
    cstream = nullptr;
  }
  bool lookahead = true;                      // RK_BICG_LOOKAHEAD=0 disables

  static constexpr size_t STEP = 2 * (MAXCOL + 1) + 2;  // g1[81] g2[81] nrm2 brk
  // misc slots
  enum { BN2 = 0, XN2, RHAT2, RHO2, TRUE2, MISC_XI = 8 };

  double* arn(int j) { return dsc + o_arn + STEP * j; }
  double* misc(int q) { return dsc + o_misc + q; }
  BiIter* bi(int i) { return reinterpret_cast<BiIter*>(dsc + o_bi) + i; }
  BiIter* hbi(int i) { return reinterpret_cast<BiIter*>(hsc + o_bi) + i; }
  double* eta(int q) { return dsc + o_eta + q * MAXCOL; }

  void fetch(size_t off, size_t n) {
    RK_CUDA(cudaMemcpyAsync(hsc + off, dsc + off, n * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
  }
  void sync() { RK_CUDA(cudaStreamSynchronize(ctx->stream)); }
  double hmisc(int q) { return hsc[o_misc + q]; }

  int kind_for(rk_method m) const { return (m == RK_RGCROT || m == RK_GMRES) ? 0 : 1; }
  bool recycles() const { return method == RK_RGCROT || method == RK_RBICGSTAB; }

  std::vector<const double*> ccols() const {
    std::vector<const double*> v;
    for (int s : order) v.push_back(Cs[s]);
    return v;
  }
  std::vector<const double*> ucols() const {
    std::vector<const double*> v;
    for (int s : order) v.push_back(Us[s]);
    return v;
  }

  // ------------------------------------------------- preconditioner chains
  // Runs n chained stencil stages (CK_SPMV1 / CK_SWEEP / CK_SPMV, chain.cu):
  // the first reads xin; sweeps use r, or t = A xin when stage 0 is CK_SPMV1
  // (t is written to out_t).  out_mid receives stage n-2's output.  Uses the
  // temporally blocked kernel (up to chain_max_stages() stages per launch)
  // when available, else one stencil launch per stage (same arithmetic).
  void run_chain(const std::vector<int>& kinds, const std::vector<double>& om, const double* xin,
                 const double* r, double* out_t, double* out_mid, double* out,
                 const std::vector<int>& local = {}, const XScale* xs = nullptr) {
    chain_run(op, kinds, om, xin, r, out_t, out_mid, out, za, zb, local, zblock(), xs);
  }
  // Line 10 (v_{j+1} = w / h) inside the first launch of step j+1's A_hat
  // chain: saves normalize_kernel's read + write of w (1 W net: the chain
  // stores v_{j+1}) and a launch per Arnoldi step; same arithmetic, so the
  // results are bit-identical to the unfused step
  bool fuse_normalize() {
    if (!nfuse || !jac() || !chain_scales_input(op)) return false;
    if (!vspare) {
      double* b;
      vspare = alloc_padded(op, &b, &nvec);
      bases.push_back(b);
    }
    return true;
  }
  // block-Jacobi: planes per z-block of the local sweeps (0 = all sweeps global) [R17]
  int zblock() const {
    return cfg.pc.zblocks > 1 ? (int)(op->g.nz_global / cfg.pc.zblocks) : 0;
  }

  // Jacobi sweeps 2..sweeps+1 (the first sweep's output is in za):
  // z <- z + w_l D^-1 (r - A_loc z) (sweeps-1 times, local [R17]), then
  // dst = z + w_g D^-1 (r - A z) (global).
  void sweeps(const double* r, double* dst, double* red) {
    const rk_precond& pc = cfg.pc;
    if (!red) {
      std::vector<int> k(pc.sweeps, CK_SWEEP);
      std::vector<double> w(pc.sweeps, pc.omega_local);
      std::vector<int> loc(pc.sweeps, 1);
      w.back() = pc.omega_global;
      loc.back() = 0;
      run_chain(k, w, za, r, nullptr, nullptr, dst, loc);
      return;
    }
    double *zin = za, *zout = zb;
    for (int q = 1; q < pc.sweeps; ++q) {
      stencil(op, SM_SWEEP, zin, r, zout, nullptr, pc.omega_local, nullptr, zblock());
      std::swap(zin, zout);
    }
    stencil(op, SM_SWEEP_NORM, zin, r, dst, nullptr, pc.omega_global, red);
  }
  bool jac() const { return cfg.pc.kind == 1; }
  // Gram-corrected CGS2 [R19] (needs the 16-byte tiled kernels: even N, aligned)
  bool gram_ortho() const { return cfg.ortho == 1 && (N % 2 == 0) && (op->P % 2 == 0); }
  bool ssor() const { return cfg.pc.kind == 2; }
  void ssor_to(const double* r, double* dst, double* red) {
    ssor_apply(op, cfg.pc, r, dst, za, red);
  }

  // dst = M^-1 A v  (left-preconditioned operator, Alg. 3 line 6):
  // stages [t = A v, z1 = w_l t/D], sweeps 2..5 (w_l, local), sweep 6 (w_g)
  // xs: v is the unnormalised w of the previous Arnoldi step, taken as
  // w / h by the chain, which also stores v_{j+1} = w / h (fuse_normalize())
  void apply_ahat(const double* v, double* dst, const XScale* xs = nullptr) {
    if (jac()) {
      std::vector<int> k(cfg.pc.sweeps + 1, CK_SWEEP);
      std::vector<double> w(cfg.pc.sweeps + 1, cfg.pc.omega_local);
      std::vector<int> loc(cfg.pc.sweeps + 1, 1);
      k[0] = CK_SPMV1;
      loc[0] = 0;
      w.back() = cfg.pc.omega_global;
      loc.back() = 0;
      run_chain(k, w, v, nullptr, t, nullptr, dst, loc, xs);
    } else if (ssor()) {
      stencil(op, SM_SPMV, v, nullptr, t, nullptr, 0.0, nullptr);
      ssor_to(t, dst, nullptr);
    } else {
      stencil(op, SM_SPMV, v, nullptr, dst, nullptr, 0.0, nullptr);
    }
  }
  // rBiCGStab: (z1 in za) -> p_hat = M^-1 p (out_mid) and v = A p_hat (out)
  void apply_right(const double* rhs, double* phat, double* v) {
    std::vector<int> k(cfg.pc.sweeps + 1, CK_SWEEP);
    std::vector<double> w(cfg.pc.sweeps + 1, cfg.pc.omega_local);
    std::vector<int> loc(cfg.pc.sweeps + 1, 1);
    w[cfg.pc.sweeps - 1] = cfg.pc.omega_global;
    loc[cfg.pc.sweeps - 1] = 0;
    k.back() = CK_SPMV;
    w.back() = 0.0;
    loc.back() = 0;
    run_chain(k, w, za, rhs, nullptr, phat, v, loc);
  }
  // dst = M^-1 r (r need not be padded), optional ||dst||^2
  void apply_minv(const double* r, double* dst, double* red) {
    if (jac()) {
      stencil(op, SM_SCALE, nullptr, r, za, nullptr, cfg.pc.omega_local, nullptr);
      sweeps(r, dst, red);
    } else if (ssor()) {
      ssor_to(r, dst, red);
    } else {
      RK_CUDA(cudaMemcpyAsync(dst, r, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
      if (red) bdot(ctx, {dst}, dst, N, red);
    }
  }

  // ---------------------------------------------------- line 1a refresh
  // C~ = op(U); C~ = C R by CholQR2 (Gram on the device, k x k Cholesky on
  // the host, in-place rotation C <- C~ R^-1, U <- U R^-1 [D14, D15]);
  // a column whose pivot is <= 1e-12 of the largest is dropped.
  int64_t refresh(int kind) {
    int k = (int)order.size();
    for (int c = 0; c < k; ++c) {
      const int s = order[c];
      if (kind == 0) apply_ahat(Us[s], Cs[s]);
      else stencil(op, SM_SPMV, Us[s], nullptr, Cs[s], nullptr, 0.0, nullptr);
    }
    const int64_t apps = k;
    for (int pass = 0; pass < 2 && !order.empty(); ++pass) {
      for (;;) {
        k = (int)order.size();
        if (k == 0) break;
        auto C = ccols();
        // Gram G = C^T C, two columns of G per read of C (the two-RHS block
        // dot): (k/2)(k+2) W instead of k(k+1) W
        for (int c = 0; c < k; c += 2) {
          if (c + 1 < k)
            bdot2(ctx, C, C[c], C[c + 1], N, dsc + o_gram + (size_t)c * k, dsc + o_gram + (size_t)(c + 1) * k);
          else
            bdot(ctx, C, C[c], N, dsc + o_gram + (size_t)c * k);
        }
        fetch(o_gram, (size_t)k * k);
        sync();
        std::vector<double> G(hsc + o_gram, hsc + o_gram + (size_t)k * k);
        double gmax = 0.0;
        for (int c = 0; c < k; ++c) gmax = std::max(gmax, G[c + c * k]);
        std::vector<double> R((size_t)k * k, 0.0);  // column-major upper
        int bad = -1;
        for (int j = 0; j < k && bad < 0; ++j) {
          double d = 0.5 * (G[j + j * k] + G[j + j * k]);
          for (int i = 0; i < j; ++i) d -= R[i + j * k] * R[i + j * k];
          if (!(d > 0.0) || std::sqrt(d) <= 1e-12 * std::sqrt(gmax)) {
            bad = j;
            break;
          }
          const double rjj = std::sqrt(d);
          R[j + j * k] = rjj;
          for (int l = j + 1; l < k; ++l) {
            double v = 0.5 * (G[j + l * k] + G[l + j * k]);
            for (int i = 0; i < j; ++i) v -= R[i + j * k] * R[i + l * k];
            R[j + l * k] = v / rjj;
          }
        }
        if (bad >= 0) {
          order.erase(order.begin() + bad);
          continue;
        }
        // T = R^-1 (upper triangular), column-major
        std::vector<double> T((size_t)k * k, 0.0);
        for (int col = 0; col < k; ++col) {
          for (int i = col; i >= 0; --i) {
            double v = (i == col) ? 1.0 : 0.0;
            for (int l = i + 1; l <= col; ++l) v -= R[i + l * k] * T[l + col * k];
            T[i + col * k] = v / R[i + i * k];
          }
        }
        std::memcpy(hsc + o_T, T.data(), sizeof(double) * k * k);
        RK_CUDA(cudaMemcpyAsync(dsc + o_T, hsc + o_T, sizeof(double) * k * k,
                                cudaMemcpyHostToDevice, ctx->stream));
        std::vector<double*> Cw, Uw;
        for (int s : order) {
          Cw.push_back(Cs[s]);
          Uw.push_back(Us[s]);
        }
        rotate(ctx, Cw, dsc + o_T, N, -1, hsc + o_T);
        rotate(ctx, Uw, dsc + o_T, N, -1, hsc + o_T);
        sync();  // the pinned T buffer is reused by the second pass
        break;
      }
    }
    c_valid = true;
    c_kind = kind;
    c_epoch = op->epoch;
    return apps;
  }

  void ensure_space(int kind, rk_report& rep) {
    if (order.empty()) {
      c_valid = true;
      c_kind = kind;
      c_epoch = op->epoch;
      return;
    }
    if (!c_valid || c_kind != kind || c_epoch != op->epoch) rep.operator_applications += refresh(kind);
  }

  void record(double mv, double tr, double pr) { history.push_back({mv, tr, pr}); }

  // ------------------------------------------------------ Alg. 3 rGCROT
  void solve_rgcrot(const double* b, double tol, rk_report& rep) {
    const int m = cfg.m;
    const bool recyc = method == RK_RGCROT && cfg.k_max > 0;
    bdot(ctx, {b}, b, N, misc(BN2));
    bdot(ctx, {x}, x, N, misc(XN2));
    fetch(o_misc, 2);
    sync();
    rep.bnorm = std::sqrt(hmisc(BN2));
    const double beta = rep.bnorm;
    if (beta == 0.0) {
      RK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, ctx->stream));
      rep.outcome = RK_CONVERGED;
      rep.final_true_res = 0.0;
      return;
    }
    if (recyc) ensure_space(0, rep);
    // line 1: r_hat = M^-1 (b - A x_hat)
    if (hmisc(XN2) == 0.0) {
      apply_minv(b, V[0], misc(RHAT2));
    } else {
      if (jac()) {
        stencil(op, SM_RESID_SWEEP1, x, b, rt, za, cfg.pc.omega_local, misc(TRUE2));
        sweeps(rt, V[0], misc(RHAT2));
      } else if (ssor()) {
        stencil(op, SM_RESID, x, b, rt, nullptr, 0.0, misc(TRUE2));
        ssor_to(rt, V[0], misc(RHAT2));
      } else {
        stencil(op, SM_RESID, x, b, V[0], nullptr, 0.0, misc(RHAT2));
      }
      rep.operator_applications += 1;
    }
    // line 1b: xi = C^T r_hat ; r0 = r_hat - C xi ; x0 = x_hat + U xi
    auto project = [&]() {
      if (!order.empty()) {
        bdot(ctx, ccols(), V[0], N, misc(MISC_XI));
        proj(ctx, ccols(), ucols(), misc(MISC_XI), V[0], x, N, misc(RHO2));
      } else {
        bdot(ctx, {V[0]}, V[0], N, misc(RHO2));
      }
    };
    project();
    fetch(o_misc, MISC_XI);
    sync();
    // [D6] zero-cycle exit
    if (std::sqrt(hmisc(RHO2)) <= tol * std::sqrt(hmisc(RHAT2))) {
      stencil(op, SM_RESID, x, b, rt, nullptr, 0.0, misc(TRUE2));
      rep.operator_applications += 1;
      fetch(o_misc, MISC_XI);
      sync();
      const double tr = std::sqrt(hmisc(TRUE2));
      if (tr <= tol * beta) {
        rep.outcome = RK_CONVERGED;
        rep.final_true_res = tr;
        rep.final_updated_res = std::sqrt(hmisc(RHO2));
        return;
      }
    }
    int cycle = 0;
    std::vector<double> H, B, y, coef;
    rep.outcome = RK_MAX_MATVECS;
    while (rep.krylov_matvecs < cfg.max_matvecs) {
      if (cycle > 0) project();  // [D20] re-projection at every cycle start
      const int k = (int)order.size();
      normalize(ctx, V[0], N, misc(RHO2), nullptr, nullptr);  // line 4: v1 = r / rho
      auto Q = ccols();
      // line 10 of step j-1 pending in the chain of step j (fuse_normalize)
      XScale pend{nullptr, nullptr, nullptr, nullptr};
      const bool fuse = fuse_normalize();
      for (int j = 0; j < m; ++j) {
        double* w = V[j + 1];
        if (pend.n2) {
          pend.out = vspare;
          apply_ahat(V[j], w, &pend);                         // lines 10 (step j-1) + 6
          std::swap(V[j], vspare);                            // v_{j} now in V[j]
          pend.n2 = nullptr;
        } else {
          apply_ahat(V[j], w);                                // line 6
        }
        Q.push_back(V[j]);
        const int ncol = (int)Q.size();
        double* g1 = arn(j);
        double* g2 = g1 + (MAXCOL + 1);
        auto Qw = Q;
        Qw.push_back(w);
        if (gram_ortho()) {
          // [R19] one read of [C V_j] for g = Q^T w (+ ||w||^2) and the lagged
          // Gram row Q^T v_j, one for w -= Q (2 g - G g); h lands in g2
          bdot2(ctx, Qw, w, V[j], N, g1, dsc + o_grow + (size_t)(k + j) * MAXCOL);
          bupd_gram(ctx, Q, k, g1, dsc + o_grow, g2, w, N, g1 + 2 * (MAXCOL + 1));
        } else {
          bdot(ctx, Qw, w, N, g1);                            // lines 6a-9, CGS pass 1 (+ ||w||^2)
          bupd(ctx, Q, g1, 1.0, w, N, {}, nullptr);
          bproject(ctx, Q, w, N, g2, {nullptr}, g1 + 2 * (MAXCOL + 1));   // CGS pass 2 [D8]
        }
        if (fuse && j + 1 < m)   // line 10 runs inside the next step's chain launch
          pend = XScale{g1 + 2 * (MAXCOL + 1), g1 + ncol, nullptr, g1 + 2 * (MAXCOL + 1) + 1};
        else
          normalize(ctx, w, N, g1 + 2 * (MAXCOL + 1), g1 + ncol, g1 + 2 * (MAXCOL + 1) + 1);  // line 10
      }
      fetch(o_arn, STEP * m);
      fetch(o_misc, MISC_XI);
      sync();
      int m_eff = m;
      for (int j = 0; j < m; ++j)
        if (hsc[o_arn + STEP * j + 2 * (MAXCOL + 1) + 1] != 0.0) {
          m_eff = j + 1;
          break;
        }
      rep.krylov_matvecs += m_eff;
      const double rho = std::sqrt(hmisc(RHO2));
      // assemble H_ (m_eff+1 x m_eff) and B (k x m_eff), both column-major
      H.assign((size_t)(m_eff + 1) * m_eff, 0.0);
      B.assign((size_t)std::max(k, 1) * m_eff, 0.0);
      for (int j = 0; j < m_eff; ++j) {
        const double* h1 = hsc + o_arn + STEP * j;
        const double* h2 = h1 + (MAXCOL + 1);
        // CGS2: h = g1 + g2; Gram-corrected [R19]: h is stored in the g2 slot
        const double g1w = gram_ortho() ? 0.0 : 1.0;
        for (int c = 0; c < k; ++c) B[c + (size_t)j * k] = g1w * h1[c] + h2[c];
        for (int l = 0; l <= j; ++l) H[l + (size_t)j * (m_eff + 1)] = g1w * h1[k + l] + h2[k + l];
        H[j + 1 + (size_t)j * (m_eff + 1)] = std::sqrt(h1[2 * (MAXCOL + 1)]);
      }
      const double prec_res = ls_givens(H, m_eff, rho, y);   // line 12
      tr_cyc.push_back(k);
      tr_cyc.push_back(m_eff);
      tr_cyc.push_back(rho);
      tr_cyc.push_back(prec_res);
      tr_cyc.insert(tr_cyc.end(), H.begin(), H.end());
      tr_cyc.insert(tr_cyc.end(), B.begin(), B.begin() + (size_t)k * m_eff);
      tr_cyc.insert(tr_cyc.end(), y.begin(), y.end());
      std::vector<double> z(k, 0.0);                          // line 12a: z = -B y
      for (int c = 0; c < k; ++c) {
        double v = 0.0;
        for (int j = 0; j < m_eff; ++j) v += B[c + (size_t)j * k] * y[j];
        z[c] = -v;
      }
      // line 14a coefficient-space algebra [D11]
      std::vector<double> zeta(m_eff + 1, 0.0);
      for (int l = 0; l <= m_eff; ++l)
        for (int j = 0; j < m_eff; ++j) zeta[l] += H[l + (size_t)j * (m_eff + 1)] * y[j];
      double gamma = 0.0;
      for (double v : zeta) gamma += v * v;
      gamma = std::sqrt(gamma);
      // columns: V_0..V_{m_eff}, then U (order)
      std::vector<const double*> cols(V.begin(), V.begin() + m_eff + 1);
      for (int s : order) cols.push_back(Us[s]);
      const int ncol = (int)cols.size();
      const int nV = m_eff + 1;
      int nout = 1;
      coef.assign((size_t)MAXOUT * ncol, 0.0);
      LcOut lo;
      std::memset(&lo, 0, sizeof(lo));
      // out0: x += V_m y + U z   (lines 13-13a per eq. (6) [D1])
      for (int j = 0; j < m_eff; ++j) coef[j] = y[j];
      for (int c = 0; c < k; ++c) coef[nV + c] = z[c];
      lo.out[0] = x;
      lo.scale[0] = 1.0;
      lo.acc[0] = 1;
      std::vector<int> newslots;
      std::vector<int> freeslots;
      for (int s = 0; s < (int)Us.size(); ++s)
        if (std::find(order.begin(), order.end(), s) == order.end()) freeslots.push_back(s);
      const bool extend = recyc && cfg.select_count >= 1 && gamma > 1e-14 * rho;
      if (extend) {
        const int s1 = freeslots[0];
        // u1 = dx / gamma ; c1 = V_{m+1} zeta / gamma
        for (int q = 0; q < ncol; ++q) coef[ncol + q] = coef[q];
        for (int l = 0; l <= m_eff; ++l) coef[2 * ncol + l] = zeta[l];
        lo.out[1] = Us[s1];
        lo.scale[1] = 1.0 / gamma;
        lo.out[2] = Cs[s1];
        lo.scale[2] = 1.0 / gamma;
        nout = 3;
        newslots.push_back(s1);
        if (cfg.select_count >= 2) {
          const int pool = std::max(1, m_eff / 2);
          int js = 0;
          for (int j = 1; j < pool; ++j)
            if (std::fabs(y[j]) > std::fabs(y[js])) js = j;
          std::vector<double> hs(m_eff + 1), zh(m_eff + 1), cp(m_eff + 1);
          double sd = 0.0, hn = 0.0;
          for (int l = 0; l <= m_eff; ++l) {
            hs[l] = H[l + (size_t)js * (m_eff + 1)];
            zh[l] = zeta[l] / gamma;
            sd += zh[l] * hs[l];
            hn += hs[l] * hs[l];
          }
          double delta = 0.0;
          for (int l = 0; l <= m_eff; ++l) {
            cp[l] = hs[l] - zh[l] * sd;
            delta += cp[l] * cp[l];
          }
          delta = std::sqrt(delta);
          if (delta > 1e-12 * std::sqrt(hn)) {
            const int s2 = freeslots[1];
            double* cu = coef.data() + 3 * ncol;
            double* cc = coef.data() + 4 * ncol;
            // u2 = (v_js - U B(:,js) - u1 sd) / delta,  u1 = (V_m y + U z) / gamma
            for (int j = 0; j < m_eff; ++j) cu[j] = -y[j] * sd / gamma;
            cu[js] += 1.0;
            for (int c = 0; c < k; ++c) cu[nV + c] = -B[c + (size_t)js * k] - z[c] * sd / gamma;
            for (int l = 0; l <= m_eff; ++l) cc[l] = cp[l];
            lo.out[3] = Us[s2];
            lo.scale[3] = 1.0 / delta;
            lo.out[4] = Cs[s2];
            lo.scale[4] = 1.0 / delta;
            nout = 5;
            newslots.push_back(s2);
          }
        }
      }
      std::memcpy(hsc + o_coef, coef.data(), sizeof(double) * nout * ncol);
      // compact rows: the kernel reads coef[o * ncol + c]
      RK_CUDA(cudaMemcpyAsync(dsc + o_coef, hsc + o_coef, sizeof(double) * nout * ncol,
                              cudaMemcpyHostToDevice, ctx->stream));
      lincomb(ctx, cols, dsc + o_coef, nout, lo, N);
      // line 14: r = b - A x (true residual), first sweep of M^-1 r fused
      if (jac()) stencil(op, SM_RESID_SWEEP1, x, b, rt, za, cfg.pc.omega_local, misc(TRUE2));
      else stencil(op, SM_RESID, x, b, rt, nullptr, 0.0, misc(TRUE2));
      rep.operator_applications += 1;
      fetch(o_misc, MISC_XI);
      sync();
      const double tr = std::sqrt(hmisc(TRUE2));
      record((double)rep.krylov_matvecs, tr, prec_res);
      // line 14a bookkeeping: truncation T1 then append [D11, D21]
      const int p = (int)newslots.size();
      if (p > 0) {
        if (k + p > cfg.k_max) {
          const int keep = std::max(0, cfg.k_keep - p);
          if (cfg.trunc == 1 && keep > 0 && keep <= std::min(k, m_eff)) {
            // T2: [U C] <- [U C] W in place, the first `keep` slots of order
            const std::vector<double> W = t2_directions(k, m_eff, B, H, keep);
            std::memcpy(hsc + o_T, W.data(), sizeof(double) * W.size());
            RK_CUDA(cudaMemcpyAsync(dsc + o_T, hsc + o_T, sizeof(double) * W.size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
            std::vector<double*> Uw, Cw;
            for (int s : order) {
              Uw.push_back(Us[s]);
              Cw.push_back(Cs[s]);
            }
            rotate(ctx, Uw, dsc + o_T, N, keep, hsc + o_T);
            rotate(ctx, Cw, dsc + o_T, N, keep, hsc + o_T);
            order.resize(keep);
            sync();  // the pinned W buffer is reused
          } else {
            order.erase(order.begin(), order.begin() + (k - keep));   // T1
          }
        }
        for (int s : newslots) order.push_back(s);
      }
      ++cycle;
      rep.cycles_or_iters = cycle;
      rep.final_true_res = tr;
      rep.final_updated_res = prec_res;
      if (!std::isfinite(tr)) {
        rep.outcome = RK_BREAKDOWN;
        break;
      }
      if (tr <= tol * beta) {
        rep.outcome = RK_CONVERGED;
        break;
      }
      if (rep.krylov_matvecs >= cfg.max_matvecs) break;
      if (jac()) sweeps(rt, V[0], nullptr);                   // r = M^-1 r_true
      else if (ssor()) ssor_to(rt, V[0], nullptr);
      else RK_CUDA(cudaMemcpyAsync(V[0], rt, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }

  // --------------------------------------------------- Alg. 4 rBiCGStab
  void solve_rbicgstab(const double* b, double tol, rk_report& rep) {
    bdot(ctx, {b}, b, N, misc(BN2));
    bdot(ctx, {x}, x, N, misc(XN2));
    fetch(o_misc, 2);
    sync();
    rep.bnorm = std::sqrt(hmisc(BN2));
    const double beta = rep.bnorm;
    if (beta == 0.0) {
      RK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, ctx->stream));
      rep.outcome = RK_CONVERGED;
      rep.final_true_res = 0.0;
      return;
    }
    const bool recyc = method == RK_RBICGSTAB;
    if (recyc) ensure_space(1, rep);   // [D3] C R = qr(A U) with plain A
    const int k = recyc ? (int)order.size() : 0;
    auto C = recyc ? ccols() : std::vector<const double*>{};
    auto U = recyc ? ucols() : std::vector<const double*>{};
    double *r = V[0], *rtl = V[1], *p = V[2], *v = V[3], *s = V[4], *tt = V[5], *ph = V[6],
           *sh = V[7];
    double* xi = misc(MISC_XI);
    const double wl = cfg.pc.omega_local;
    bool xnz = hmisc(XN2) != 0.0;
    rep.outcome = RK_MAX_MATVECS;
    for (;;) {
      // line 1: r_hat = b - A x_hat
      if (xnz) {
        stencil(op, SM_RESID, x, b, r, nullptr, 0.0, misc(TRUE2));
        rep.operator_applications += 1;
      } else {
        RK_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
      }
      // line 1c: eta = C^T r ; r -= C eta ; xi = -eta ; r~ = r0 [D16]
      if (k > 0) {
        bdot(ctx, C, r, N, eta(2));
        proj(ctx, C, {}, eta(2), r, nullptr, N, &bi(0)->rho);
      } else {
        bdot(ctx, {r}, r, N, &bi(0)->rho);
      }
      bicg_setup(ctx, xi, eta(2), k, bi(0));
      RK_CUDA(cudaMemcpyAsync(rtl, r, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
      if (k > 0) bdot(ctx, C, rtl, N, eta(3));   // C^T r~ for bicg_proj_s [R20]
      fetch(o_bi, 8);
      sync();
      double rr = hbi(0)->rr;
      const double r0n = std::sqrt(rr);
      const double thr_conv = tol * beta, thr_div = cfg.divergence_factor * r0n;
      // One rBiCGStab iteration (lines 5-15) on the stream, ending with the
      // copy of its scalar records to the host and an event.  Iteration j+1
      // is enqueued before the host has read iteration j (lookahead): its
      // bicg_p re-takes the host's stop decision on the device (line 3's
      // test, line 5, the breakdown / exact-exit flags of j, [D17]) and, if
      // it stops, every later kernel of j+1 returns at once (ctx->gate).
      auto enqueue = [&](int j) {
        struct GateReset {
          rk_ctx* c;
          ~GateReset() { c->gate = nullptr; }
        } gate_reset{ctx};
        BiIter* cur = bi(j);
        const BiIter* prev = j ? bi(j - 1) : cur;
        // line 6 + p_hat = M^-1 p (right preconditioning) ; line 7: v = A p_hat
        if (jac()) {
          bicg_p(op, r, p, v, za, wl, true, cur, prev, j == 0, thr_conv, thr_div);
          ctx->gate = j ? &cur->stop : nullptr;
          apply_right(p, ph, v);               // p_hat = M^-1 p ; v = A p_hat
        } else {
          bicg_p(op, r, p, v, ph, 1.0, false, cur, prev, j == 0, thr_conv, thr_div);
          ctx->gate = j ? &cur->stop : nullptr;
          if (ssor()) ssor_to(p, ph, nullptr);   // p_hat = M^-1 p (SSOR, R18)
          stencil(op, SM_SPMV, ph, nullptr, v, nullptr, 0.0, nullptr);
        }
        // line 7a: eta1 = C^T v ; v -= C eta1 ; sigma = r~^T v
        // line 8: alpha = rho / sigma ; s = r - alpha v (+ first sweep of s_hat)
        const bool fused = k > 0 &&
                           bicg_proj_s(op, C, v, rtl, eta(3), eta(0), r, s, jac() ? za : sh, wl, jac(), cur,
                                       eta(4));
        if (!fused) {
          if (k > 0) {
            bproject(ctx, C, v, N, eta(0), {rtl}, &cur->sigma);
          } else {
            bdot(ctx, {rtl}, v, N, &cur->sigma);
          }
          bicg_s(op, r, v, s, jac() ? za : sh, wl, jac(), cur);
        }
        if (jac()) {
          apply_right(s, sh, tt);               // s_hat = M^-1 s ; t = A s_hat (line 12)
        } else {
          if (ssor()) ssor_to(s, sh, nullptr);
          stencil(op, SM_SPMV, sh, nullptr, tt, nullptr, 0.0, nullptr);
        }
        if (k > 0) {                                              // line 12a
          // several ranks: ||s||^2 (left rank-local by bicg_proj_s), t^T s and
          // t^T t -- adjacent in the record -- in ONE all-reduce
          const bool merge = fused && ctx->nranks > 1;
          bproject(ctx, C, tt, N, eta(1), {s, nullptr}, &cur->ts, !merge);
          if (merge) allreduce(ctx, &cur->ss, 3);
        } else {
          bdot(ctx, {s, tt}, tt, N, &cur->ts);
        }
        // lines 13-15 (+13a): omega ; x ; r ; xi ; next rho, ||r||^2
        bicg_xr(ctx, x, r, s, tt, ph, sh, rtl, N, cur, bi(j + 1), xi, eta(0), eta(1), k);
        ctx->gate = nullptr;
        fetch(o_bi + 8 * (size_t)j, 16);
        RK_CUDA(cudaEventRecord(bev[j & 1], ctx->stream));
      };
      const int m0 = rep.krylov_matvecs;
      int i = 0;
      int queued = 0;   // iterations 0 .. queued-1 are on the stream
      int status = -1;
      while (std::sqrt(rr) > tol * beta && rep.krylov_matvecs < cfg.max_matvecs) {  // line 3
        RK_REQUIRE(i + 1 < max_it, RK_ESTATE, "rBiCGStab iteration record overflow");
        if (hbi(i)->rho == 0.0) {                                  // line 5
          status = RK_BREAKDOWN;
          break;
        }
        if (queued == i) enqueue(queued++);
        // lookahead: iteration i+1 runs iff i ends normally, which spends
        // exactly two matvecs per iteration
        if (lookahead && queued == i + 1 && i + 2 < max_it && m0 + 2 * (i + 1) < cfg.max_matvecs)
          enqueue(queued++);
        RK_CUDA(cudaEventSynchronize(bev[i & 1]));
        rep.krylov_matvecs += 2;
        const BiIter hc = *hbi(i);
        if (hc.sigma == 0.0) {
          rep.krylov_matvecs -= 1;   // the oracle stops before t = A s_hat
          status = RK_BREAKDOWN;
          break;
        }
        if (hc.flag == 1.0) {        // ||s|| == 0: lines 10-10a
          rep.krylov_matvecs -= 1;
          ++i;
          rr = 0.0;
          break;
        }
        if (hc.flag == 2.0) {
          status = RK_BREAKDOWN;
          break;
        }
        ++i;
        rr = hbi(i)->rr;
        tr_bi.insert(tr_bi.end(), {hc.rho, hc.sigma, hc.ss, hc.ts, hc.tt, rr});
        record((double)rep.krylov_matvecs, std::numeric_limits<double>::quiet_NaN(), std::sqrt(rr));
        if (!(std::sqrt(rr) <= thr_div)) {   // [D17] instability
          status = RK_UNSTABLE;
          break;
        }
      }
      // a speculative iteration still on the stream gates itself off; the
      // records of a stopped iteration are never read
      rep.cycles_or_iters += i;
      // line 17a: x = x - U xi
      if (k > 0) {
        LcOut lo;
        std::memset(&lo, 0, sizeof(lo));
        lo.out[0] = x;
        lo.scale[0] = -1.0;
        lo.acc[0] = 1;
        lincomb(ctx, U, xi, 1, lo, N);
      }
      // certification [D23]
      stencil(op, SM_RESID, x, b, r, nullptr, 0.0, misc(TRUE2));
      rep.operator_applications += 1;
      fetch(o_misc, MISC_XI);
      sync();
      rep.final_true_res = std::sqrt(hmisc(TRUE2));
      rep.final_updated_res = std::sqrt(rr);
      if (status >= 0) {
        rep.outcome = (rk_outcome)status;
        break;
      }
      if (rep.final_true_res <= tol * beta) {
        rep.outcome = RK_CONVERGED;
        break;
      }
      if (rep.krylov_matvecs >= cfg.max_matvecs) {
        rep.outcome = std::sqrt(rr) <= tol * beta ? RK_DRIFT : RK_MAX_MATVECS;
        break;
      }
      if (i == 0) {
        rep.outcome = RK_DRIFT;
        break;
      }
      xnz = true;  // [D23] restart from x_hat = x
    }
  }
};

// ===================================================================== ABI
extern "C" {

const char* rk_last_error(void) { return g_err.c_str(); }

const char* rk_version(void) {
  return "librk 0.1 (sm_100a, fp64"
#ifdef RK_WITH_NCCL
         ", nccl"
#endif
         ")";
}

rk_status rk_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    RK_REQUIRE(out, RK_EINVAL, "out is NULL");
#ifdef RK_WITH_NCCL
    ncclUniqueId id;
    RK_REQUIRE(ncclGetUniqueId(&id) == ncclSuccess, RK_ENCCL, "ncclGetUniqueId failed");
    std::memcpy(out, &id, 128);
#else
    throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
  });
}

rk_status rk_ctx_create(int device, int rank, int nranks, const uint8_t* uid, void* cuda_stream,
                        rk_ctx** out) {
  return guarded([&] {
    RK_REQUIRE(out, RK_EINVAL, "out is NULL");
    RK_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, RK_EINVAL, "bad rank/nranks");
    RK_REQUIRE((nranks == 1) == (uid == nullptr), RK_EINVAL, "uid must be NULL iff nranks == 1");
    auto* c = new rk_ctx();
    try {
      c->device = device;
      c->rank = rank;
      c->nranks = nranks;
      RK_CUDA(cudaSetDevice(device));
      if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
      } else {
        RK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
      }
      init_ctx_kernels(c);
      if (nranks > 1 && local_uid(uid)) {
        local_join(c, uid);
      } else if (nranks > 1) {
#ifdef RK_WITH_NCCL
        ncclUniqueId id;
        std::memcpy(&id, uid, 128);
        RK_REQUIRE(ncclCommInitRank(&c->comm, nranks, id, rank) == ncclSuccess, RK_ENCCL,
                   "ncclCommInitRank failed");
#else
        throw Error(RK_EUNSUPPORTED, "librk built without NCCL");
#endif
      }
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void rk_ctx_destroy(rk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  cudaFree(c->partials);
  cudaFree(c->dpartials);
  cudaFree(c->counter);
#ifdef RK_WITH_NCCL
  if (c->comm) ncclCommDestroy(c->comm);
#endif
  local_leave(c);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

rk_status rk_op_create(rk_ctx* ctx, const rk_grid* g, int nbands, const int8_t* offsets,
                       const double* bands, rk_op** out) {
  return guarded([&] {
    RK_REQUIRE(ctx && g && offsets && bands && out, RK_EINVAL, "NULL argument");
    RK_REQUIRE(g->nx >= 1 && g->ny >= 1 && g->nz_local >= 1 && g->nz_global >= g->nz_local &&
                   g->z0 >= 0 && g->z0 + g->nz_local <= g->nz_global,
               RK_EINVAL, "bad grid");
    RK_REQUIRE(g->nx <= (1 << 30) && g->ny <= (1 << 30), RK_EINVAL, "grid too large");
    RK_REQUIRE(nbands >= 1 && nbands <= 27, RK_EINVAL, "1..27 bands");
    if (ctx->nranks == 1)
      RK_REQUIRE(g->z0 == 0 && g->nz_local == g->nz_global, RK_EINVAL,
                 "single rank must own the whole grid");
    bool in7 = true, in19 = true, has0 = false;
    std::vector<int> seen(27, 0);
    for (int d = 0; d < nbands; ++d) {
      const int dx = offsets[3 * d], dy = offsets[3 * d + 1], dz = offsets[3 * d + 2];
      RK_REQUIRE(dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1, RK_EINVAL,
                 "offsets must be in {-1,0,1}^3 (one ghost plane)");
      const int e = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
      RK_REQUIRE(!seen[e]++, RK_EINVAL, "duplicate offset");
      if (canonical_slot(7, dx, dy, dz) < 0) in7 = false;
      if (canonical_slot(19, dx, dy, dz) < 0) in19 = false;
      if (!dx && !dy && !dz) has0 = true;
    }
    RK_REQUIRE(has0, RK_EINVAL, "the diagonal offset (0,0,0) is required");
    RK_CUDA(cudaSetDevice(ctx->device));
    auto* op = new rk_op();
    try {
      op->ctx = ctx;
      op->g = *g;
      op->S = in7 ? 7 : (in19 ? 19 : 27);
      op->P = g->nx * g->ny;
      op->N = op->P * g->nz_local;
      op->wrapz = ((g->periodic_mask & 4) && ctx->nranks == 1) ? 1 : 0;
      // [S][N] bands + [N] inverse diagonal (band S, see compute_invdiag)
      cudaError_t e = cudaMalloc(&op->bands, sizeof(double) * (op->S + 1) * op->N);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(RK_ENOMEM, "cudaMalloc of the bands failed");
      }
      copy_bands(op, offsets, nbands, bands);
      const int bad = validate_bands(op);
      RK_REQUIRE(bad == 0, RK_EINVAL,
                 "bands violate truncation (S:39) or have a zero diagonal: " +
                     std::to_string(bad) + " bad coefficients");
      compute_invdiag(op);
      exchange_ghost_bands(op);
      op->user_offsets.assign(offsets, offsets + 3 * nbands);
      op->no_chain = std::getenv("RK_NO_CHAIN") != nullptr;
      op->force_chain = std::getenv("RK_FORCE_CHAIN") != nullptr;
    } catch (...) {
      cudaFree(op->bands);
      cudaFree(op->gbands);
      delete op;
      throw;
    }
    *out = op;
  });
}

rk_status rk_op_update_bands(rk_op* op, const double* bands) {
  return guarded([&] {
    RK_REQUIRE(op && bands, RK_EINVAL, "NULL argument");
    copy_bands(op, op->user_offsets.data(), (int)op->user_offsets.size() / 3, bands);
    const int bad = validate_bands(op);
    RK_REQUIRE(bad == 0, RK_EINVAL, "bands violate truncation (S:39) or have a zero diagonal");
    compute_invdiag(op);
    exchange_ghost_bands(op);
    ++op->epoch;
  });
}

void rk_op_destroy(rk_op* op) {
  if (!op) return;
  cudaSetDevice(op->ctx->device);
  cudaStreamSynchronize(op->ctx->stream);
  cudaFree(op->bands);
  cudaFree(op->gbands);
  cudaFree(op->rscratch_base);
  for (int i = 0; i < 2; ++i) cudaFree(op->scratch_base[i]);
  delete op;
}

static void op_scratch(rk_op* op) {
  for (int i = 0; i < 2; ++i)
    if (!op->scratch_base[i]) op->scratch[i] = alloc_padded(op, &op->scratch_base[i], nullptr);
}

rk_status rk_op_apply(rk_op* op, const double* x, double* y) {
  return guarded([&] {
    RK_REQUIRE(op && x && y, RK_EINVAL, "NULL argument");
    RK_CUDA(cudaSetDevice(op->ctx->device));
    op_scratch(op);
    RK_CUDA(cudaMemcpyAsync(op->scratch[0], x, sizeof(double) * op->N, cudaMemcpyDeviceToDevice,
                            op->ctx->stream));
    stencil(op, SM_SPMV, op->scratch[0], nullptr, y, nullptr, 0.0, nullptr);
    RK_CUDA(cudaStreamSynchronize(op->ctx->stream));
  });
}

rk_status rk_precond_apply(rk_op* op, const rk_precond* pc, const double* r, double* z) {
  return guarded([&] {
    RK_REQUIRE(op && pc && r && z, RK_EINVAL, "NULL argument");
    RK_CUDA(cudaSetDevice(op->ctx->device));
    if (pc->kind == 0) {
      RK_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * op->N, cudaMemcpyDeviceToDevice,
                              op->ctx->stream));
    } else if (pc->kind == 2) {
      RK_REQUIRE(pc->sweeps >= 1, RK_EINVAL, "bad preconditioner");
      check_ssor(op, *pc);
      op_scratch(op);
      ssor_apply(op, *pc, r, z, op->scratch[0], nullptr);
    } else {
      RK_REQUIRE(pc->kind == 1 && pc->sweeps >= 1, RK_EINVAL, "bad preconditioner");
      check_zblocks(op, *pc);
      op_scratch(op);
      double *za = op->scratch[0], *zb = op->scratch[1];
      stencil(op, SM_SCALE, nullptr, r, za, nullptr, pc->omega_local, nullptr);
      std::vector<int> k(pc->sweeps, CK_SWEEP);
      std::vector<double> w(pc->sweeps, pc->omega_local);
      std::vector<int> loc(pc->sweeps, 1);
      w.back() = pc->omega_global;
      loc.back() = 0;
      const int zbl = pc->zblocks > 1 ? (int)(op->g.nz_global / pc->zblocks) : 0;
      const double* rr = r;
      if (op->ctx->nranks > 1 && chain_max_stages(op) > 0) {
        // the fused chain reads the sweeps' right-hand side beyond the slab:
        // a padded copy whose ghost planes chain_run fills
        double* rp = op->rscratch_base ? op->rscratch_base + GHOST * op->P
                                       : alloc_padded(op, &op->rscratch_base, nullptr);
        RK_CUDA(cudaMemcpyAsync(rp, r, sizeof(double) * op->N, cudaMemcpyDeviceToDevice, op->ctx->stream));
        rr = rp;
      }
      chain_run(op, k, w, za, rr, nullptr, nullptr, z, za, zb, loc, zbl);
    }
    RK_CUDA(cudaStreamSynchronize(op->ctx->stream));
  });
}

rk_status rk_solver_create(rk_op* op, const rk_config* cfg, rk_solver** out) {
  return guarded([&] {
    RK_REQUIRE(op && cfg && out, RK_EINVAL, "NULL argument");
    RK_REQUIRE(cfg->m >= 1, RK_EINVAL, "m >= 1");
    RK_REQUIRE(cfg->k_max >= 0 && cfg->k_max + cfg->m + 1 <= MAXCOL, RK_EINVAL,
               "k_max + m + 1 must be <= 80");
    RK_REQUIRE(cfg->k_max <= 46, RK_EINVAL, "k_max <= 46");
    RK_REQUIRE(cfg->select_count >= 0 && cfg->select_count <= 2, RK_EINVAL, "select_count 0..2");
    RK_REQUIRE(cfg->k_keep >= 0 && cfg->k_keep <= cfg->k_max, RK_EINVAL, "0 <= k_keep <= k_max");
    RK_REQUIRE(cfg->ortho == 0 || cfg->ortho == 1, RK_EINVAL, "ortho: 0 (CGS2) or 1 (Gram-corrected CGS2)");
    RK_REQUIRE(cfg->trunc == 0 || cfg->trunc == 1, RK_EINVAL, "trunc: 0 (T1) or 1 (T2)");
    RK_REQUIRE(cfg->pc.kind == 0 || ((cfg->pc.kind == 1 || cfg->pc.kind == 2) && cfg->pc.sweeps >= 1),
               RK_EINVAL, "bad preconditioner");
    check_ssor(op, cfg->pc);
    if (cfg->pc.kind == 1) check_zblocks(op, cfg->pc);
    RK_REQUIRE(cfg->max_matvecs >= 1, RK_EINVAL, "max_matvecs >= 1");
    RK_CUDA(cudaSetDevice(op->ctx->device));
    auto* s = new rk_solver();
    try {
      s->op = op;
      s->ctx = op->ctx;
      s->cfg = *cfg;
      if (s->cfg.divergence_factor <= 0) s->cfg.divergence_factor = 1e4;
      s->method = cfg->method;
      s->N = op->N;
      const int nv = std::max(cfg->m + 1, 8);
      auto pad = [&]() {
        double* b;
        double* v = alloc_padded(op, &b, &s->nvec);
        s->bases.push_back(b);
        return v;
      };
      for (int i = 0; i < nv; ++i) s->V.push_back(pad());
      const int slots = cfg->k_max > 0 ? cfg->k_max + 2 : 0;
      for (int i = 0; i < slots; ++i) {
        s->Us.push_back(pad());
        s->Cs.push_back(pad());
      }
      s->x = pad();
      s->t = pad();
      s->za = pad();
      s->zb = pad();
      s->rt = pad();
      s->c_epoch = op->epoch;
      s->max_it = (int)std::min<int64_t>(cfg->max_matvecs / 2 + 4, 1 << 20);
      // scalar arena
      size_t o = 0;
      s->o_arn = o;
      o += rk_solver::STEP * (size_t)cfg->m;
      s->o_misc = o;
      o += rk_solver::MISC_XI + MAXCOL;
      s->o_coef = o;
      o += (size_t)MAXOUT * MAXCOL;
      s->o_gram = o;
      o += (size_t)MAXCOL * MAXCOL;
      s->o_T = o;
      o += (size_t)MAXCOL * MAXCOL;
      s->o_grow = o;                       // lagged Gram rows [R19]
      o += (size_t)MAXCOL * MAXCOL;
      o = (o + 7) & ~size_t(7);
      s->o_bi = o;
      o += 8 * (size_t)(s->max_it + 2);
      s->o_eta = o;
      o += 5 * (size_t)MAXCOL;   // eta(0..2) + C^T r~ + all-reduce staging (rBiCGStab)
      s->nsc = o;
      RK_CUDA(cudaMalloc(&s->dsc, o * sizeof(double)));
      RK_CUDA(cudaMemsetAsync(s->dsc, 0, o * sizeof(double), s->ctx->stream));
      RK_CUDA(cudaMallocHost(&s->hsc, o * sizeof(double)));
      for (auto& e : s->bev) RK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      if (const char* la = std::getenv("RK_BICG_LOOKAHEAD")) s->lookahead = std::atoi(la) != 0;
      if (const char* nf = std::getenv("RK_NFUSE")) s->nfuse = std::atoi(nf) != 0;
      std::memset(s->hsc, 0, o * sizeof(double));
      RK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    } catch (...) {
      for (auto b : s->bases) cudaFree(b);
      cudaFree(s->dsc);
      cudaFreeHost(s->hsc);
      for (auto e : s->bev)
        if (e) cudaEventDestroy(e);
      delete s;
      throw;
    }
    *out = s;
  });
}

void rk_solver_destroy(rk_solver* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  for (auto b : s->bases) cudaFree(b);
  cudaFree(s->bdev);
  s->free_pipeline();
  cudaFree(s->dsc);
  cudaFreeHost(s->hsc);
  for (auto e : s->bev)
    if (e) cudaEventDestroy(e);
  delete s;
}

rk_status rk_solver_set_method(rk_solver* s, rk_method m) {
  return guarded([&] {
    RK_REQUIRE(s, RK_EINVAL, "NULL solver");
    RK_REQUIRE(m >= RK_GMRES && m <= RK_RBICGSTAB, RK_EINVAL, "bad method");
    s->method = m;  // C validity is re-derived from the operator kind [D3]
  });
}

rk_status rk_recycle_set(rk_solver* s, int k, const double* U, const double* C, const double* R,
                         int64_t ld) {
  return guarded([&] {
    RK_REQUIRE(s, RK_EINVAL, "NULL solver");
    RK_REQUIRE(k >= 0 && k <= s->cfg.k_max, RK_EINVAL, "0 <= k <= k_max");
    RK_REQUIRE(k == 0 || (U && ld >= s->N), RK_EINVAL, "U NULL or ld < N");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    s->order.clear();
    for (int c = 0; c < k; ++c) {
      RK_CUDA(cudaMemcpyAsync(s->Us[c], U + (int64_t)c * ld, sizeof(double) * s->N,
                              cudaMemcpyDeviceToDevice, s->ctx->stream));
      if (C)
        RK_CUDA(cudaMemcpyAsync(s->Cs[c], C + (int64_t)c * ld, sizeof(double) * s->N,
                                cudaMemcpyDeviceToDevice, s->ctx->stream));
      s->order.push_back(c);
    }
    if (k > 0 && R) {  // absorb R: U <- U R^-1 [D14]
      std::vector<double> T((size_t)k * k, 0.0);
      for (int col = 0; col < k; ++col)
        for (int i = col; i >= 0; --i) {
          double v = (i == col) ? 1.0 : 0.0;
          for (int l = i + 1; l <= col; ++l) v -= R[i + l * k] * T[l + col * k];
          RK_REQUIRE(R[i + i * k] != 0.0, RK_EINVAL, "R singular");
          T[i + col * k] = v / R[i + i * k];
        }
      std::memcpy(s->hsc + s->o_T, T.data(), sizeof(double) * k * k);
      RK_CUDA(cudaMemcpyAsync(s->dsc + s->o_T, s->hsc + s->o_T, sizeof(double) * k * k,
                              cudaMemcpyHostToDevice, s->ctx->stream));
      std::vector<double*> Uw(s->Us.begin(), s->Us.begin() + k);
      rotate(s->ctx, Uw, s->dsc + s->o_T, s->N, -1, s->hsc + s->o_T);
    }
    s->c_valid = (C != nullptr) || k == 0;
    s->c_kind = s->kind_for(s->method);
    s->c_epoch = s->op->epoch;
    RK_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

rk_status rk_recycle_dim(rk_solver* s, int* k) {
  return guarded([&] {
    RK_REQUIRE(s && k, RK_EINVAL, "NULL argument");
    *k = (int)s->order.size();
  });
}

rk_status rk_recycle_export(rk_solver* s, double* U, double* C, double* R, int64_t ld) {
  return guarded([&] {
    RK_REQUIRE(s, RK_EINVAL, "NULL solver");
    const int k = (int)s->order.size();
    RK_REQUIRE(k == 0 || ld >= s->N, RK_EINVAL, "ld < N");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    for (int c = 0; c < k; ++c) {
      const int sl = s->order[c];
      if (U)
        RK_CUDA(cudaMemcpyAsync(U + (int64_t)c * ld, s->Us[sl], sizeof(double) * s->N,
                                cudaMemcpyDeviceToDevice, s->ctx->stream));
      if (C)
        RK_CUDA(cudaMemcpyAsync(C + (int64_t)c * ld, s->Cs[sl], sizeof(double) * s->N,
                                cudaMemcpyDeviceToDevice, s->ctx->stream));
    }
    if (R)
      for (int i = 0; i < k * k; ++i) R[i] = (i % (k + 1) == 0) ? 1.0 : 0.0;
    RK_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

rk_status rk_solve(rk_solver* s, const double* b, double* xu, double tol, rk_report* rep_out) {
  return guarded([&] {
    RK_REQUIRE(s && b && xu, RK_EINVAL, "NULL argument");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    const auto t0 = std::chrono::steady_clock::now();
    if (!(tol > 0)) tol = s->cfg.tol;
    rk_report rep;
    std::memset(&rep, 0, sizeof(rep));
    rep.final_true_res = std::numeric_limits<double>::quiet_NaN();
    rep.final_updated_res = std::numeric_limits<double>::quiet_NaN();
    s->history.clear();
    s->tr_cyc.clear();
    s->tr_bi.clear();
    RK_CUDA(cudaMemcpyAsync(s->x, xu, sizeof(double) * s->N, cudaMemcpyDeviceToDevice,
                            s->ctx->stream));
    if (s->method == RK_RGCROT || s->method == RK_GMRES) s->solve_rgcrot(b, tol, rep);
    else s->solve_rbicgstab(b, tol, rep);
    RK_CUDA(cudaMemcpyAsync(xu, s->x, sizeof(double) * s->N, cudaMemcpyDeviceToDevice,
                            s->ctx->stream));
    RK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    rep.k_after = (int)s->order.size();
    rep.history_len = (int64_t)s->history.size();
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s->last = rep;
    if (rep_out) *rep_out = rep;
  });
}

rk_status rk_solve_host_ex(rk_solver* s, const double* bh, const double* x0h, double* xh, double tol,
                           rk_report* rep) {
  return guarded([&] {
    RK_REQUIRE(s && bh && xh, RK_EINVAL, "NULL argument");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    if (!s->bdev) RK_CUDA(cudaMalloc(&s->bdev, sizeof(double) * s->N));
    const auto t0 = std::chrono::steady_clock::now();
    RK_CUDA(cudaMemcpyAsync(s->bdev, bh, sizeof(double) * s->N, cudaMemcpyHostToDevice,
                            s->ctx->stream));
    if (x0h)
      RK_CUDA(cudaMemcpyAsync(s->x, x0h, sizeof(double) * s->N, cudaMemcpyHostToDevice,
                              s->ctx->stream));
    else
      RK_CUDA(cudaMemsetAsync(s->x, 0, sizeof(double) * s->N, s->ctx->stream));
    if (!(tol > 0)) tol = s->cfg.tol;
    rk_report r;
    std::memset(&r, 0, sizeof(r));
    s->history.clear();
    s->tr_cyc.clear();
    s->tr_bi.clear();
    if (s->method == RK_RGCROT || s->method == RK_GMRES) s->solve_rgcrot(s->bdev, tol, r);
    else s->solve_rbicgstab(s->bdev, tol, r);
    RK_CUDA(cudaMemcpyAsync(xh, s->x, sizeof(double) * s->N, cudaMemcpyDeviceToHost,
                            s->ctx->stream));
    RK_CUDA(cudaStreamSynchronize(s->ctx->stream));
    r.k_after = (int)s->order.size();
    r.history_len = (int64_t)s->history.size();
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s->last = r;
    if (rep) *rep = r;
  });
}

rk_status rk_solve_host(rk_solver* s, const double* bh, double* xh, double tol, rk_report* rep) {
  return rk_solve_host_ex(s, bh, xh, xh, tol, rep);
}

rk_status rk_stage_rhs(rk_solver* s, int slot, const double* bh) {
  return guarded([&] {
    RK_REQUIRE(s && bh, RK_EINVAL, "NULL argument");
    RK_REQUIRE(slot == 0 || slot == 1, RK_EINVAL, "slot must be 0 or 1");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    s->ensure_pipeline();
    RK_CUDA(cudaMemcpyAsync(s->bstage[slot], bh, sizeof(double) * s->N, cudaMemcpyHostToDevice,
                            s->cstream));
    RK_CUDA(cudaEventRecord(s->staged_ev[slot], s->cstream));
    s->staged_ok[slot] = true;
  });
}

rk_status rk_solve_staged(rk_solver* s, int slot, double* xh, double tol, rk_report* rep) {
  return guarded([&] {
    RK_REQUIRE(s && xh, RK_EINVAL, "NULL argument");
    RK_REQUIRE(slot == 0 || slot == 1, RK_EINVAL, "slot must be 0 or 1");
    RK_REQUIRE(s->cstream && s->staged_ok[slot], RK_EINVAL, "slot was never staged");
    RK_CUDA(cudaSetDevice(s->ctx->device));
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t ls = s->ctx->stream;
    RK_CUDA(cudaStreamWaitEvent(ls, s->staged_ev[slot], 0));   // b has landed
    RK_CUDA(cudaMemsetAsync(s->x, 0, sizeof(double) * s->N, ls));   // x_hat = 0
    if (!(tol > 0)) tol = s->cfg.tol;
    rk_report r;
    std::memset(&r, 0, sizeof(r));
    s->history.clear();
    s->tr_cyc.clear();
    s->tr_bi.clear();
    if (s->method == RK_RGCROT || s->method == RK_GMRES) s->solve_rgcrot(s->bstage[slot], tol, r);
    else s->solve_rbicgstab(s->bstage[slot], tol, r);
    // snapshot x (after the previous download finished with the snapshot
    // buffer) and download it on the copy stream; the next solve overlaps it
    if (s->xcopy_pending) RK_CUDA(cudaStreamWaitEvent(ls, s->xcopied, 0));
    RK_CUDA(cudaMemcpyAsync(s->xstage, s->x, sizeof(double) * s->N, cudaMemcpyDeviceToDevice, ls));
    RK_CUDA(cudaEventRecord(s->xready, ls));
    RK_CUDA(cudaStreamWaitEvent(s->cstream, s->xready, 0));
    RK_CUDA(cudaMemcpyAsync(xh, s->xstage, sizeof(double) * s->N, cudaMemcpyDeviceToHost,
                            s->cstream));
    RK_CUDA(cudaEventRecord(s->xcopied, s->cstream));
    s->xcopy_pending = true;
    r.k_after = (int)s->order.size();
    r.history_len = (int64_t)s->history.size();
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s->last = r;
    if (rep) *rep = r;
  });
}

rk_status rk_host_sync(rk_solver* s) {
  return guarded([&] {
    RK_REQUIRE(s, RK_EINVAL, "NULL argument");
    if (!s->cstream) return;
    RK_CUDA(cudaSetDevice(s->ctx->device));
    if (s->xcopy_pending) RK_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->xcopied, 0));
    RK_CUDA(cudaStreamSynchronize(s->cstream));
    s->xcopy_pending = false;
  });
}

rk_status rk_history(rk_solver* s, double* out, int64_t cap, int64_t* len) {
  return guarded([&] {
    RK_REQUIRE(s && len, RK_EINVAL, "NULL argument");
    *len = (int64_t)s->history.size();
    if (out)
      for (int64_t i = 0; i < std::min<int64_t>(cap, *len); ++i)
        for (int q = 0; q < 3; ++q) out[3 * i + q] = s->history[i][q];
  });
}

rk_status rk_trace(rk_solver* s, int what, double* out, int64_t cap, int64_t* len) {
  return guarded([&] {
    RK_REQUIRE(s && len, RK_EINVAL, "NULL argument");
    RK_REQUIRE(what == 0 || what == 1, RK_EINVAL, "what: 0 (rGCROT cycles) or 1 (rBiCGStab iterations)");
    const std::vector<double>& v = what == 0 ? s->tr_cyc : s->tr_bi;
    *len = (int64_t)v.size();
    if (out) std::memcpy(out, v.data(), sizeof(double) * (size_t)std::min<int64_t>(cap, *len));
  });
}

rk_status rk_solver_workspace(rk_solver* s, int64_t* nvec) {
  return guarded([&] {
    RK_REQUIRE(s && nvec, RK_EINVAL, "NULL argument");
    *nvec = s->nvec;
  });
}

rk_status rk_launch_count(rk_ctx* ctx, int64_t* count) {
  return guarded([&] {
    RK_REQUIRE(ctx && count, RK_EINVAL, "NULL argument");
    *count = ctx->launches;
  });
}

rk_status rk_comm_count(rk_ctx* ctx, int64_t* allreduces, int64_t* halos) {
  return guarded([&] {
    RK_REQUIRE(ctx, RK_EINVAL, "NULL ctx");
    if (allreduces) *allreduces = ctx->n_allreduce;
    if (halos) *halos = ctx->n_halo;
  });
}

rk_status rk_profile_enable(rk_ctx* ctx, int on, const char* filter) {
  return guarded([&] {
    RK_REQUIRE(ctx, RK_EINVAL, "NULL ctx");
    ctx->prof_on = on != 0;
    ctx->prof_filter = filter ? filter : "";
  });
}

rk_status rk_profile_every(rk_ctx* ctx, int every) {
  return guarded([&] {
    RK_REQUIRE(ctx && every >= 1, RK_EINVAL, "every >= 1");
    ctx->prof_every = every;
    ctx->prof_seen = 0;
  });
}

rk_status rk_profile_read(rk_ctx* ctx, int cap, char* names, int64_t* launches, double* ms,
                          double* bytes, int* n) {
  return guarded([&] {
    RK_REQUIRE(ctx && n, RK_EINVAL, "NULL argument");
    RK_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& p : ctx->pending) {
      float t = 0.f;
      RK_CUDA(cudaEventElapsedTime(&t, p.a, p.b));
      auto& a = ctx->agg[p.cls];
      a.launches += 1;
      a.ms += t;
      a.bytes += p.bytes;
      ctx->pool.push_back(p.a);
      ctx->pool.push_back(p.b);
    }
    ctx->pending.clear();
    int i = 0;
    for (auto& kv : ctx->agg) {
      if (i < cap) {
        if (names) {
          std::strncpy(names + 32 * i, kv.first.c_str(), 31);
          names[32 * i + 31] = 0;
        }
        if (launches) launches[i] = kv.second.launches;
        if (ms) ms[i] = kv.second.ms;
        if (bytes) bytes[i] = kv.second.bytes;
      }
      ++i;
    }
    *n = i;
    if (cap < 0) ctx->agg.clear();  // cap < 0: reset
  });
}

}  // extern "C"

// ------------------------------------------------------- per-kernel entry points
// (include/rk.h "Per-kernel entry points"): one kernel family each, through
// the solvers' own host launch functions, on one rank, synchronised.
namespace {
static_assert(sizeof(rk_bicg_iter) == sizeof(rk::BiIter) &&
                  offsetof(rk_bicg_iter, stop) == offsetof(rk::BiIter, stop) &&
                  offsetof(rk_bicg_iter, ts) == offsetof(rk::BiIter, ts),
              "rk_bicg_iter must mirror rk::BiIter");

void kernel_entry(rk_ctx* ctx) {
  RK_REQUIRE(ctx, RK_EINVAL, "NULL ctx");
  RK_REQUIRE(ctx->nranks == 1, RK_EUNSUPPORTED, "per-kernel entry points need a one-rank context");
  RK_CUDA(cudaSetDevice(ctx->device));
  ctx->gate = nullptr;
}

std::vector<const double*> col_list(int ncol, const double* const* Q, int maxcol) {
  RK_REQUIRE(Q && ncol >= 1 && ncol <= maxcol, RK_EINVAL, "need 1 <= ncol <= " + std::to_string(maxcol));
  std::vector<const double*> v(Q, Q + ncol);
  for (auto p : v) RK_REQUIRE(p, RK_EINVAL, "NULL column pointer");
  return v;
}

void kernel_done(rk_ctx* ctx) { RK_CUDA(cudaStreamSynchronize(ctx->stream)); }
}  // namespace

extern "C" {

rk_status rk_block_dot(rk_ctx* ctx, int ncol, const double* const* Q, const double* w,
                       const double* v, int64_t n, double* out_w, double* out_v) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cols = col_list(ncol, Q, MAXCOL);
    RK_REQUIRE(w && out_w && n >= 1 && (!v || out_v), RK_EINVAL, "NULL argument or n < 1");
    if (v) bdot2(ctx, cols, w, v, n, out_w, out_v);
    else bdot(ctx, cols, w, n, out_w);
    kernel_done(ctx);
  });
}

rk_status rk_block_update(rk_ctx* ctx, int ncol, const double* const* Q, const double* g,
                          double* w, int64_t n, int ndots, const double* const* dots,
                          double* red) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cols = col_list(ncol, Q, MAXCOL);
    RK_REQUIRE(g && w && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    RK_REQUIRE(ndots >= 0 && ndots <= 3 && (ndots == 0 || (dots && red)), RK_EINVAL,
               "0 <= ndots <= 3, dots and red given when ndots > 0");
    std::vector<const double*> d(dots, dots + ndots);
    bupd(ctx, cols, g, 1.0, w, n, d, ndots ? red : nullptr);
    kernel_done(ctx);
  });
}

rk_status rk_block_project(rk_ctx* ctx, int ncol, const double* const* Q, double* w, int64_t n,
                           double* eta, double* nrm2) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cols = col_list(ncol, Q, 40);
    RK_REQUIRE(w && eta && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    if (nrm2) bproject(ctx, cols, w, n, eta, {nullptr}, nrm2);
    else bproject(ctx, cols, w, n, eta, {}, nullptr);
    kernel_done(ctx);
  });
}

rk_status rk_gram_update(rk_ctx* ctx, int ncol, int k, const double* const* Q, const double* g,
                         const double* grow, double* h_out, double* w, int64_t n, double* nrm2) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cols = col_list(ncol, Q, MAXCOL);
    RK_REQUIRE(k >= 0 && k <= ncol, RK_EINVAL, "need 0 <= k <= ncol");
    RK_REQUIRE(g && grow && h_out && w && nrm2 && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    bupd_gram(ctx, cols, k, g, grow, h_out, w, n, nrm2);
    kernel_done(ctx);
  });
}

rk_status rk_project_update(rk_ctx* ctx, int k, const double* const* C, const double* const* U,
                            const double* xi, double* r, double* x, int64_t n, double* nrm2) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cc = col_list(k, C, 48);
    std::vector<const double*> uu;
    if (x) {
      RK_REQUIRE(U, RK_EINVAL, "U needed with x");
      uu = col_list(k, U, 48);
    }
    RK_REQUIRE(xi && r && nrm2 && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    proj(ctx, cc, uu, xi, r, x, n, nrm2);
    kernel_done(ctx);
  });
}

rk_status rk_normalize(rk_ctx* ctx, double* w, int64_t n, const double* nrm2, const double* nin2,
                       double* flag) {
  return guarded([&] {
    kernel_entry(ctx);
    RK_REQUIRE(w && nrm2 && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    normalize(ctx, w, n, nrm2, nin2, flag);
    kernel_done(ctx);
  });
}

rk_status rk_lincomb(rk_ctx* ctx, int ncol, const double* const* Q, const double* coef, int nout,
                     double* const* out, const double* scale, const int* acc, int64_t n) {
  return guarded([&] {
    kernel_entry(ctx);
    auto cols = col_list(ncol, Q, MAXCOL);
    RK_REQUIRE(coef && out && scale && acc && n >= 1, RK_EINVAL, "NULL argument or n < 1");
    RK_REQUIRE(nout >= 1 && nout <= MAXOUT, RK_EINVAL, "need 1 <= nout <= 5");
    LcOut lo;
    memset(&lo, 0, sizeof(lo));
    for (int o = 0; o < nout; ++o) {
      RK_REQUIRE(out[o], RK_EINVAL, "NULL output pointer");
      lo.out[o] = out[o];
      lo.scale[o] = scale[o];
      lo.acc[o] = acc[o] != 0;
    }
    lincomb(ctx, cols, coef, nout, lo, n);
    kernel_done(ctx);
  });
}

rk_status rk_rotate(rk_ctx* ctx, int k, double* const* Q, const double* T, int kout, int64_t n) {
  return guarded([&] {
    kernel_entry(ctx);
    RK_REQUIRE(Q && T && n >= 1 && k >= 1 && k <= MAXCOL, RK_EINVAL, "NULL argument, n < 1 or bad k");
    std::vector<double*> cols(Q, Q + k);
    for (auto p : cols) RK_REQUIRE(p, RK_EINVAL, "NULL column pointer");
    std::vector<double> Th((size_t)k * k);
    RK_CUDA(cudaMemcpyAsync(Th.data(), T, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
    RK_CUDA(cudaStreamSynchronize(ctx->stream));   // T may come from work queued on the context stream
    rotate(ctx, cols, T, n, kout, Th.data());
    kernel_done(ctx);
  });
}

rk_status rk_bicg_p(rk_op* op, int first, const double* r, double* p, const double* v, double* z,
                    double omega_l, int jacobi, rk_bicg_iter* cur, const rk_bicg_iter* prev,
                    double thr_conv, double thr_div) {
  return guarded([&] {
    RK_REQUIRE(op, RK_EINVAL, "NULL op");
    kernel_entry(op->ctx);
    RK_REQUIRE(r && p && z && cur && (first || (v && prev)), RK_EINVAL, "NULL argument");
    bicg_p(op, r, p, v, z, omega_l, jacobi != 0, reinterpret_cast<BiIter*>(cur),
           reinterpret_cast<const BiIter*>(prev), first ? 1 : 0, thr_conv, thr_div);
    kernel_done(op->ctx);
  });
}

rk_status rk_bicg_s(rk_op* op, const double* r, const double* v, double* s, double* z,
                    double omega_l, int jacobi, rk_bicg_iter* cur) {
  return guarded([&] {
    RK_REQUIRE(op, RK_EINVAL, "NULL op");
    kernel_entry(op->ctx);
    RK_REQUIRE(r && v && s && z && cur, RK_EINVAL, "NULL argument");
    bicg_s(op, r, v, s, z, omega_l, jacobi != 0, reinterpret_cast<BiIter*>(cur));
    kernel_done(op->ctx);
  });
}

rk_status rk_bicg_project_s(rk_op* op, int k, const double* const* C, double* v, const double* rt,
                            const double* ctr, double* eta, const double* r, double* s, double* z,
                            double omega_l, int jacobi, rk_bicg_iter* cur) {
  return guarded([&] {
    RK_REQUIRE(op, RK_EINVAL, "NULL op");
    kernel_entry(op->ctx);
    auto cols = col_list(k, C, 39);
    RK_REQUIRE(v && rt && ctr && eta && r && s && z && cur, RK_EINVAL, "NULL argument");
    const bool ok = bicg_proj_s(op, cols, v, rt, ctr, eta, r, s, z, omega_l, jacobi != 0,
                                reinterpret_cast<BiIter*>(cur), nullptr);
    RK_REQUIRE(ok, RK_EUNSUPPORTED,
               "fused projection needs even n, 16-byte aligned pointers and deferred coefficients");
    kernel_done(op->ctx);
  });
}

rk_status rk_bicg_xr(rk_op* op, double* x, double* r, const double* s, const double* t,
                     const double* p_hat, const double* s_hat, const double* rt,
                     rk_bicg_iter* cur, rk_bicg_iter* next, double* xi, const double* eta1,
                     const double* eta2, int k) {
  return guarded([&] {
    RK_REQUIRE(op, RK_EINVAL, "NULL op");
    kernel_entry(op->ctx);
    RK_REQUIRE(x && r && s && t && p_hat && s_hat && rt && cur && next, RK_EINVAL, "NULL argument");
    RK_REQUIRE(k >= 0 && (k == 0 || (xi && eta1 && eta2)), RK_EINVAL, "xi, eta1, eta2 needed for k > 0");
    bicg_xr(op->ctx, x, r, s, t, p_hat, s_hat, rt, op->N, reinterpret_cast<BiIter*>(cur),
            reinterpret_cast<BiIter*>(next), xi, eta1, eta2, k);
    kernel_done(op->ctx);
  });
}

}  // extern "C"
