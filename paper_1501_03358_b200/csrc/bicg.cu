// sm_100a rBiCGStab kernels of librk (K6): fused vector updates with the
// first Jacobi sweep and the iteration reductions (PAPER Alg. 4).
#include "kcommon.cuh"

namespace rk {

// ------------------------------------------------------------ K6 rBiCGStab
// Alg. 4 line 6 fused with the first Jacobi sweep of p_hat = M^-1 p:
// p = r (i = 0) or p = r + beta (p - omega v), beta = (rho_i/rho_{i-1})(alpha/omega);
// z = w_l p / D (D == nullptr: no preconditioner, z = p).
template <int VEC>
__global__ void __launch_bounds__(256) bicg_p_kernel(const double* __restrict__ r, double* __restrict__ p,
                                                     const double* __restrict__ v, const double* __restrict__ D,
                                                     double* __restrict__ z, double wl, int64_t N,
                                                     BiIter* cur, const BiIter* prev, int first,
                                                     double thr_conv, double thr_div) {
  RK_PDL_ENTRY();
  // the first element's operands do not depend on the scalars below: their
  // loads are issued before the scalar round trip
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Vec<VEC> r0v{}, p0v{}, v0v{}, d0v{};
  if (e0 < NE) {
    r0v = ldv_ro<VEC>(r + e0 * VEC);
    if (!first) {
      p0v = ldv<VEC>(p + e0 * VEC);
      v0v = ldv_ro<VEC>(v + e0 * VEC);
    }
    if (D) d0v = ldv_stream<VEC>(D + e0 * VEC);
  }
  // lookahead gate: every CTA takes the same decision from the records
  // written by the previous iteration (flag, sigma) and its bicg_xr (rho, rr)
  bool stop = false;
  if (!first) {
    const double rn2 = sqrt(cur->rr);
    stop = prev->flag != 0.0 || prev->sigma == 0.0 || !(rn2 > thr_conv) || cur->rho == 0.0 ||
           !(rn2 <= thr_div);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cur->stop = stop ? 1.0 : 0.0;
  if (stop) return;
  double beta = 0.0, omega = 0.0;
  if (!first) {
    const double alpha = prev->rho / prev->sigma;
    omega = prev->ts / prev->tt;
    beta = (cur->rho / prev->rho) * (alpha / omega);
  }
  auto body = [&](int64_t n, const Vec<VEC>& rn, const Vec<VEC>& po, const Vec<VEC>& vn,
                  const Vec<VEC>& dn) {
    Vec<VEC> pn;
    if (first) {
      pn = rn;
    } else {
#pragma unroll
      for (int t = 0; t < VEC; ++t) pn.v[t] = rn.v[t] + beta * (po.v[t] - omega * vn.v[t]);
    }
    stv<VEC>(p + n, pn);
    Vec<VEC> zn = pn;
    if (D) {
#pragma unroll
      for (int t = 0; t < VEC; ++t) zn.v[t] = (wl * pn.v[t]) * dn.v[t];
    }
    stv<VEC>(z + n, zn);
  };
  if (e0 < NE) body(e0 * VEC, r0v, p0v, v0v, d0v);
  for (int64_t e = e0 + stride; e < NE; e += stride) {
    const int64_t n = e * VEC;
    const Vec<VEC> rn = ldv_ro<VEC>(r + n);
    Vec<VEC> po{}, vn{}, dn{};
    if (!first) {
      po = ldv<VEC>(p + n);
      vn = ldv_ro<VEC>(v + n);
    }
    if (D) dn = ldv_stream<VEC>(D + n);
    body(n, rn, po, vn, dn);
  }
}

// Alg. 4 line 8 fused with the first sweep of s_hat = M^-1 s:
// alpha = rho/sigma; s = r - alpha v; z = w_l s / D; red ||s||^2.
template <int VEC>
__global__ void __launch_bounds__(256) bicg_s_kernel(const double* __restrict__ r, const double* __restrict__ v,
                                                     double* __restrict__ s, const double* __restrict__ D,
                                                     double* __restrict__ z, double wl, int64_t N,
                                                     const BiIter* cur, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  const double alpha = cur->rho / cur->sigma;
  double acc[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t n = e * VEC;
    const Vec<VEC> rn = ldv_ro<VEC>(r + n);
    const Vec<VEC> vn = ldv_ro<VEC>(v + n);
    Vec<VEC> sn, zn;
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      sn.v[t] = rn.v[t] - alpha * vn.v[t];
      acc[0] = fma(sn.v[t], sn.v[t], acc[0]);
    }
    stv<VEC>(s + n, sn);
    zn = sn;
    if (D) {
      const Vec<VEC> dn = ldv_stream<VEC>(D + n);
#pragma unroll
      for (int t = 0; t < VEC; ++t) zn.v[t] = (wl * sn.v[t]) * dn.v[t];
    }
    stv<VEC>(z + n, zn);
  }
  block_reduce_store<1>(acc, 1, ra);
}

// Alg. 4 lines 13-15 (+10-10a exact exit), with the breakdown guards of
// reading D17 evaluated on the device so a breakdown never touches x:
// x += alpha p_hat + omega s_hat ; r = s - omega t ; xi += alpha eta1 + omega eta2 ;
// red (r~^T r, ||r||^2) -> next->rho, next->rr.
template <int VEC>
__global__ void __launch_bounds__(256) bicg_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                      const double* __restrict__ s, const double* __restrict__ t,
                                                      const double* __restrict__ ph, const double* __restrict__ sh,
                                                      const double* __restrict__ rt, int64_t N, BiIter* cur,
                                                      double* xi, const double* eta1, const double* eta2,
                                                      int k, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  const double alpha = cur->rho / cur->sigma;
  const double omega = cur->ts / cur->tt;
  int mode;  // 0 full update, 1 exact exit, 2 breakdown (no update)
  if (cur->sigma == 0.0) mode = 2;
  else if (cur->ss == 0.0) mode = 1;
  else if (cur->tt == 0.0 || omega == 0.0) mode = 2;
  else mode = 0;
  double acc[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t n = e * VEC;
    Vec<VEC> rn;
    if (mode == 0) {
      Vec<VEC> xn = ldv<VEC>(x + n);
      const Vec<VEC> pn = ldv_ro<VEC>(ph + n), sn = ldv_ro<VEC>(sh + n);
      const Vec<VEC> s0 = ldv_ro<VEC>(s + n), t0 = ldv_ro<VEC>(t + n);
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        xn.v[q] = xn.v[q] + alpha * pn.v[q] + omega * sn.v[q];
        rn.v[q] = s0.v[q] - omega * t0.v[q];
      }
      stv<VEC>(x + n, xn);
      stv<VEC>(r + n, rn);
    } else if (mode == 1) {
      Vec<VEC> xn = ldv<VEC>(x + n);
      const Vec<VEC> pn = ldv_ro<VEC>(ph + n);
#pragma unroll
      for (int q = 0; q < VEC; ++q) xn.v[q] = xn.v[q] + alpha * pn.v[q];
      stv<VEC>(x + n, xn);
      rn = ldv_ro<VEC>(s + n);
      stv<VEC>(r + n, rn);
    } else {
      rn = ldv<VEC>(r + n);
    }
    const Vec<VEC> rtn = ldv_ro<VEC>(rt + n);
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[0] = fma(rtn.v[q], rn.v[q], acc[0]);
      acc[1] = fma(rn.v[q], rn.v[q], acc[1]);
    }
  }
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      if (mode == 0) xi[c] = xi[c] + alpha * eta1[c] + omega * eta2[c];
      else if (mode == 1) xi[c] = xi[c] + alpha * eta1[c];
    }
    if (threadIdx.x == 0) cur->flag = (double)mode;
  }
  block_reduce_store<2>(acc, 2, ra);
}

// Alg. 4 line 1c bookkeeping: xi = -eta0 ; rho_0 = ||r_0||^2 (r~ = r_0).
__global__ void bicg_setup_kernel(double* xi, const double* eta0, int k, BiIter* it0) {
  RK_PDL_ENTRY();
  for (int c = threadIdx.x; c < k; c += blockDim.x) xi[c] = -eta0[c];
  if (threadIdx.x == 0) it0->rr = it0->rho;
}


// =================================================================== host
void bicg_p(rk_op* op, const double* r, double* p, const double* v, double* z, double wl,
            bool jacobi, BiIter* cur, const BiIter* prev, int first, double thr_conv, double thr_div) {
  rk_ctx* ctx = op->ctx;
  const double* D = jacobi ? op->invd() : nullptr;   // 1 / D
  const int vec = pick_vec(op->N, {r, p, v, z, D});
  Launch L(ctx, "bicg_p", 8.0 * op->N * ((first ? 3 : 5) + (jacobi ? 1 : 0)));
  if (vec == 2)
    launch_k(ctx, bicg_p_kernel<2>, op->N / 2, dim3(256), r, p, v, D, z, wl, op->N, cur, prev, first,
             thr_conv, thr_div);
  else
    launch_k(ctx, bicg_p_kernel<1>, op->N, dim3(256), r, p, v, D, z, wl, op->N, cur, prev, first,
             thr_conv, thr_div);
  L.done();
}

void bicg_s(rk_op* op, const double* r, const double* v, double* s, double* z, double wl,
            bool jacobi, BiIter* cur) {
  rk_ctx* ctx = op->ctx;
  const double* D = jacobi ? op->invd() : nullptr;   // 1 / D
  RedArgs ra = red_args(ctx, &cur->ss);
  const int vec = pick_vec(op->N, {r, v, s, z, D});
  Launch L(ctx, "bicg_s", 8.0 * op->N * (jacobi ? 5 : 4));
  if (vec == 2)
    launch_k(ctx, bicg_s_kernel<2>, op->N / 2, dim3(256), r, v, s, D, z, wl, op->N,
             (const BiIter*)cur, ra);
  else
    launch_k(ctx, bicg_s_kernel<1>, op->N, dim3(256), r, v, s, D, z, wl, op->N,
             (const BiIter*)cur, ra);
  L.done();
  allreduce(ctx, &cur->ss, 1);
}

void bicg_xr(rk_ctx* ctx, double* x, double* r, const double* s, const double* t, const double* ph,
             const double* sh, const double* rt, int64_t N, BiIter* cur, BiIter* next, double* xi,
             const double* eta1, const double* eta2, int k) {
  RedArgs ra = red_args(ctx, &next->rho);
  const int vec = pick_vec(N, {x, r, s, t, ph, sh, rt});
  Launch L(ctx, "bicg_xr", 8.0 * N * 8);
  if (vec == 2)
    launch_k(ctx, bicg_xr_kernel<2>, N / 2, dim3(256), x, r, s, t, ph, sh, rt, N, cur, xi, eta1,
             eta2, k, ra);
  else
    launch_k(ctx, bicg_xr_kernel<1>, N, dim3(256), x, r, s, t, ph, sh, rt, N, cur, xi, eta1,
             eta2, k, ra);
  L.done();
  allreduce(ctx, &next->rho, 2);
}

void bicg_setup(rk_ctx* ctx, double* xi, const double* eta0, int k, BiIter* it0) {
  Launch L(ctx, "bicg_setup", 0);
  launch_pdl(ctx, bicg_setup_kernel, dim3(1), dim3(128), 0, xi, eta0, k, it0);
  L.done();
}

}  // namespace rk
