// sm_100a kernels of librk: the per-iteration hot path of rGCROT / rBiCGStab
// (SURVEY.md §2.4 K1-K8).  Every kernel here is HBM-bound fp64 work on the
// CUDA cores (0.1-0.3 flop/B, SURVEY §8(a) "Tensor cores"):
//  * coalesced x-fastest rows, two consecutive cells per thread with 16-byte
//    loads wherever the data allows (VEC = 2);
//  * streaming (ld.global.nc.L1::no_allocate) loads for data read once per
//    launch (bands, basis columns);
//  * grids sized from each instantiation's occupancy: SMs x resident CTAs,
//    grid-stride loops;
//  * deterministic two-stage reductions (per-CTA partials + fixed-order
//    finalisation by the last CTA; no floating-point atomics).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <initializer_list>

#include "rk_internal.h"

namespace rk {

// ------------------------------------------------------------------ helpers
template <int VEC>
struct Vec {
  double v[VEC];
};

template <int VEC>
__device__ __forceinline__ Vec<VEC> ldv_stream(const double* p) {
  Vec<VEC> r;
  if constexpr (VEC == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r.v[0]) : "l"(p));
  }
  return r;
}

// read-only (non-coherent) path: data not written by the same launch
template <int VEC>
__device__ __forceinline__ Vec<VEC> ldv_ro(const double* p) {
  Vec<VEC> r;
  if constexpr (VEC == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    r.v[0] = t.x;
    r.v[1] = t.y;
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ Vec<VEC> ldv(const double* p) {
  Vec<VEC> r;
  if constexpr (VEC == 2) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    r.v[0] = t.x;
    r.v[1] = t.y;
  } else {
    r.v[0] = *p;
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ void stv(double* p, const Vec<VEC>& a) {
  if constexpr (VEC == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(a.v[0], a.v[1]);
  } else {
    *p = a.v[0];
  }
}

// Canonical stencil layouts.  Band 0 is the diagonal.
//  7: 0, -x, +x, -y, +y, -z, +z
// 19: 7-point + xy edges (-1,-1)(1,-1)(-1,1)(1,1), yz edges (y,z) = (-1,-1)(1,-1)(-1,1)(1,1),
//     xz edges (x,z) = (-1,-1)(1,-1)(-1,1)(1,1)
// 27: centre, then the other 26 offsets in lexicographic (dz, dy, dx) order.
template <int ST>
__host__ __device__ constexpr void offs(int d, int& dx, int& dy, int& dz) {
  if (ST == 27) {
    const int e = d == 0 ? 13 : (d <= 13 ? d - 1 : d);
    dx = e % 3 - 1;
    dy = (e / 3) % 3 - 1;
    dz = e / 9 - 1;
    return;
  }
  constexpr int DX[19] = {0, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1};
  constexpr int DY[19] = {0, 0, 0, -1, 1, 0, 0, -1, -1, 1, 1, -1, 1, -1, 1, 0, 0, 0, 0};
  constexpr int DZ[19] = {0, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, -1, 1, 1, -1, -1, 1, 1};
  dx = DX[d];
  dy = DY[d];
  dz = DZ[d];
}

template <int ST>
__host__ __device__ constexpr bool uses(int dx, int dy, int dz) {
  for (int d = 0; d < ST; ++d) {
    int a = 0, b = 0, c = 0;
    offs<ST>(d, a, b, c);
    if (a == dx && b == dy && c == dz) return true;
  }
  return false;
}

// Block reduction of NV per-thread values -> per-CTA partials -> the last CTA
// to finish sums the partials of every value in a fixed order (deterministic).
template <int NV>
__device__ __forceinline__ void block_reduce_store(const double (&v)[NV], int nv,
                                                   const RedArgs& ra) {
  __shared__ double sm[NV][33];
  __shared__ bool last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nthreads = blockDim.x * blockDim.y;
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q < nv) {
      double s = v[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) sm[q][warp] = s;
    }
  }
  __syncthreads();
  const int G = gridDim.x;
  for (int q = warp; q < nv; q += nwarps) {
    double s = lane < nwarps ? sm[q][lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) ra.partials[(int64_t)q * G + blockIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(ra.counter, 1u) == (unsigned)(G - 1));
  __syncthreads();
  if (last) {
    __threadfence();
    for (int q = warp; q < nv; q += nwarps) {
      double s = 0.0;
      for (int c = lane; c < G; c += 32) s += __ldcg(ra.partials + (int64_t)q * G + c);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) ra.out[q] = s;
    }
    if (tid == 0) atomicExch(ra.counter, 0u);
  }
}

// -------------------------------------------------------------- K1 / K2
// Each thread owns VEC consecutive cells of an x-row (VEC = 2: 16-byte band
// and centre loads, the x-1 / x+VEC neighbours as scalars); rows (j, k) are
// grid-strided over the CTAs.  Out-of-grid neighbours on non-periodic x/y
// are clamped onto a valid cell (their coefficient is 0 by the truncation
// invariant); z neighbours read the ghost planes (zero, or halo data from the
// neighbouring rank), or wrap for a single-rank periodic z.
template <int ST, int MODE, int VEC>
__global__ void __launch_bounds__(256) stencil_kernel(StencilParams sp) {
  constexpr bool RED = (MODE == SM_SWEEP_NORM || MODE == SM_RESID || MODE == SM_RESID_SWEEP1);
  const int BX = blockDim.x, BY = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  double red[1] = {0.0};
  const int64_t R = (int64_t)sp.ny * sp.nzl;
  const int nxv = sp.nx / VEC;
  for (int64_t row = (int64_t)blockIdx.x * BY + ty; row < R; row += (int64_t)gridDim.x * BY) {
    const int k = (int)(row / sp.ny);
    const int j = (int)(row - (int64_t)k * sp.ny);
    const int64_t base = (int64_t)k * sp.P + (int64_t)j * sp.nx;
    if constexpr (MODE == SM_SCALE) {
      for (int iv = tx; iv < nxv; iv += BX) {
        const int64_t n = base + (int64_t)iv * VEC;
        const Vec<VEC> D = ldv_stream<VEC>(sp.bands + n);
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
        Vec<VEC> o;
#pragma unroll
        for (int t = 0; t < VEC; ++t) o.v[t] = (sp.omega * r.v[t]) * (1.0 / D.v[t]);
        stv<VEC>(sp.out0 + n, o);
      }
      continue;
    }
    int64_t zo[3], yo[3];
    {
      int km = k - 1, kp = k + 1;
      if (sp.wrapz) {
        if (km < 0) km = sp.nzl - 1;
        if (kp >= sp.nzl) kp = 0;
      }
      int jm = j - 1, jp = j + 1;
      if (sp.py) {
        if (jm < 0) jm = sp.ny - 1;
        if (jp >= sp.ny) jp = 0;
      } else {
        jm = jm < 0 ? 0 : jm;
        jp = jp >= sp.ny ? sp.ny - 1 : jp;
      }
      zo[0] = (int64_t)km * sp.P;
      zo[1] = (int64_t)k * sp.P;
      zo[2] = (int64_t)kp * sp.P;
      yo[0] = (int64_t)jm * sp.nx;
      yo[1] = (int64_t)j * sp.nx;
      yo[2] = (int64_t)jp * sp.nx;
    }
    for (int iv = tx; iv < nxv; iv += BX) {
      const int i0 = iv * VEC;
      const int64_t n = base + i0;
      int im = i0 - 1, ip = i0 + VEC;
      if (sp.px) {
        if (im < 0) im = sp.nx - 1;
        if (ip >= sp.nx) ip = 0;
      } else {
        im = im < 0 ? 0 : im;
        ip = ip >= sp.nx ? sp.nx - 1 : ip;
      }
      // gather the x values the stencil touches: per (dy, dz) a centre
      // vector plus the left / right scalar when the stencil reaches dx = -1/+1
      Vec<VEC> xc[3][3];
      double xl[3][3], xr[3][3];
#pragma unroll
      for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
          const bool any = uses<ST>(-1, dy, dz) || uses<ST>(0, dy, dz) || uses<ST>(1, dy, dz);
          if (any) {
            const double* p = sp.x + zo[dz + 1] + yo[dy + 1];
            xc[dy + 1][dz + 1] = ldv_ro<VEC>(p + i0);
            if (uses<ST>(-1, dy, dz)) xl[dy + 1][dz + 1] = __ldg(p + im);
            if (uses<ST>(1, dy, dz)) xr[dy + 1][dz + 1] = __ldg(p + ip);
          }
        }
      // two interleaved FMA chains (even / odd bands), summed at the end --
      // the same order as the fused chain kernel (chain.cu)
      double y[VEC], ya[VEC], yb[VEC], a0[VEC];
#pragma unroll
      for (int t = 0; t < VEC; ++t) ya[t] = yb[t] = 0.0;
#pragma unroll
      for (int d = 0; d < ST; ++d) {
        int dx = 0, dy = 0, dz = 0;
        offs<ST>(d, dx, dy, dz);
        const Vec<VEC> a = ldv_stream<VEC>(sp.bands + (int64_t)d * sp.N + n);
        const Vec<VEC>& c = xc[dy + 1][dz + 1];
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          double xv;
          if (dx == 0) xv = c.v[t];
          else if (dx < 0) xv = (t == 0) ? xl[dy + 1][dz + 1] : c.v[t - 1];
          else xv = (t == VEC - 1) ? xr[dy + 1][dz + 1] : c.v[t + 1];
          if (d == 0) a0[t] = a.v[t];
          if (d % 2 == 0) ya[t] = fma(a.v[t], xv, ya[t]);
          else yb[t] = fma(a.v[t], xv, yb[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < VEC; ++t) y[t] = ya[t] + yb[t];
      const Vec<VEC>& x0 = xc[1][1];
      Vec<VEC> o0, o1;
      if constexpr (MODE == SM_SPMV) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) o0.v[t] = y[t];
        stv<VEC>(sp.out0 + n, o0);
      } else if constexpr (MODE == SM_SPMV_SWEEP1) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = y[t];
          o1.v[t] = (sp.omega * y[t]) * (1.0 / a0[t]);
        }
        stv<VEC>(sp.out0 + n, o0);
        stv<VEC>(sp.out1 + n, o1);
      } else if constexpr (MODE == SM_SWEEP || MODE == SM_SWEEP_NORM) {
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = fma(sp.omega * (r.v[t] - y[t]), 1.0 / a0[t], x0.v[t]);
          if constexpr (MODE == SM_SWEEP_NORM) red[0] = fma(o0.v[t], o0.v[t], red[0]);
        }
        stv<VEC>(sp.out0 + n, o0);
      } else {  // residual
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = r.v[t] - y[t];
          red[0] = fma(o0.v[t], o0.v[t], red[0]);
          if constexpr (MODE == SM_RESID_SWEEP1) o1.v[t] = (sp.omega * o0.v[t]) * (1.0 / a0[t]);
        }
        stv<VEC>(sp.out0 + n, o0);
        if constexpr (MODE == SM_RESID_SWEEP1) stv<VEC>(sp.out1 + n, o1);
      }
    }
  }
  if constexpr (RED) block_reduce_store<1>(red, 1, sp.red);
}

// Truncation check: counts coefficients that reach outside a
// non-periodic axis and zero diagonals.
template <int ST>
__global__ void validate_kernel(const double* bands, int64_t N, int nx, int ny, int z0,
                                int nz_global, int pmask, unsigned* bad) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(n % nx);
    const int j = (int)((n / nx) % ny);
    const int k = (int)(n / ((int64_t)nx * ny)) + z0;
    unsigned cnt = 0;
    if (bands[n] == 0.0) ++cnt;
    for (int d = 1; d < ST; ++d) {
      int dx = 0, dy = 0, dz = 0;
      offs<ST>(d, dx, dy, dz);
      bool out = false;
      if (!(pmask & 1) && (i + dx < 0 || i + dx >= nx)) out = true;
      if (!(pmask & 2) && (j + dy < 0 || j + dy >= ny)) out = true;
      if (!(pmask & 4) && (k + dz < 0 || k + dz >= nz_global)) out = true;
      if (out && bands[(int64_t)d * N + n] != 0.0) ++cnt;
    }
    if (cnt) atomicAdd(bad, cnt);
  }
}

// Columns are processed in groups of 8 with unguarded loads (the host pads
// the last group with a duplicate pointer and zero coefficients), so every
// thread keeps 8 x VEC loads in flight per group.
constexpr int GRP = 8;

// ----------------------------------------------------------------- K3
// g_c = Q_c^T w for c < ncol (block dot, "[C V_j]^T w").  NC accumulators
// per thread; every column is streamed once, w once.
template <int NC, int VEC>
__global__ void __launch_bounds__(256) bdot_kernel(ColPtrs Q, int ncol, const double* __restrict__ w,
                                                   int64_t N, RedArgs ra) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t r = e * VEC;
    const Vec<VEC> wv = ldv_ro<VEC>(w + r);
#pragma unroll
    for (int g = 0; g < NC / GRP; ++g) {
      if (g * GRP < ncol) {
        Vec<VEC> q[GRP];
#pragma unroll
        for (int u = 0; u < GRP; ++u) q[u] = ldv_stream<VEC>(Q.p[g * GRP + u] + r);
#pragma unroll
        for (int u = 0; u < GRP; ++u)
#pragma unroll
          for (int t = 0; t < VEC; ++t) acc[g * GRP + u] = fma(q[u].v[t], wv.v[t], acc[g * GRP + u]);
      }
    }
  }
  block_reduce_store<NC>(acc, ncol, ra);
}

// ----------------------------------------------------------------- K4
// w <- w - sum_c Q_c gs*g_c, then optional dots of the new w with up to 3
// vectors (nullptr = w itself).
template <int NC, int ND, int VEC>
__global__ void __launch_bounds__(256) bupd_kernel(ColPtrs Q, int ncol, const double* __restrict__ g,
                                                   double gs, double* __restrict__ w, int64_t N,
                                                   const double* d0, const double* d1,
                                                   const double* d2, RedArgs ra) {
  __shared__ double gsh[NC];
  for (int c = threadIdx.x; c < NC; c += blockDim.x) gsh[c] = c < ncol ? gs * g[c] : 0.0;
  __syncthreads();
  double acc[ND > 0 ? ND : 1];
#pragma unroll
  for (int q = 0; q < (ND > 0 ? ND : 1); ++q) acc[q] = 0.0;
  const double* dv[3] = {d0, d1, d2};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t r = e * VEC;
    Vec<VEC> wv = ldv<VEC>(w + r);
#pragma unroll
    for (int gi = 0; gi < NC / GRP; ++gi) {
      if (gi * GRP < ncol) {
        Vec<VEC> q[GRP];
#pragma unroll
        for (int u = 0; u < GRP; ++u) q[u] = ldv_stream<VEC>(Q.p[gi * GRP + u] + r);
#pragma unroll
        for (int u = 0; u < GRP; ++u)
#pragma unroll
          for (int t = 0; t < VEC; ++t) wv.v[t] = fma(-gsh[gi * GRP + u], q[u].v[t], wv.v[t]);
      }
    }
    stv<VEC>(w + r, wv);
#pragma unroll
    for (int q = 0; q < ND; ++q) {
      Vec<VEC> o = wv;
      if (dv[q]) o = ldv_ro<VEC>(dv[q] + r);
#pragma unroll
      for (int t = 0; t < VEC; ++t) acc[q] = fma(o.v[t], wv.v[t], acc[q]);
    }
  }
  if constexpr (ND > 0) block_reduce_store<(ND > 0 ? ND : 1)>(acc, ND, ra);
}

// v_{j+1} = w / h_{j+1,j}, with the happy-breakdown test h <= 1e-14 ||A_hat v_j||
// (reading D18): on breakdown v_{j+1} = 0 and *flag = 1.
template <int VEC>
__global__ void __launch_bounds__(256) normalize_kernel(double* __restrict__ w, int64_t N,
                                                        const double* nrm2, const double* nin2,
                                                        double* flag) {
  const double h = sqrt(*nrm2);
  bool brk = false;
  if (nin2) brk = !(h > 1e-14 * sqrt(*nin2));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    Vec<VEC> v = ldv<VEC>(w + e * VEC);
#pragma unroll
    for (int t = 0; t < VEC; ++t) v.v[t] = brk ? 0.0 : v.v[t] / h;
    stv<VEC>(w + e * VEC, v);
  }
  if (flag && blockIdx.x == 0 && threadIdx.x == 0) *flag = brk ? 1.0 : 0.0;
}

// ----------------------------------------------------------------- K5
// out_o = scale_o * sum_c Q_c coef[o][c]  (+ out_o if acc_o), o < nout.
template <int NC, int VEC>
__global__ void __launch_bounds__(256) lincomb_kernel(ColPtrs Q, int ncol, const double* __restrict__ coef,
                                                      int nout, LcOut lo, int64_t N) {
  __shared__ double cs[MAXOUT][NC];
  for (int t = threadIdx.x; t < MAXOUT * NC; t += blockDim.x) {
    const int o = t / NC, c = t % NC;
    cs[o][c] = (o < nout && c < ncol) ? coef[o * ncol + c] : 0.0;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t r = e * VEC;
    double s[MAXOUT][VEC];
#pragma unroll
    for (int o = 0; o < MAXOUT; ++o)
#pragma unroll
      for (int t = 0; t < VEC; ++t) s[o][t] = 0.0;
#pragma unroll
    for (int gi = 0; gi < NC / GRP; ++gi) {
      if (gi * GRP < ncol) {
        Vec<VEC> q[GRP];
#pragma unroll
        for (int u = 0; u < GRP; ++u) q[u] = ldv_stream<VEC>(Q.p[gi * GRP + u] + r);
#pragma unroll
        for (int o = 0; o < MAXOUT; ++o) {
          if (o < nout) {
#pragma unroll
            for (int u = 0; u < GRP; ++u)
#pragma unroll
              for (int t = 0; t < VEC; ++t) s[o][t] = fma(q[u].v[t], cs[o][gi * GRP + u], s[o][t]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < MAXOUT; ++o) {
      if (o < nout) {
        Vec<VEC> v;
#pragma unroll
        for (int t = 0; t < VEC; ++t) v.v[t] = lo.scale[o] * s[o][t];
        if (lo.acc[o]) {
          const Vec<VEC> old = ldv<VEC>(lo.out[o] + r);
#pragma unroll
          for (int t = 0; t < VEC; ++t) v.v[t] = old.v[t] + v.v[t];
        }
        stv<VEC>(lo.out[o] + r, v);
      }
    }
  }
}

// Projection (Alg. 3 line 1b, Alg. 4 line 1c, reading D20):
// r <- r - C xi ; x <- x + U xi (x may be null) ; red ||r||^2.
template <int NC, int VEC>
__global__ void __launch_bounds__(256) proj_kernel(ColPtrs C, ColPtrs U, int k, const double* __restrict__ xi,
                                                   double* __restrict__ r, double* __restrict__ x,
                                                   int64_t N, RedArgs ra) {
  __shared__ double xs[NC];
  for (int c = threadIdx.x; c < NC; c += blockDim.x) xs[c] = c < k ? xi[c] : 0.0;
  __syncthreads();
  double acc[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t n = e * VEC;
    Vec<VEC> cr, ux;
#pragma unroll
    for (int t = 0; t < VEC; ++t) cr.v[t] = ux.v[t] = 0.0;
#pragma unroll
    for (int gi = 0; gi < NC / GRP; ++gi) {
      if (gi * GRP < k) {
        Vec<VEC> q[GRP];
#pragma unroll
        for (int u = 0; u < GRP; ++u) q[u] = ldv_stream<VEC>(C.p[gi * GRP + u] + n);
#pragma unroll
        for (int u = 0; u < GRP; ++u)
#pragma unroll
          for (int t = 0; t < VEC; ++t) cr.v[t] = fma(q[u].v[t], xs[gi * GRP + u], cr.v[t]);
        if (x) {
#pragma unroll
          for (int u = 0; u < GRP; ++u) q[u] = ldv_stream<VEC>(U.p[gi * GRP + u] + n);
#pragma unroll
          for (int u = 0; u < GRP; ++u)
#pragma unroll
            for (int t = 0; t < VEC; ++t) ux.v[t] = fma(q[u].v[t], xs[gi * GRP + u], ux.v[t]);
        }
      }
    }
    Vec<VEC> rv = ldv<VEC>(r + n);
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      rv.v[t] = rv.v[t] - cr.v[t];
      acc[0] = fma(rv.v[t], rv.v[t], acc[0]);
    }
    stv<VEC>(r + n, rv);
    if (x) {
      Vec<VEC> xv = ldv<VEC>(x + n);
#pragma unroll
      for (int t = 0; t < VEC; ++t) xv.v[t] = xv.v[t] + ux.v[t];
      stv<VEC>(x + n, xv);
    }
  }
  block_reduce_store<1>(acc, 1, ra);
}

// In-place column rotation  [q_0 .. q_{k-1}] <- [q_0 .. q_{k-1}] T  (T k x k,
// column-major): the QR refresh C <- C~ R^-1, U <- U R^-1 (K8).  Each thread
// owns whole rows, so in-place is race free.
template <int NC>
__global__ void __launch_bounds__(256) rotate_kernel(ColPtrs Qc, int k, const double* __restrict__ T,
                                                     int64_t N) {
  __shared__ double ts[NC * NC];
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) ts[t] = T[t];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += stride) {
    double in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < k) in[c] = Qc.p[c][n];
#pragma unroll
    for (int o = 0; o < NC; ++o) {
      if (o < k) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c < k) s = fma(in[c], ts[o * k + c], s);
        const_cast<double*>(Qc.p[o])[n] = s;
      }
    }
  }
}

// ------------------------------------------------------------ K6 rBiCGStab
// Alg. 4 line 6 fused with the first Jacobi sweep of p_hat = M^-1 p:
// p = r (i = 0) or p = r + beta (p - omega v), beta = (rho_i/rho_{i-1})(alpha/omega);
// z = w_l p / D (D == nullptr: no preconditioner, z = p).
template <int VEC>
__global__ void __launch_bounds__(256) bicg_p_kernel(const double* __restrict__ r, double* __restrict__ p,
                                                     const double* __restrict__ v, const double* __restrict__ D,
                                                     double* __restrict__ z, double wl, int64_t N,
                                                     const BiIter* cur, const BiIter* prev, int first) {
  double beta = 0.0, omega = 0.0;
  if (!first) {
    const double alpha = prev->rho / prev->sigma;
    omega = prev->ts / prev->tt;
    beta = (cur->rho / prev->rho) * (alpha / omega);
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t n = e * VEC;
    const Vec<VEC> rn = ldv_ro<VEC>(r + n);
    Vec<VEC> pn;
    if (first) {
      pn = rn;
    } else {
      const Vec<VEC> po = ldv<VEC>(p + n);
      const Vec<VEC> vn = ldv_ro<VEC>(v + n);
#pragma unroll
      for (int t = 0; t < VEC; ++t) pn.v[t] = rn.v[t] + beta * (po.v[t] - omega * vn.v[t]);
    }
    stv<VEC>(p + n, pn);
    Vec<VEC> zn = pn;
    if (D) {
      const Vec<VEC> dn = ldv_stream<VEC>(D + n);
#pragma unroll
      for (int t = 0; t < VEC; ++t) zn.v[t] = (wl * pn.v[t]) * (1.0 / dn.v[t]);
    }
    stv<VEC>(z + n, zn);
  }
}

// Alg. 4 line 8 fused with the first sweep of s_hat = M^-1 s:
// alpha = rho/sigma; s = r - alpha v; z = w_l s / D; red ||s||^2.
template <int VEC>
__global__ void __launch_bounds__(256) bicg_s_kernel(const double* __restrict__ r, const double* __restrict__ v,
                                                     double* __restrict__ s, const double* __restrict__ D,
                                                     double* __restrict__ z, double wl, int64_t N,
                                                     const BiIter* cur, RedArgs ra) {
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
      for (int t = 0; t < VEC; ++t) zn.v[t] = (wl * sn.v[t]) * (1.0 / dn.v[t]);
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
  for (int c = threadIdx.x; c < k; c += blockDim.x) xi[c] = -eta0[c];
  if (threadIdx.x == 0) it0->rr = it0->rho;
}

// =================================================================== host
namespace {

// Grid = min(work / CTA, SMs x resident CTAs of this instantiation).
template <typename... KArgs, typename... Args>
void launch_k(rk_ctx* ctx, void (*kern)(KArgs...), int64_t work_threads, dim3 blk,
              Args&&... args) {
  const int threads = (int)(blk.x * blk.y);
  auto it = ctx->occ_cache.find((const void*)kern);
  int occ;
  if (it == ctx->occ_cache.end()) {
    RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0));
    occ = std::max(1, occ);
    ctx->occ_cache[(const void*)kern] = occ;
  } else {
    occ = it->second;
  }
  const int64_t want = std::max<int64_t>(1, (work_threads + threads - 1) / threads);
  const int grid = (int)std::min<int64_t>(want, (int64_t)ctx->sms * occ);
  kern<<<grid, blk, 0, ctx->stream>>>(std::forward<Args>(args)...);
}

inline RedArgs red_args(rk_ctx* ctx, double* out) {
  return RedArgs{ctx->partials, ctx->counter, out};
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// VEC = 2 iff N is even and every pointer is 16-byte aligned.
int pick_vec(int64_t N, std::initializer_list<const void*> ps,
             const std::vector<const double*>& cols = {}) {
  if (N & 1) return 1;
  for (auto p : ps)
    if (p && !aligned16(p)) return 1;
  for (auto p : cols)
    if (p && !aligned16(p)) return 1;
  return 2;
}

// Pad to a multiple of GRP with the first column of the last group.
ColPtrs make_cols_padded(const std::vector<const double*>& v, int nc) {
  ColPtrs c;
  memset(&c, 0, sizeof(c));
  for (size_t i = 0; i < v.size(); ++i) c.p[i] = v[i];
  for (int i = (int)v.size(); i < nc && !v.empty(); ++i) {
    const int g0 = (i / GRP) * GRP;
    c.p[i] = v[g0 < (int)v.size() ? g0 : 0];
  }
  return c;
}

inline int nc_round(int n) { return ((std::max(n, 1) + GRP - 1) / GRP) * GRP; }

inline int nc_bucket(int n) {
  if (n <= 8) return 8;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  RK_REQUIRE(n <= 48, RK_EINVAL, "rotation supports k <= 48");
  return 48;
}

const char* stencil_cls(int mode) {
  switch (mode) {
    case SM_SPMV: return "stencil_spmv";
    case SM_SPMV_SWEEP1: return "stencil_spmv_sweep1";
    case SM_SWEEP: return "stencil_sweep";
    case SM_SWEEP_NORM: return "stencil_sweep";
    case SM_RESID: return "stencil_resid";
    case SM_RESID_SWEEP1: return "stencil_resid_sweep1";
    default: return "stencil_scale";
  }
}

// Algorithmic bytes per launch in units of W = 8 N.
double stencil_words(int S, int mode) {
  switch (mode) {
    case SM_SPMV: return S + 2;           // bands, x, y
    case SM_SPMV_SWEEP1: return S + 3;    // bands, x, t, z
    case SM_SWEEP:
    case SM_SWEEP_NORM: return S + 3;     // bands, z_in, r, z_out
    case SM_RESID: return S + 3;          // bands, x, b, r
    case SM_RESID_SWEEP1: return S + 4;   // bands, x, b, r, z
    default: return 3;                    // D, r, z
  }
}

template <int ST, int MODE>
void stencil_launch(rk_op* op, const StencilParams& sp, int vec, int64_t work, dim3 blk) {
  if (vec == 2) launch_k(op->ctx, stencil_kernel<ST, MODE, 2>, work, blk, sp);
  else launch_k(op->ctx, stencil_kernel<ST, MODE, 1>, work, blk, sp);
}

template <int ST>
void stencil_dispatch(rk_op* op, int mode, const StencilParams& sp, int vec, int64_t work, dim3 blk) {
  switch (mode) {
    case SM_SPMV: stencil_launch<ST, SM_SPMV>(op, sp, vec, work, blk); break;
    case SM_SPMV_SWEEP1: stencil_launch<ST, SM_SPMV_SWEEP1>(op, sp, vec, work, blk); break;
    case SM_SWEEP: stencil_launch<ST, SM_SWEEP>(op, sp, vec, work, blk); break;
    case SM_SWEEP_NORM: stencil_launch<ST, SM_SWEEP_NORM>(op, sp, vec, work, blk); break;
    case SM_RESID: stencil_launch<ST, SM_RESID>(op, sp, vec, work, blk); break;
    case SM_RESID_SWEEP1: stencil_launch<ST, SM_RESID_SWEEP1>(op, sp, vec, work, blk); break;
    case SM_SCALE: stencil_launch<ST, SM_SCALE>(op, sp, vec, work, blk); break;
    default: throw Error(RK_EINVAL, "bad stencil mode");
  }
}

}  // namespace

void init_ctx_kernels(rk_ctx* ctx) {
  int sms = 0;
  RK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  ctx->sms = sms;
  // per-CTA partials for up to MAXCOL + 4 values, up to 8 resident 256-thread CTAs per SM
  ctx->partials_cap = (size_t)(MAXCOL + 4) * sms * 8;
  RK_CUDA(cudaMalloc(&ctx->partials, ctx->partials_cap * sizeof(double)));
  RK_CUDA(cudaMalloc(&ctx->counter, 64));
  RK_CUDA(cudaMemset(ctx->counter, 0, 64));
}

void stencil(rk_op* op, int mode, const double* x, const double* r, double* out0, double* out1,
             double omega, double* red_out) {
  rk_ctx* ctx = op->ctx;
  if (mode != SM_SCALE) halo(op, x);
  StencilParams sp;
  sp.bands = op->bands;
  sp.N = op->N;
  sp.P = op->P;
  sp.nx = (int)op->g.nx;
  sp.ny = (int)op->g.ny;
  sp.nzl = (int)op->g.nz_local;
  sp.px = (op->g.periodic_mask & 1) ? 1 : 0;
  sp.py = (op->g.periodic_mask & 2) ? 1 : 0;
  sp.wrapz = op->wrapz;
  sp.x = x;
  sp.r = r;
  sp.out0 = out0;
  sp.out1 = out1;
  sp.omega = omega;
  const bool red = (mode == SM_SWEEP_NORM || mode == SM_RESID || mode == SM_RESID_SWEEP1);
  sp.red = red ? red_args(ctx, red_out) : RedArgs{nullptr, nullptr, nullptr};
  // VEC = 2 needs even rows and 16-byte aligned rows of every array
  int vec = (sp.nx % 2 == 0 && op->P % 2 == 0) ? pick_vec(op->N, {op->bands, x, r, out0, out1}) : 1;
  const int nxv = sp.nx / vec;
  const int bx = nxv >= 128 ? 128 : ((nxv + 31) / 32) * 32;
  dim3 blk(bx, 256 / bx);
  const int64_t rows = (int64_t)sp.ny * sp.nzl;
  const int64_t work = ((rows + blk.y - 1) / blk.y) * 256;
  Launch L(ctx, stencil_cls(mode), 8.0 * op->N * stencil_words(op->S, mode));
  switch (op->S) {
    case 7: stencil_dispatch<7>(op, mode, sp, vec, work, blk); break;
    case 19: stencil_dispatch<19>(op, mode, sp, vec, work, blk); break;
    case 27: stencil_dispatch<27>(op, mode, sp, vec, work, blk); break;
    default: throw Error(RK_EINVAL, "unsupported stencil");
  }
  L.done();
  if (red) allreduce(ctx, red_out, 1);
}

int validate_bands(rk_op* op) {
  rk_ctx* ctx = op->ctx;
  unsigned* bad;
  RK_CUDA(cudaMalloc(&bad, sizeof(unsigned)));
  RK_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), ctx->stream));
  const int grid = ctx->sms * 4;
  Launch L(ctx, "validate", 0);
#define RK_VAL(STV)                                                                              \
  validate_kernel<STV><<<grid, 256, 0, ctx->stream>>>(op->bands, op->N, (int)op->g.nx,          \
                                                      (int)op->g.ny, (int)op->g.z0,             \
                                                      (int)op->g.nz_global,                     \
                                                      (int)op->g.periodic_mask, bad)
  if (op->S == 7) RK_VAL(7);
  else if (op->S == 19) RK_VAL(19);
  else RK_VAL(27);
#undef RK_VAL
  L.done();
  unsigned h = 0;
  RK_CUDA(cudaMemcpyAsync(&h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  RK_CUDA(cudaStreamSynchronize(ctx->stream));
  RK_CUDA(cudaFree(bad));
  return (int)h;
}

// bdot launches cover <= 40 columns each (register budget: 40 accumulators).
void bdot(rk_ctx* ctx, const std::vector<const double*>& cols_all, const double* w, int64_t N,
          double* out) {
  const int total = (int)cols_all.size();
  RK_REQUIRE(total <= MAXCOL, RK_EINVAL, "too many columns in a block product");
  for (int off = 0; off < total; off += 40) {
    std::vector<const double*> cols(cols_all.begin() + off,
                                    cols_all.begin() + std::min(total, off + 40));
    const int ncol = (int)cols.size();
    const int nc = nc_round(ncol);
    const int vec = pick_vec(N, {w}, cols);
    RedArgs ra = red_args(ctx, out + off);
    ColPtrs Q = make_cols_padded(cols, nc);
    const int64_t work = N / vec;
    Launch L(ctx, "bdot", 8.0 * N * (ncol + 1));
#define RK_BDOT(NCV)                                                                     \
  if (vec == 2) launch_k(ctx, bdot_kernel<NCV, 2>, work, dim3(256), Q, ncol, w, N, ra);  \
  else launch_k(ctx, bdot_kernel<NCV, 1>, work, dim3(256), Q, ncol, w, N, ra);
    switch (nc) {
      case 8: RK_BDOT(8); break;
      case 16: RK_BDOT(16); break;
      case 24: RK_BDOT(24); break;
      case 32: RK_BDOT(32); break;
      default: RK_BDOT(40); break;
    }
#undef RK_BDOT
    L.done();
    allreduce(ctx, out + off, ncol);
  }
}

void bupd(rk_ctx* ctx, const std::vector<const double*>& cols, const double* g, double gscale,
          double* w, int64_t N, const std::vector<const double*>& dots, double* red_out) {
  const int ncol = (int)cols.size();
  const int nd = (int)dots.size();
  RK_REQUIRE(nd <= 3, RK_EINVAL, "bupd: at most 3 dots");
  RK_REQUIRE(ncol <= MAXCOL, RK_EINVAL, "too many columns in a block product");
  const int nc = nc_round(ncol);
  const int vec = pick_vec(N, {w, nd > 0 ? dots[0] : nullptr, nd > 1 ? dots[1] : nullptr,
                               nd > 2 ? dots[2] : nullptr}, cols);
  RedArgs ra = nd ? red_args(ctx, red_out) : RedArgs{nullptr, nullptr, nullptr};
  ColPtrs Q = make_cols_padded(cols, nc);
  const double* d[3] = {nullptr, nullptr, nullptr};
  for (int q = 0; q < nd; ++q) d[q] = dots[q];
  double words = ncol + 2;
  for (int q = 0; q < nd; ++q) words += dots[q] ? 1 : 0;
  const int64_t work = N / vec;
  Launch L(ctx, "bupd", 8.0 * N * words);
#define RK_BUPD(NCV, NDV)                                                                      \
  if (vec == 2)                                                                                \
    launch_k(ctx, bupd_kernel<NCV, NDV, 2>, work, dim3(256), Q, ncol, g, gscale, w, N, d[0],   \
             d[1], d[2], ra);                                                                  \
  else                                                                                         \
    launch_k(ctx, bupd_kernel<NCV, NDV, 1>, work, dim3(256), Q, ncol, g, gscale, w, N, d[0],   \
             d[1], d[2], ra);
#define RK_BUPD_NC(NCV)               \
  switch (nd) {                       \
    case 0: RK_BUPD(NCV, 0); break;   \
    case 1: RK_BUPD(NCV, 1); break;   \
    case 2: RK_BUPD(NCV, 2); break;   \
    default: RK_BUPD(NCV, 3); break;  \
  }
  switch (nc) {
    case 8: RK_BUPD_NC(8); break;
    case 16: RK_BUPD_NC(16); break;
    case 24: RK_BUPD_NC(24); break;
    case 32: RK_BUPD_NC(32); break;
    case 40: RK_BUPD_NC(40); break;
    case 48: RK_BUPD_NC(48); break;
    case 56: RK_BUPD_NC(56); break;
    case 64: RK_BUPD_NC(64); break;
    case 72: RK_BUPD_NC(72); break;
    default: RK_BUPD_NC(80); break;
  }
#undef RK_BUPD_NC
#undef RK_BUPD
  L.done();
  if (nd) allreduce(ctx, red_out, nd);
}

void normalize(rk_ctx* ctx, double* w, int64_t N, const double* nrm2, const double* nin2,
               double* flag) {
  const int vec = pick_vec(N, {w});
  Launch L(ctx, "normalize", 16.0 * N);
  if (vec == 2) launch_k(ctx, normalize_kernel<2>, N / 2, dim3(256), w, N, nrm2, nin2, flag);
  else launch_k(ctx, normalize_kernel<1>, N, dim3(256), w, N, nrm2, nin2, flag);
  L.done();
}

void lincomb(rk_ctx* ctx, const std::vector<const double*>& cols, const double* coef, int nout,
             const LcOut& lo, int64_t N) {
  const int ncol = (int)cols.size();
  RK_REQUIRE(nout >= 1 && nout <= MAXOUT, RK_EINVAL, "lincomb: 1..5 outputs");
  RK_REQUIRE(ncol >= 1 && ncol <= MAXCOL, RK_EINVAL, "lincomb: 1..80 columns");
  const int nc = nc_round(ncol);
  ColPtrs Q = make_cols_padded(cols, nc);
  int vec = pick_vec(N, {}, cols);
  for (int o = 0; o < nout; ++o)
    if (!aligned16(lo.out[o])) vec = 1;
  double words = ncol;
  for (int o = 0; o < nout; ++o) words += lo.acc[o] ? 2 : 1;
  const int64_t work = N / vec;
  Launch L(ctx, "lincomb", 8.0 * N * words);
#define RK_LC(NCV)                                                                              \
  if (vec == 2) launch_k(ctx, lincomb_kernel<NCV, 2>, work, dim3(256), Q, ncol, coef, nout, lo, N); \
  else launch_k(ctx, lincomb_kernel<NCV, 1>, work, dim3(256), Q, ncol, coef, nout, lo, N);
  switch (nc) {
    case 8: RK_LC(8); break;
    case 16: RK_LC(16); break;
    case 24: RK_LC(24); break;
    case 32: RK_LC(32); break;
    case 40: RK_LC(40); break;
    case 48: RK_LC(48); break;
    case 56: RK_LC(56); break;
    case 64: RK_LC(64); break;
    case 72: RK_LC(72); break;
    default: RK_LC(80); break;
  }
#undef RK_LC
  L.done();
}

void proj(rk_ctx* ctx, const std::vector<const double*>& C, const std::vector<const double*>& U,
          const double* xi, double* r, double* x, int64_t N, double* red_out) {
  const int k = (int)C.size();
  RK_REQUIRE(k >= 1 && k <= 48, RK_EINVAL, "projection supports 1 <= k <= 48");
  const int nc = nc_round(k);
  RedArgs ra = red_args(ctx, red_out);
  ColPtrs Cp = make_cols_padded(C, nc), Up = make_cols_padded(U, nc);
  int vec = pick_vec(N, {r, x}, C);
  if (x && pick_vec(N, {}, U) == 1) vec = 1;
  const int64_t work = N / vec;
  Launch L(ctx, "proj", 8.0 * N * (k * (x ? 2 : 1) + 2 + (x ? 2 : 0)));
#define RK_PJ(NCV)                                                                               \
  if (vec == 2) launch_k(ctx, proj_kernel<NCV, 2>, work, dim3(256), Cp, Up, k, xi, r, x, N, ra); \
  else launch_k(ctx, proj_kernel<NCV, 1>, work, dim3(256), Cp, Up, k, xi, r, x, N, ra);
  switch (nc) {
    case 8: RK_PJ(8); break;
    case 16: RK_PJ(16); break;
    case 24: RK_PJ(24); break;
    case 32: RK_PJ(32); break;
    case 40: RK_PJ(40); break;
    default: RK_PJ(48); break;
  }
#undef RK_PJ
  L.done();
  allreduce(ctx, red_out, 1);
}

void rotate(rk_ctx* ctx, const std::vector<double*>& cols, const double* T, int64_t N) {
  const int k = (int)cols.size();
  if (k == 0) return;
  const int nc = nc_bucket(k);
  ColPtrs Q;
  memset(&Q, 0, sizeof(Q));
  for (int c = 0; c < k; ++c) Q.p[c] = cols[c];
  Launch L(ctx, "rotate", 16.0 * N * k);
  switch (nc) {
    case 8: launch_k(ctx, rotate_kernel<8>, N, dim3(256), Q, k, T, N); break;
    case 16: launch_k(ctx, rotate_kernel<16>, N, dim3(256), Q, k, T, N); break;
    case 32: launch_k(ctx, rotate_kernel<32>, N, dim3(256), Q, k, T, N); break;
    default: launch_k(ctx, rotate_kernel<48>, N, dim3(256), Q, k, T, N); break;
  }
  L.done();
}

void bicg_p(rk_op* op, const double* r, double* p, const double* v, double* z, double wl,
            bool jacobi, const BiIter* cur, const BiIter* prev, int first) {
  rk_ctx* ctx = op->ctx;
  const double* D = jacobi ? op->bands : nullptr;
  const int vec = pick_vec(op->N, {r, p, v, z, D});
  Launch L(ctx, "bicg_p", 8.0 * op->N * ((first ? 3 : 5) + (jacobi ? 1 : 0)));
  if (vec == 2)
    launch_k(ctx, bicg_p_kernel<2>, op->N / 2, dim3(256), r, p, v, D, z, wl, op->N, cur, prev, first);
  else
    launch_k(ctx, bicg_p_kernel<1>, op->N, dim3(256), r, p, v, D, z, wl, op->N, cur, prev, first);
  L.done();
}

void bicg_s(rk_op* op, const double* r, const double* v, double* s, double* z, double wl,
            bool jacobi, BiIter* cur) {
  rk_ctx* ctx = op->ctx;
  const double* D = jacobi ? op->bands : nullptr;
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
  bicg_setup_kernel<<<1, 128, 0, ctx->stream>>>(xi, eta0, k, it0);
  L.done();
}

}  // namespace rk
