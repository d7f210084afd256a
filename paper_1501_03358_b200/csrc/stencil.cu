// sm_100a stencil kernels of librk (SURVEY.md §2.4 K1 SpMV, K2 Jacobi
// sweeps), one stage per launch; the temporally blocked chain is chain.cu.
// HBM-bound fp64 work on the CUDA cores (0.1-0.3 flop/B).
#include <cstdlib>

#include "kcommon.cuh"

namespace rk {

// -------------------------------------------------------------- K1 / K2
// Each thread owns VEC consecutive cells of an x-row (VEC = 2: 16-byte band
// and centre loads, the x-1 / x+VEC neighbours as scalars); rows (j, k) are
// grid-strided over the CTAs.  Out-of-grid neighbours on non-periodic x/y
// are clamped onto a valid cell (their coefficient is 0 by the truncation
// invariant); z neighbours read the ghost planes (zero, or halo data from the
// neighbouring rank), or wrap for a single-rank periodic z.
template <int ST, int MODE, int VEC>
__global__ void __launch_bounds__(256) stencil_kernel(StencilParams sp) {
  RK_PDL_ENTRY();
  RK_GATE(sp.gate);
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
        const Vec<VEC> iD = ldv_stream<VEC>(sp.invd + n);
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
        Vec<VEC> o;
#pragma unroll
        for (int t = 0; t < VEC; ++t) o.v[t] = (sp.omega * r.v[t]) * iD.v[t];
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
      // block-Jacobi local sweep (R17): no coupling across z-block boundaries
      if (sp.zb > 0) {
        const int g = sp.zg0 + k;
        const bool cut_m = (g % sp.zb) == 0, cut_p = ((g + 1) % sp.zb) == 0;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
#pragma unroll
          for (int t = 0; t < VEC; ++t) {
            if (cut_m) xc[dy][0].v[t] = 0.0;
            if (cut_p) xc[dy][2].v[t] = 0.0;
          }
          if (cut_m) xl[dy][0] = xr[dy][0] = 0.0;
          if (cut_p) xl[dy][2] = xr[dy][2] = 0.0;
        }
      }
      // interleaved FMA chains -- two (even / odd bands) for 7 points, four
      // (band d mod 4) for 19 / 27 points, summed at the end as (c0 + c1) + (c2
      // + c3) -- the same order as the fused chain kernels (chain.cu,
      // chain_x2.cuh, chain19.cuh)
      constexpr int NCH = ST >= 19 ? 4 : 2;
      double y[VEC], acc[NCH][VEC], a0[VEC];
#pragma unroll
      for (int t = 0; t < VEC; ++t)
#pragma unroll
        for (int q = 0; q < NCH; ++q) acc[q][t] = 0.0;
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
          acc[d % NCH][t] = fma(a.v[t], xv, acc[d % NCH][t]);
        }
      }
#pragma unroll
      for (int t = 0; t < VEC; ++t)
        y[t] = NCH == 4 ? (acc[0][t] + acc[1][t]) + (acc[2 % NCH][t] + acc[3 % NCH][t]) : acc[0][t] + acc[1][t];
      const Vec<VEC>& x0 = xc[1][1];
      Vec<VEC> o0, o1, iD;
      if constexpr (MODE == SM_SPMV_SWEEP1 || MODE == SM_SWEEP || MODE == SM_SWEEP_NORM ||
                    MODE == SM_RESID_SWEEP1)
        iD = ldv_stream<VEC>(sp.invd + n);
      if constexpr (MODE == SM_SPMV) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) o0.v[t] = y[t];
        stv<VEC>(sp.out0 + n, o0);
      } else if constexpr (MODE == SM_SPMV_SWEEP1) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = y[t];
          o1.v[t] = (sp.omega * y[t]) * iD.v[t];
        }
        stv<VEC>(sp.out0 + n, o0);
        stv<VEC>(sp.out1 + n, o1);
      } else if constexpr (MODE == SM_SWEEP || MODE == SM_SWEEP_NORM) {
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = fma(sp.omega * (r.v[t] - y[t]), iD.v[t], x0.v[t]);
          if constexpr (MODE == SM_SWEEP_NORM) red[0] = fma(o0.v[t], o0.v[t], red[0]);
        }
        stv<VEC>(sp.out0 + n, o0);
      } else {  // residual
        const Vec<VEC> r = ldv_ro<VEC>(sp.r + n);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          o0.v[t] = r.v[t] - y[t];
          red[0] = fma(o0.v[t], o0.v[t], red[0]);
          if constexpr (MODE == SM_RESID_SWEEP1) o1.v[t] = (sp.omega * o0.v[t]) * iD.v[t];
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
  RK_PDL_ENTRY();
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


// =================================================================== host
namespace {

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
  int l2 = 0;
  RK_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
  ctx->l2_bytes = l2;
  ctx->pdl = std::getenv("RK_NO_PDL") == nullptr;
  if (const char* m = std::getenv("RK_PDL_MODE")) ctx->pdl_mode = std::atoi(m);
  if (const char* m = std::getenv("RK_BDOT_BULK")) ctx->bdot_bulk = std::atoi(m);
  if (const char* m = std::getenv("RK_BUPD_BULK")) ctx->bupd_bulk = std::atoi(m);
  if (const char* m = std::getenv("RK_DEFER_COEF")) ctx->defer_coef = std::atoi(m) != 0;
  // per-CTA partials for up to MAXCOL + 4 values, up to 8 resident 256-thread CTAs per SM
  ctx->partials_cap = (size_t)(MAXCOL + 4) * sms * 8;
  RK_CUDA(cudaMalloc(&ctx->partials, ctx->partials_cap * sizeof(double)));
  RK_CUDA(cudaMalloc(&ctx->dpartials, ctx->partials_cap * sizeof(double)));
  RK_CUDA(cudaMalloc(&ctx->counter, 64));
  RK_CUDA(cudaMemset(ctx->counter, 0, 64));
}

void stencil(rk_op* op, int mode, const double* x, const double* r, double* out0, double* out1,
             double omega, double* red_out, int zb) {
  rk_ctx* ctx = op->ctx;
  // a local sweep on ranks that own whole z-blocks needs no halo (R17)
  const bool no_halo = zb > 0 && op->g.z0 % zb == 0 && op->g.nz_local % zb == 0;
  if (mode != SM_SCALE && !no_halo) halo(op, x);
  StencilParams sp;
  sp.bands = op->bands;
  sp.invd = op->invd();
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
  sp.zb = zb;
  sp.zg0 = (int)op->g.z0;
  sp.gate = ctx->gate;
  const bool red = (mode == SM_SWEEP_NORM || mode == SM_RESID || mode == SM_RESID_SWEEP1);
  sp.red = red ? red_args(ctx, red_out) : RedArgs{nullptr, nullptr, nullptr};
  // VEC = 2 needs even rows and 16-byte aligned rows of every array
  int vec = (sp.nx % 2 == 0 && op->P % 2 == 0) ? pick_vec(op->N, {op->bands, op->invd(), x, r, out0, out1}) : 1;
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

// Multicolour SOR pass of the SSOR preconditioner (reading R18): the cells
// of colour c = (i&1) + 2 (j&1) + 4 (k_global&1) are relaxed in place,
// z_n += w (r_n - (A z)_n) / D_n; they only couple to other colours (every
// stencil offset is in {-1,0,1}^3), so the pass is race free.  One thread
// per cell of the colour; x/y neighbours clamped (zero coefficient) or
// wrapped, z neighbours from the ghost planes or wrapped (single rank).
template <int ST>
__global__ void __launch_bounds__(256) colour_sweep_kernel(StencilParams sp, int colour) {
  RK_PDL_ENTRY();
  RK_GATE(sp.gate);
  const int ci = colour & 1, cj = (colour >> 1) & 1, ck = (colour >> 2) & 1;
  const int hx = (sp.nx - ci + 1) / 2;                 // cells of parity ci in a row
  const int hy = (sp.ny - cj + 1) / 2;
  const int kstart = ((ck - sp.zg0) % 2 + 2) % 2;      // first local plane of parity ck (global)
  const int hz = (sp.nzl - kstart + 1) / 2;
  const int64_t total = (int64_t)hx * hy * hz;
  double* z = const_cast<double*>(sp.x);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = ci + 2 * (int)(e % hx);
    const int64_t rest = e / hx;
    const int j = cj + 2 * (int)(rest % hy);
    const int k = kstart + 2 * (int)(rest / hy);
    const int64_t n = (int64_t)k * sp.P + (int64_t)j * sp.nx + i;
    double ya = 0.0, yb = 0.0;
#pragma unroll
    for (int d = 0; d < ST; ++d) {
      int dx = 0, dy = 0, dz = 0;
      offs<ST>(d, dx, dy, dz);
      int ii = i + dx, jj = j + dy, kk = k + dz;
      if (sp.px) ii = ii < 0 ? sp.nx - 1 : (ii >= sp.nx ? 0 : ii);
      else ii = ii < 0 ? 0 : (ii >= sp.nx ? sp.nx - 1 : ii);
      if (sp.py) jj = jj < 0 ? sp.ny - 1 : (jj >= sp.ny ? 0 : jj);
      else jj = jj < 0 ? 0 : (jj >= sp.ny ? sp.ny - 1 : jj);
      if (sp.wrapz) kk = kk < 0 ? sp.nzl - 1 : (kk >= sp.nzl ? 0 : kk);
      const double a = sp.bands[(int64_t)d * sp.N + n];
      const double xv = z[(int64_t)kk * sp.P + (int64_t)jj * sp.nx + ii];
      if (d % 2 == 0) ya = fma(a, xv, ya);
      else yb = fma(a, xv, yb);
    }
    z[n] = fma(sp.omega * (sp.r[n] - (ya + yb)), sp.invd[n], z[n]);
  }
}

void colour_sweep(rk_op* op, double* z, const double* r, double omega, int colour) {
  rk_ctx* ctx = op->ctx;
  halo(op, z);
  StencilParams sp{};
  sp.bands = op->bands;
  sp.invd = op->invd();
  sp.N = op->N;
  sp.P = op->P;
  sp.nx = (int)op->g.nx;
  sp.ny = (int)op->g.ny;
  sp.nzl = (int)op->g.nz_local;
  sp.px = (op->g.periodic_mask & 1) ? 1 : 0;
  sp.py = (op->g.periodic_mask & 2) ? 1 : 0;
  sp.wrapz = op->wrapz;
  sp.x = z;
  sp.r = r;
  sp.omega = omega;
  sp.zg0 = (int)op->g.z0;
  sp.gate = ctx->gate;
  const int64_t cells = (op->N + 7) / 8;
  Launch L(ctx, "ssor_colour", 8.0 * op->N * (op->S + 4) / 8.0);
  switch (op->S) {
    case 7: launch_k(ctx, colour_sweep_kernel<7>, cells, dim3(256), sp, colour); break;
    case 19: launch_k(ctx, colour_sweep_kernel<19>, cells, dim3(256), sp, colour); break;
    default: launch_k(ctx, colour_sweep_kernel<27>, cells, dim3(256), sp, colour); break;
  }
  L.done();
}

__global__ void invdiag_kernel(const double* __restrict__ D, double* __restrict__ inv, int64_t N) {
  RK_PDL_ENTRY();
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x)
    inv[n] = 1.0 / D[n];
}

void compute_invdiag(rk_op* op) {
  rk_ctx* ctx = op->ctx;
  Launch L(ctx, "invdiag", 16.0 * op->N);
  invdiag_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(op->bands, op->bands + (int64_t)op->S * op->N,
                                                       op->N);
  L.done();
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

}  // namespace rk
