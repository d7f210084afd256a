// 19-point chain, variant G (included by chain.cu): the bands do not pass
// through shared memory.  In chain19_kernel every band value crosses the
// SM's L1TEX / shared-memory port twice (TMA write into the band slot, LDS
// into registers) -- 20 of the ~23 arrays a launch streams -- and ncu put
// that port at ~70 % busy next to DRAM at ~80 %, which is why the kernel
// slows with the power-capped SM clock.  Here each thread loads its own
// cell's 20 band values (and the sweep's rhs) for plane tau + 1 from global
// memory straight into registers during step tau (one full step of lead; the
// band boxes of plane tau + 3 are prefetched into L2 by TMA so those loads
// hit L2), holding three register sets: plane tau + 1 (in flight), tau
// (stage 0) and tau - 1 (stage 1).  Shared memory keeps only the input-tile
// ring (6 slots, three x regions each, as chain19.cuh) and the stage ring.
// The step loop is unrolled 12 times, so every slot, ring plane, register
// set and barrier parity is a compile-time constant.  Per-cell arithmetic
// is stencil_kernel<19>'s (four FMA chains, 1/D band): bit-identical results.
#pragma once

namespace rk {

template <int TX, int TY>
struct C19GGeom {
  static constexpr int NST = 2, ST = 19, NBAND = 20;
  static constexpr int H = 1, EY = TY + 2, EX = TX + 2, HW = 2, XROWS = EY + 2;
  static_assert(TX == 32, "one warp per tile row");
  static constexpr int NWM = EY, NHALO = 2 * H * EY, NWH = (NHALO + 31) / 32;
  static constexpr int NTHR = 32 * (NWM + NWH);
  static constexpr int NXB = 6;                        // input-tile ring (planes tau-1 .. tau+4)
  __host__ __device__ static constexpr int al(int b) { return (b + 127) / 128 * 128; }
  static constexpr int XL_BYTES = XROWS * HW * 8, XM_BYTES = XROWS * TX * 8;
  static constexpr int X_BYTES = 2 * XL_BYTES + XM_BYTES;
  static constexpr int X_M = al(XL_BYTES), X_R = X_M + al(XM_BYTES);
  static constexpr int XSLOT = X_R + al(XL_BYTES);
  static constexpr int RING_BASE = NXB * XSLOT;
  static constexpr int RING = 4 * EY * EX * 8;
  static constexpr int BAR_BASE = RING_BASE + al(RING);
  static constexpr int SMEM = BAR_BASE + 8 * NXB + 128;
};

__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

template <int TX, int TY, int K0, int K1, int FL>
__global__ void __launch_bounds__(C19GGeom<TX, TY>::NTHR, 1)
chain19g_kernel(const __grid_constant__ CUtensorMap mbM, const __grid_constant__ CUtensorMap mbH,
                const __grid_constant__ CUtensorMap mxM, const __grid_constant__ CUtensorMap mxH,
                const __grid_constant__ CUtensorMap mgM, const __grid_constant__ CUtensorMap mgH,
                ChainParams cp) {
  RK_PDL_ENTRY();
  RK_GATE(cp.gate);
  using G = C19GGeom<TX, TY>;
  constexpr int H = G::H, EY = G::EY, EX = G::EX, HW = G::HW, NXB = G::NXB, NBAND = G::NBAND;
  constexpr bool LOAD_R = (K0 != CK_SPMV1);
  constexpr bool pz = (FL & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BAR_BASE);
  double* ring = reinterpret_cast<double*>(smem + G::RING_BASE);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  int c, ry;
  bool active;
  if (warp < G::NWM) {
    c = lane;
    ry = warp;
    active = true;
  } else {
    const int e = (warp - G::NWM) * 32 + lane;
    active = e < G::NHALO;
    const int ee = active ? e : 0;
    const int col = ee / EY;
    ry = ee - col * EY;
    c = col < H ? col - H : TX + (col - H);
  }
  const int nx = cp.nx, ny = cp.ny, nz = cp.nz;
  const int gx0 = (int)blockIdx.x * TX, gy0 = (int)blockIdx.y * TY - H;
  int gx = gx0 + c;
  if (cp.px) gx = gx < 0 ? gx + nx : (gx >= nx ? gx - nx : gx);
  const int gy = gy0 + ry;
  const bool inside = active && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
  const bool interior = active && c >= 0 && c < TX && ry >= H && ry < H + TY && inside;
  const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
  int xo[3][3];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx)
      xo[dy + 1][dx + 1] = region_off<TX, HW>(c + dx, ry + 1 + dy, G::X_M / 8, G::X_R / 8);
  const int gofs = ry * EX + (c + H);

  const int z0 = (int)blockIdx.z * cp.zc;
  const int z1 = min(nz, z0 + cp.zc);
  const int tau0 = z0 - H, tau_end = z1 + H;
  const int qfirst = tau0 - 1, qlast = tau_end;
  auto pl_of = [&](int q) { return pz ? (q < 0 ? q + nz : (q >= nz ? q - nz : q)) : q; };
  int xl = gx0 - HW, xr = gx0 + TX;
  if (cp.px) {
    xl = xl < 0 ? xl + nx : xl;
    xr = xr >= nx ? xr - nx : xr;
  }
  auto issue_x = [&](int q, int xs) {
    unsigned char* xb = smem + xs * G::XSLOT;
    const int z = pl_of(q) + GHOST;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bars[xs], G::X_BYTES);
    tma_load_3d(xb, &mxH, &bars[xs], xl, gy0 - 1, z);
    tma_load_3d(xb + G::X_M, &mxM, &bars[xs], gx0, gy0 - 1, z);
    tma_load_3d(xb + G::X_R, &mxH, &bars[xs], xr, gy0 - 1, z);
  };
  // L2 prefetch of the band boxes of plane q (ghost bands on several ranks)
  auto prefetch_b = [&](int q) {
    const int pl = pl_of(q);
    if ((FL & 4) && (pl < 0 || pl >= nz)) {
      const int gz = pl < 0 ? pl + BGHOST : pl - nz + BGHOST;
      tma_prefetch_4d(&mgM, gx0, gy0, gz, 0);
    } else if (pl >= 0 && pl < nz) {
      tma_prefetch_4d(&mbM, gx0, gy0, pl, 0);
      tma_prefetch_4d(&mbH, xl, gy0, pl, 0);
      tma_prefetch_4d(&mbH, xr, gy0, pl, 0);
    }
  };
  // this thread's bands (and rhs) of plane q into a register set; zero
  // outside the grid (the zero-ghost value)
  const int64_t N = cp.N, P = cp.P;
  auto load_b = [&](int q, double (&b)[NBAND], double& r) {
    const int pl = pl_of(q);
    const double* src = nullptr;
    const double* rsrc = nullptr;
    int64_t bs = N;
    if (inside) {
      if (pl >= 0 && pl < nz) {
        src = cp.bands + (int64_t)pl * P + cxy;
        if (LOAD_R) rsrc = cp.r + (int64_t)pl * P + cxy;
      } else if (FL & 4) {
        const int gz = pl < 0 ? pl + BGHOST : pl - nz + BGHOST;
        src = cp.gbands + (int64_t)gz * P + cxy;
        bs = (int64_t)(2 * BGHOST) * P;
        if (LOAD_R) rsrc = cp.r + (int64_t)pl * P + cxy;   // padded rhs: ghost planes filled
      }
    }
    if (src) {
#pragma unroll
      for (int d = 0; d < NBAND; ++d) b[d] = __ldg(src + d * bs);
    } else {
#pragma unroll
      for (int d = 0; d < NBAND; ++d) b[d] = 0.0;
    }
    if (LOAD_R) r = rsrc ? __ldg(rsrc) : 0.0;
  };

  if (tid == 0) {
    for (int s = 0; s < NXB; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int p = qfirst; p <= min(qfirst + NXB - 1, qlast); ++p) issue_x(p, p - qfirst);
    for (int q = tau0 + 1; q <= min(tau0 + 3, tau_end - 1); ++q) prefetch_b(q);
  }
  const double* xbase = reinterpret_cast<const double*>(smem);
  constexpr int XS = G::XSLOT / 8, RP = EY * EX;
  double bnd[3][NBAND];
  double rr[3] = {0.0, 0.0, 0.0};
  load_b(tau0, bnd[0], rr[0]);
#pragma unroll
  for (int d = 0; d < NBAND; ++d) bnd[1][d] = bnd[2][d] = 0.0;
  mbar_wait(&bars[0], 0);
  mbar_wait(&bars[1], 0);
  double xcm = xbase[xo[1][1]], xcc = xbase[XS + xo[1][1]];   // planes qfirst, tau0
  double hm = 0.0, hc = 0.0;

  auto apply19 = [](const double (&a)[NBAND], const double (&v)[19]) {
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < 19; ++d) s4[d % 4] = fma(a[d], v[d], s4[d % 4]);
    return (s4[0] + s4[1]) + (s4[2] + s4[3]);
  };

  // plane tau - tau0 = 12 it + U: register set U % 3 (tau), (U + 1) % 3
  // (tau + 1, loaded this step), (U + 2) % 3 (tau - 1, stage 1); input
  // tiles of planes tau-1, tau, tau+1 in slots U, U+1, U+2 (mod 6), the
  // latter's barrier in round 2 it + (U + 2) / 6
#define RK_C19G_STEP(U)                                                                           \
  {                                                                                               \
    if (tau >= tau_end) break;                                                                    \
    constexpr int S0 = (U) % 3, SN = ((U) + 1) % 3, S1 = ((U) + 2) % 3;                           \
    constexpr int XM = (U) % 6, X0 = ((U) + 1) % 6, XP = ((U) + 2) % 6;                           \
    if (tau + 1 < tau_end) load_b(tau + 1, bnd[SN], rr[SN]);                                      \
    mbar_wait(&bars[XP], (uint32_t)((((U) + 2) / 6) & 1));                                         \
    double v0 = 0.0;                                                                              \
    if (active) {                                                                                 \
      const double* tm = xbase + XM * XS;                                                         \
      const double* t0 = xbase + X0 * XS;                                                         \
      const double* tp = xbase + XP * XS;                                                         \
      bool cut_m = false, cut_p = false;                                                          \
      if ((FL & 1) && cp.zb > 0 && cp.local[0]) {                                                 \
        const int g = cp.zg0 + pl_of(tau);                                                        \
        cut_m = (g % cp.zb) == 0;                                                                 \
        cut_p = ((g + 1) % cp.zb) == 0;                                                           \
      }                                                                                           \
      const double xn = tp[xo[1][1]];                                                             \
      double v[19];                                                                               \
      v[0] = xcc;                                                                                 \
      v[1] = t0[xo[1][0]];                                                                        \
      v[2] = t0[xo[1][2]];                                                                        \
      v[3] = t0[xo[0][1]];                                                                        \
      v[4] = t0[xo[2][1]];                                                                        \
      v[5] = cut_m ? 0.0 : xcm;                                                                   \
      v[6] = cut_p ? 0.0 : xn;                                                                    \
      v[7] = t0[xo[0][0]];                                                                        \
      v[8] = t0[xo[0][2]];                                                                        \
      v[9] = t0[xo[2][0]];                                                                        \
      v[10] = t0[xo[2][2]];                                                                       \
      v[11] = cut_m ? 0.0 : tm[xo[0][1]];                                                         \
      v[12] = cut_m ? 0.0 : tm[xo[2][1]];                                                         \
      v[13] = cut_p ? 0.0 : tp[xo[0][1]];                                                         \
      v[14] = cut_p ? 0.0 : tp[xo[2][1]];                                                         \
      v[15] = cut_m ? 0.0 : tm[xo[1][0]];                                                         \
      v[16] = cut_m ? 0.0 : tm[xo[1][2]];                                                         \
      v[17] = cut_p ? 0.0 : tp[xo[1][0]];                                                         \
      v[18] = cut_p ? 0.0 : tp[xo[1][2]];                                                         \
      const double y = apply19(bnd[S0], v);                                                       \
      const double inv = bnd[S0][19];                                                             \
      if (K0 == CK_SPMV1) {                                                                       \
        rr[S0] = y;                                                                               \
        v0 = (cp.omega[0] * y) * inv;                                                             \
      } else if (K0 == CK_SWEEP) {                                                                \
        v0 = fma(cp.omega[0] * (rr[S0] - y), inv, xcc);                                           \
      } else {                                                                                    \
        v0 = y;                                                                                   \
      }                                                                                           \
      if (interior && tau >= z0 && tau < z1 && (pz || tau < nz)) {                                \
        const int64_t nn = (int64_t)pl_of(tau) * cp.P + cxy;                                      \
        if (K0 == CK_SPMV1 && cp.out_t) cp.out_t[nn] = y;                                         \
        if (cp.out_mid) cp.out_mid[nn] = v0;                                                      \
      }                                                                                           \
      ring[((U) & 3) * RP + gofs] = v0;                                                           \
      xcm = xcc;                                                                                  \
      xcc = xn;                                                                                   \
    }                                                                                             \
    __syncthreads();                                                                              \
    if (tid == 0) {                                                                               \
      if (tau + NXB - 1 <= qlast) issue_x(tau + NXB - 1, XM);                                     \
      if (tau + 4 <= tau_end - 1) prefetch_b(tau + 4);                                            \
    }                                                                                             \
    {                                                                                             \
      constexpr int RM = ((U) + 2) & 3, R0 = ((U) + 3) & 3, RQ = (U) & 3;                         \
      const int q = tau - 1;                                                                      \
      if (tau >= tau0 + 2 && interior) {                                                          \
        const double* rm = ring + RM * RP + gofs;                                                 \
        const double* r0 = ring + R0 * RP + gofs;                                                 \
        const double* rp = ring + RQ * RP + gofs;                                                 \
        bool cut_m = false, cut_p = false;                                                        \
        if ((FL & 1) && cp.zb > 0 && cp.local[1]) {                                               \
          const int g = cp.zg0 + pl_of(q);                                                        \
          cut_m = (g % cp.zb) == 0;                                                               \
          cut_p = ((g + 1) % cp.zb) == 0;                                                         \
        }                                                                                         \
        double v[19];                                                                             \
        v[0] = hc;                                                                                \
        v[1] = r0[-1];                                                                            \
        v[2] = r0[1];                                                                             \
        v[3] = r0[-EX];                                                                           \
        v[4] = r0[EX];                                                                            \
        v[5] = cut_m ? 0.0 : hm;                                                                  \
        v[6] = cut_p ? 0.0 : v0;                                                                  \
        v[7] = r0[-EX - 1];                                                                       \
        v[8] = r0[-EX + 1];                                                                       \
        v[9] = r0[EX - 1];                                                                        \
        v[10] = r0[EX + 1];                                                                       \
        v[11] = cut_m ? 0.0 : rm[-EX];                                                            \
        v[12] = cut_m ? 0.0 : rm[EX];                                                             \
        v[13] = cut_p ? 0.0 : rp[-EX];                                                            \
        v[14] = cut_p ? 0.0 : rp[EX];                                                             \
        v[15] = cut_m ? 0.0 : rm[-1];                                                             \
        v[16] = cut_m ? 0.0 : rm[1];                                                              \
        v[17] = cut_p ? 0.0 : rp[-1];                                                             \
        v[18] = cut_p ? 0.0 : rp[1];                                                              \
        const double y = apply19(bnd[S1], v);                                                     \
        const double vs = (K1 == CK_SWEEP) ? fma(cp.omega[1] * (rr[S1] - y), bnd[S1][19], hc) : y; \
        if (q >= z0 && q < z1) cp.out[(int64_t)pl_of(q) * cp.P + cxy] = vs;                       \
      }                                                                                           \
      hm = hc;                                                                                    \
      hc = v0;                                                                                    \
    }                                                                                             \
    ++tau;                                                                                        \
  }

  for (int tau = tau0; tau < tau_end;) {
    RK_C19G_STEP(0)
    RK_C19G_STEP(1)
    RK_C19G_STEP(2)
    RK_C19G_STEP(3)
    RK_C19G_STEP(4)
    RK_C19G_STEP(5)
    RK_C19G_STEP(6)
    RK_C19G_STEP(7)
    RK_C19G_STEP(8)
    RK_C19G_STEP(9)
    RK_C19G_STEP(10)
    RK_C19G_STEP(11)
  }
#undef RK_C19G_STEP
}

}  // namespace rk
