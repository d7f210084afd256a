// 19-point chain, THREE stages per launch on a CTA pair (included by
// chain.cu).  One CTA cannot hold three planes of 20-band coefficients per
// cell for a tile of useful size (chain19.cuh stops at two stages), so a
// thread-block cluster of two CTAs on neighbouring SMs shares the work of one
// x-y tile:
//   * the PRODUCER (cluster rank 0) runs stage 0 over the tile + 2-cell halo
//     (TMA-fed input ring, bands / rhs of plane tau) and stores its outputs
//     (and t = A x when stage 0 is CK_SPMV1) straight into the CONSUMER's
//     shared memory (DSMEM st.shared::cluster), one 4-plane ring; after the
//     step's barrier one thread publishes the plane (cluster-scope fence,
//     release-arrive on the consumer's "full" mbarrier);
//   * the CONSUMER (rank 1) runs stages 1 (tile + 1-cell halo) and 2 (tile)
//     with its own TMA-fed bands / rhs, as chain19.cuh's stages 0 and 1, and
//     hands each ring plane back with a release-arrive on the producer's
//     "empty" mbarrier once stage 1 no longer needs it.
// Every band value still crosses HBM once per three stages: a 6-stage
// preconditioned operator takes 2 launches of ~23 W instead of 3.  The
// producer runs up to 3 planes ahead of the consumer (ring depth).  Both
// step loops are unrolled 12 times so that every slot index and barrier
// parity is a compile-time constant (plus one run-time bit per 12 steps for
// the empty / full barriers).  Per-cell arithmetic is stencil_kernel<19>'s.
#pragma once

namespace rk {

template <int TY>
struct C19CGeom {
  static constexpr int TX = 32, NBAND = 20;
  // producer: stage 0 over rows [0, EY0) = tile rows + 2 halo each side,
  // columns [-2, TX + 2)
  static constexpr int EY0 = TY + 4, EX = TX + 4;
  static constexpr int HW0 = 4;                                // halo x-region width (even, >= 3)
  static constexpr int XROWS = EY0 + 2;                        // input tile rows (+1 y halo)
  static constexpr int NWM0 = EY0, NHALO0 = 4 * EY0, NWH0 = (NHALO0 + 31) / 32;
  static constexpr int NW0 = NWM0 + NWH0;
  // consumer: stage 1 over rows [1, EY0 - 1), columns [-1, TX + 1); stage 2 over the tile
  static constexpr int EY1 = TY + 2, HW1 = 2;
  static constexpr int NWM1 = EY1, NHALO1 = 2 * EY1, NWH1 = (NHALO1 + 31) / 32;
  static constexpr int NW1 = NWM1 + NWH1;
  static constexpr int NTHR = 32 * (NW0 > NW1 ? NW0 : NW1);
  static constexpr int NXB = 6, NB0 = 2, NB1 = 3;
  __host__ __device__ static constexpr int al(int b) { return (b + 127) / 128 * 128; }
  // producer slots
  static constexpr int XL = XROWS * HW0 * 8, XM = XROWS * TX * 8;
  static constexpr int X_M = al(XL), X_R = X_M + al(XM), XSLOT = X_R + al(XL), X_BYTES = 2 * XL + XM;
  static constexpr int B0L = NBAND * EY0 * HW0 * 8, B0M = NBAND * EY0 * TX * 8;
  static constexpr int B0_M = al(B0L), B0_R = B0_M + al(B0M), B0SLOT = B0_R + al(B0L);
  static constexpr int B0_BYTES = 2 * B0L + B0M;
  static constexpr int R0L = EY0 * HW0 * 8, R0M = EY0 * TX * 8;
  static constexpr int R0_M = al(R0L), R0_R = R0_M + al(R0M), R0SLOT = R0_R + al(R0L);
  static constexpr int R0_BYTES = 2 * R0L + R0M;
  static constexpr int P_XBASE = 0, P_BBASE = NXB * XSLOT, P_RBASE = P_BBASE + NB0 * B0SLOT;
  static constexpr int P_END = P_RBASE + NB0 * R0SLOT;
  // consumer slots
  static constexpr int B1L = NBAND * EY1 * HW1 * 8, B1M = NBAND * EY1 * TX * 8;
  static constexpr int B1_M = al(B1L), B1_R = B1_M + al(B1M), B1SLOT = B1_R + al(B1L);
  static constexpr int B1_BYTES = 2 * B1L + B1M;
  static constexpr int R1L = EY1 * HW1 * 8, R1M = EY1 * TX * 8;
  static constexpr int R1_M = al(R1L), R1_R = R1_M + al(R1M), R1SLOT = R1_R + al(R1L);
  static constexpr int R1_BYTES = 2 * R1L + R1M;
  static constexpr int RINGP = EY0 * EX;                       // doubles per ring plane
  static constexpr int C_BBASE = 0, C_RBASE = NB1 * B1SLOT;
  static constexpr int C_RING0 = al(C_RBASE + NB1 * R1SLOT);   // stage 0 outputs (written by the producer)
  static constexpr int C_RINGT = C_RING0 + 4 * RINGP * 8;      // t = A x (CK_SPMV1)
  static constexpr int C_RING1 = C_RINGT + 4 * RINGP * 8;      // stage 1 outputs
  static constexpr int C_END = C_RING1 + 4 * RINGP * 8;
  static constexpr int BAR_BASE = al(P_END > C_END ? P_END : C_END);
  // barriers: producer x (6), producer bands (2), producer empty (4);
  //           consumer bands (3), consumer full (4)
  static constexpr int BAR_PX = 0, BAR_PB = 6, BAR_PE = 8, BAR_CB = 12, BAR_CF = 15, NBAR = 19;
  static constexpr int SMEM = BAR_BASE + 8 * NBAR + 128;
};

__device__ __forceinline__ uint32_t mapa_peer(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_cluster(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0; !mbar_try_cluster(b, parity); ++it)
    if (it > (1u << 26)) __trap();
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// y = sum_d a_d v_d in stencil_kernel<19>'s order (four FMA chains)
__device__ __forceinline__ double apply19c(const double (&a)[20], const double (&v)[19]) {
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int d = 0; d < 19; ++d) s4[d % 4] = fma(a[d], v[d], s4[d % 4]);
  return (s4[0] + s4[1]) + (s4[2] + s4[3]);
}

// FL bit 0: block-Jacobi cuts, bit 1: periodic z (one rank), bit 2: ghost bands (ranks > 1)
template <int TY, int K0, int K1, int K2, int FL>
__global__ void __launch_bounds__(C19CGeom<TY>::NTHR, 1)   // 14 warps: <= 128 registers (4 warps per SM sub-partition)
chain19c_kernel(const __grid_constant__ CUtensorMap b0M, const __grid_constant__ CUtensorMap b0H,
                const __grid_constant__ CUtensorMap r0M, const __grid_constant__ CUtensorMap r0H,
                const __grid_constant__ CUtensorMap xM, const __grid_constant__ CUtensorMap xH,
                const __grid_constant__ CUtensorMap g0M, const __grid_constant__ CUtensorMap g0H,
                const __grid_constant__ CUtensorMap b1M, const __grid_constant__ CUtensorMap b1H,
                const __grid_constant__ CUtensorMap r1M, const __grid_constant__ CUtensorMap r1H,
                const __grid_constant__ CUtensorMap g1M, const __grid_constant__ CUtensorMap g1H,
                ChainParams cp) {
  RK_PDL_ENTRY();
  using G = C19CGeom<TY>;
  constexpr int TX = G::TX, EX = G::EX, EY0 = G::EY0, EY1 = G::EY1, NBAND = G::NBAND, RP = G::RINGP;
  constexpr bool LOAD_R = (K0 != CK_SPMV1);
  constexpr bool pz = (FL & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BAR_BASE);
  const uint32_t role = cluster_rank();   // 0 producer, 1 consumer
  const bool gated = cp.gate != nullptr && *cp.gate != 0.0;   // both CTAs read the same flag

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nx = cp.nx, ny = cp.ny, nz = cp.nz;
  const int gx0 = (int)(blockIdx.x >> 1) * TX, ty0 = (int)blockIdx.y * TY;   // tile origin
  const int z0 = (int)blockIdx.z * cp.zc;
  const int z1 = min(nz, z0 + cp.zc);
  const int tau0 = z0 - 2, tau_end = z1 + 2;      // stage-0 planes
  auto pl_of = [&](int q) { return pz ? (q < 0 ? q + nz : (q >= nz ? q - nz : q)) : q; };
  auto wrapx = [&](int x) { return cp.px ? (x < 0 ? x + nx : (x >= nx ? x - nx : x)) : x; };

  if (tid == 0) {
    for (int s = 0; s < G::NBAR; ++s) {
      mbar_init(&bars[s], 1u);   // one arrive per phase: a TMA batch or one signalling thread
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();   // both CTAs' barriers exist before any remote arrive
  if (gated) {
    cluster_sync_all();
    return;
  }

  if (role == 0) {
    // ================================================================ producer
    int c, ry;
    bool active;
    if (warp < G::NWM0) {
      c = lane;
      ry = warp;
      active = true;
    } else {
      const int e = (warp - G::NWM0) * 32 + lane;
      active = e < G::NHALO0;
      const int ee = active ? e : 0;
      const int col = ee / EY0;                  // 0..3
      ry = ee - col * EY0;
      c = col < 2 ? col - 2 : TX + (col - 2);    // -2, -1, TX, TX+1
    }
    const int gy0 = ty0 - 2;                     // global y of row 0
    const int gx = wrapx(gx0 + c), gy = gy0 + ry;
    const bool inside = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    const bool interior = active && c >= 0 && c < TX && ry >= 2 && ry < 2 + TY && inside;
    const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
    constexpr int HW = G::HW0;
    const int boff = region_off<TX, HW>(c, ry, G::B0_M / 8, G::B0_R / 8);
    const int bstr = EY0 * region_pitch<TX, HW>(c);
    const int roff = region_off<TX, HW>(c, ry, G::R0_M / 8, G::R0_R / 8);
    int xo[3][3];
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx)
        xo[dy + 1][dx + 1] = region_off<TX, HW>(c + dx, ry + 1 + dy, G::X_M / 8, G::X_R / 8);
    const uint32_t peer = 1u;
    const int gofs = ry * EX + (c + 2);
    const uint32_t ring0r = mapa_peer(smem + G::C_RING0, peer) + 8u * (uint32_t)gofs;
    const uint32_t ringtr = mapa_peer(smem + G::C_RINGT, peer) + 8u * (uint32_t)gofs;
    const uint32_t fullr = mapa_peer(&bars[G::BAR_CF], peer);
    const int xl = wrapx(gx0 - HW), xr = wrapx(gx0 + TX);
    const int qfirst = tau0 - 1, qlast = tau_end;
    auto issue_x = [&](int q, int xs) {
      unsigned char* xb = smem + G::P_XBASE + xs * G::XSLOT;
      uint64_t* bar = &bars[G::BAR_PX + xs];
      const int z = pl_of(q) + GHOST;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, G::X_BYTES);
      tma_load_3d(xb, &xH, bar, xl, gy0 - 1, z);
      tma_load_3d(xb + G::X_M, &xM, bar, gx0, gy0 - 1, z);
      tma_load_3d(xb + G::X_R, &xH, bar, xr, gy0 - 1, z);
    };
    auto issue_b = [&](int q, int bs) {
      unsigned char* bb = smem + G::P_BBASE + bs * G::B0SLOT;
      unsigned char* rb = smem + G::P_RBASE + bs * G::R0SLOT;
      uint64_t* bar = &bars[G::BAR_PB + bs];
      const int pl = pl_of(q);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, G::B0_BYTES + (LOAD_R ? G::R0_BYTES : 0));
      if ((FL & 4) && (pl < 0 || pl >= nz)) {
        const int gz = pl < 0 ? pl + BGHOST : pl - nz + BGHOST;
        tma_load_4d(bb, &g0H, bar, xl, gy0, gz, 0);
        tma_load_4d(bb + G::B0_M, &g0M, bar, gx0, gy0, gz, 0);
        tma_load_4d(bb + G::B0_R, &g0H, bar, xr, gy0, gz, 0);
      } else {
        tma_load_4d(bb, &b0H, bar, xl, gy0, pl, 0);
        tma_load_4d(bb + G::B0_M, &b0M, bar, gx0, gy0, pl, 0);
        tma_load_4d(bb + G::B0_R, &b0H, bar, xr, gy0, pl, 0);
      }
      if (LOAD_R) {
        const int rz = pl + cp.rz;
        tma_load_3d(rb, &r0H, bar, xl, gy0, rz);
        tma_load_3d(rb + G::R0_M, &r0M, bar, gx0, gy0, rz);
        tma_load_3d(rb + G::R0_R, &r0H, bar, xr, gy0, rz);
      }
    };
    if (tid == 0) {
      for (int p = qfirst; p <= min(qfirst + G::NXB - 1, qlast); ++p) issue_x(p, p - qfirst);
      for (int q = tau0; q <= min(tau0 + G::NB0 - 1, tau_end - 1); ++q) issue_b(q, q - tau0);
    }
    const double* xbase = reinterpret_cast<const double*>(smem + G::P_XBASE);
    const double* bbase = reinterpret_cast<const double*>(smem + G::P_BBASE);
    const double* rbase = reinterpret_cast<const double*>(smem + G::P_RBASE);
    constexpr int XS = G::XSLOT / 8, BSD = G::B0SLOT / 8, RSD = G::R0SLOT / 8;
    mbar_wait(&bars[G::BAR_PX + 0], 0);
    mbar_wait(&bars[G::BAR_PX + 1], 0);
    double xcm = xbase[xo[1][1]], xcc = xbase[XS + xo[1][1]];
    const bool mwarp = warp < G::NWM0;
    double bnd[NBAND];
    uint32_t itp = 0;   // parity bit of the 12-step round
    // plane tau - tau0 = 12 it + U: input tiles of tau-1, tau, tau+1 in slots
    // U, U+1, U+2 (mod 6); bands in slot U % 2; ring slot U % 4
#define RK_C19C_P(U)                                                                              \
  {                                                                                               \
    if (tau >= tau_end) break;                                                                    \
    constexpr int XM_ = (U) % 6, X0_ = ((U) + 1) % 6, XP_ = ((U) + 2) % 6, BS_ = (U) % 2;          \
    constexpr int RS_ = (U) % 4;                                                                  \
    mbar_wait(&bars[G::BAR_PB + BS_], (uint32_t)(((U) / 2) & 1));                                 \
    mbar_wait(&bars[G::BAR_PX + XP_], (uint32_t)((((U) + 2) / 6) & 1));                            \
    double v0 = 0.0, y = 0.0;                                                                     \
    if (active) {                                                                                 \
      const double* bsl = bbase + BS_ * BSD + boff;                                               \
      if (mwarp) {                                                                                \
        _Pragma("unroll") for (int d = 0; d < NBAND; ++d) bnd[d] = bsl[d * (EY0 * TX)];          \
      } else {                                                                                    \
        _Pragma("unroll") for (int d = 0; d < NBAND; ++d) bnd[d] = bsl[d * bstr];                \
      }                                                                                           \
      const double rv = LOAD_R ? rbase[BS_ * RSD + roff] : 0.0;                                   \
      const double* tm = xbase + XM_ * XS;                                                        \
      const double* t0 = xbase + X0_ * XS;                                                        \
      const double* tp = xbase + XP_ * XS;                                                        \
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
      y = apply19c(bnd, v);                                                                       \
      if (K0 == CK_SPMV1) v0 = (cp.omega[0] * y) * bnd[19];                                       \
      else if (K0 == CK_SWEEP) v0 = fma(cp.omega[0] * (rv - y), bnd[19], xcc);                    \
      else v0 = y;                                                                                \
      if (K0 == CK_SPMV1 && cp.out_t && interior && tau >= z0 && tau < z1)                        \
        cp.out_t[(int64_t)pl_of(tau) * cp.P + cxy] = y;                                           \
      xcm = xcc;                                                                                  \
      xcc = xn;                                                                                   \
    }                                                                                             \
    /* the consumer handed ring slot RS_ back (plane tau - 4 done) */                             \
    if (tau - tau0 >= 4) mbar_wait_cluster(&bars[G::BAR_PE + RS_], ((((U) / 4) + 1) ^ itp) & 1u);  \
    if (active) {                                                                                 \
      st_cluster_f64(ring0r + 8u * RS_ * RP, v0);                                                 \
      if (K0 == CK_SPMV1) st_cluster_f64(ringtr + 8u * RS_ * RP, y);                              \
    }                                                                                             \
    __syncthreads();                                                                              \
    if (tid == 0) {                                                                               \
      /* every thread's DSMEM stores precede the barrier; one cluster-scope   */                  \
      /* fence + release-arrive publishes them (one fence per plane, not 448) */                  \
      asm volatile("fence.acq_rel.cluster;" ::: "memory");                                        \
      mbar_arrive_remote(fullr + 8u * RS_);                                                       \
      if (tau + G::NXB - 1 <= qlast) issue_x(tau + G::NXB - 1, XM_);                              \
      if (tau + G::NB0 <= tau_end - 1) issue_b(tau + G::NB0, BS_);                                \
    }                                                                                             \
    ++tau;                                                                                        \
  }
    for (int tau = tau0; tau < tau_end; itp ^= 1u) {
      RK_C19C_P(0) RK_C19C_P(1) RK_C19C_P(2) RK_C19C_P(3) RK_C19C_P(4) RK_C19C_P(5)
      RK_C19C_P(6) RK_C19C_P(7) RK_C19C_P(8) RK_C19C_P(9) RK_C19C_P(10) RK_C19C_P(11)
    }
#undef RK_C19C_P
  } else {
    // ================================================================ consumer
    int c, ry;   // ry: row of the stage-0 region (1 .. EY0 - 2)
    bool active;
    if (warp < G::NWM1) {
      c = lane;
      ry = warp + 1;
      active = true;
    } else {
      const int e = (warp - G::NWM1) * 32 + lane;
      active = warp < G::NW1 && e < G::NHALO1;
      const int ee = active ? e : 0;
      const int col = ee / EY1;                  // 0, 1
      ry = ee - col * EY1 + 1;
      c = col == 0 ? -1 : TX;
    }
    const int gy0 = ty0 - 2;
    const int gx = wrapx(gx0 + c), gy = gy0 + ry;
    const bool inside = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    const bool interior = active && c >= 0 && c < TX && ry >= 2 && ry < 2 + TY && inside;
    const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
    constexpr int HW = G::HW1;
    const int boff = region_off<TX, HW>(c, ry - 1, G::B1_M / 8, G::B1_R / 8);
    const int bstr = EY1 * region_pitch<TX, HW>(c);
    const int roff = region_off<TX, HW>(c, ry - 1, G::R1_M / 8, G::R1_R / 8);
    const int gofs = ry * EX + (c + 2);
    const uint32_t emptyr = mapa_peer(&bars[G::BAR_PE], 0u);
    const int xl = wrapx(gx0 - HW), xr = wrapx(gx0 + TX);
    const int q0 = z0 - 1, q_end = z1 + 1;       // stage-1 planes
    auto issue_b = [&](int q, int bs) {
      unsigned char* bb = smem + G::C_BBASE + bs * G::B1SLOT;
      unsigned char* rb = smem + G::C_RBASE + bs * G::R1SLOT;
      uint64_t* bar = &bars[G::BAR_CB + bs];
      const int pl = pl_of(q);
      const int by = gy0 + 1;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, G::B1_BYTES + (LOAD_R ? G::R1_BYTES : 0));
      if ((FL & 4) && (pl < 0 || pl >= nz)) {
        const int gz = pl < 0 ? pl + BGHOST : pl - nz + BGHOST;
        tma_load_4d(bb, &g1H, bar, xl, by, gz, 0);
        tma_load_4d(bb + G::B1_M, &g1M, bar, gx0, by, gz, 0);
        tma_load_4d(bb + G::B1_R, &g1H, bar, xr, by, gz, 0);
      } else {
        tma_load_4d(bb, &b1H, bar, xl, by, pl, 0);
        tma_load_4d(bb + G::B1_M, &b1M, bar, gx0, by, pl, 0);
        tma_load_4d(bb + G::B1_R, &b1H, bar, xr, by, pl, 0);
      }
      if (LOAD_R) {
        const int rz = pl + cp.rz;
        tma_load_3d(rb, &r1H, bar, xl, by, rz);
        tma_load_3d(rb + G::R1_M, &r1M, bar, gx0, by, rz);
        tma_load_3d(rb + G::R1_R, &r1H, bar, xr, by, rz);
      }
    };
    if (tid == 0)
      for (int q = q0; q <= min(q0 + G::NB1 - 1, q_end - 1); ++q) issue_b(q, q - q0);
    const double* bbase = reinterpret_cast<const double*>(smem + G::C_BBASE);
    const double* rbase = reinterpret_cast<const double*>(smem + G::C_RBASE);
    const double* ring0 = reinterpret_cast<const double*>(smem + G::C_RING0) + gofs;
    const double* ringt = reinterpret_cast<const double*>(smem + G::C_RINGT) + gofs;
    double* ring1 = reinterpret_cast<double*>(smem + G::C_RING1) + gofs;
    constexpr int BSD = G::B1SLOT / 8, RSD = G::R1SLOT / 8;
    const bool mwarp = warp < G::NWM1;
    double bnd[2][NBAND];
    double rr[2] = {0.0, 0.0};
    double hm = 0.0, hc = 0.0;   // own stage-1 column at planes q-2, q-1
    // stage-0 planes q0 - 1 and q0 (ring slots 0 and 1, rounds 0)
    mbar_wait_cluster(&bars[G::BAR_CF + 0], 0);
    mbar_wait_cluster(&bars[G::BAR_CF + 1], 0);
    uint32_t itc = 0;
    // consumer step V = q - q0 = 12 it + U: stage-0 planes q-1, q, q+1 in ring
    // slots (U+0..2) % 4 (plane p in slot (p - tau0) % 4, p - tau0 = V + 1 ...);
    // bands of q in slot U % 3; register set U % 2
#define RK_C19C_C(U)                                                                              \
  {                                                                                               \
    if (q >= q_end) break;                                                                        \
    constexpr int SM_ = (U) % 4, S0_ = ((U) + 1) % 4, SP_ = ((U) + 2) % 4, BS_ = (U) % 3;          \
    constexpr int A_ = (U) % 2, B_ = ((U) + 1) % 2;                                               \
    /* plane q + 1: index q + 1 - tau0 = V + 2, round (V + 2) / 4 */                              \
    mbar_wait_cluster(&bars[G::BAR_CF + SP_], ((((U) + 2) / 4) ^ itc) & 1u);                       \
    mbar_wait(&bars[G::BAR_CB + BS_], (uint32_t)(((U) / 3) & 1));                                 \
    double v1 = 0.0;                                                                              \
    if (active) {                                                                                 \
      const double* bsl = bbase + BS_ * BSD + boff;                                               \
      if (mwarp) {                                                                                \
        _Pragma("unroll") for (int d = 0; d < NBAND; ++d) bnd[A_][d] = bsl[d * (EY1 * TX)];      \
      } else {                                                                                    \
        _Pragma("unroll") for (int d = 0; d < NBAND; ++d) bnd[A_][d] = bsl[d * bstr];            \
      }                                                                                           \
      rr[A_] = (K0 == CK_SPMV1) ? ringt[S0_ * RP] : (LOAD_R ? rbase[BS_ * RSD + roff] : 0.0);     \
      const double* rm = ring0 + SM_ * RP;                                                        \
      const double* r0 = ring0 + S0_ * RP;                                                        \
      const double* rp = ring0 + SP_ * RP;                                                        \
      bool cut_m = false, cut_p = false;                                                          \
      if ((FL & 1) && cp.zb > 0 && cp.local[1]) {                                                 \
        const int g = cp.zg0 + pl_of(q);                                                          \
        cut_m = (g % cp.zb) == 0;                                                                 \
        cut_p = ((g + 1) % cp.zb) == 0;                                                           \
      }                                                                                           \
      const double cc = r0[0];                                                                    \
      double v[19];                                                                               \
      v[0] = cc;                                                                                  \
      v[1] = r0[-1];                                                                              \
      v[2] = r0[1];                                                                               \
      v[3] = r0[-EX];                                                                             \
      v[4] = r0[EX];                                                                              \
      v[5] = cut_m ? 0.0 : rm[0];                                                                 \
      v[6] = cut_p ? 0.0 : rp[0];                                                                 \
      v[7] = r0[-EX - 1];                                                                         \
      v[8] = r0[-EX + 1];                                                                         \
      v[9] = r0[EX - 1];                                                                          \
      v[10] = r0[EX + 1];                                                                         \
      v[11] = cut_m ? 0.0 : rm[-EX];                                                              \
      v[12] = cut_m ? 0.0 : rm[EX];                                                               \
      v[13] = cut_p ? 0.0 : rp[-EX];                                                              \
      v[14] = cut_p ? 0.0 : rp[EX];                                                               \
      v[15] = cut_m ? 0.0 : rm[-1];                                                               \
      v[16] = cut_m ? 0.0 : rm[1];                                                                \
      v[17] = cut_p ? 0.0 : rp[-1];                                                               \
      v[18] = cut_p ? 0.0 : rp[1];                                                                \
      const double y = apply19c(bnd[A_], v);                                                      \
      v1 = (K1 == CK_SWEEP) ? fma(cp.omega[1] * (rr[A_] - y), bnd[A_][19], cc) : y;               \
      if (cp.out_mid && interior && q >= z0 && q < z1)                                            \
        cp.out_mid[(int64_t)pl_of(q) * cp.P + cxy] = v1;                                          \
      ring1[SM_ * RP] = v1;                 /* stage-1 plane q in ring-1 slot (q - q0) % 4 */      \
    }                                                                                             \
    __syncthreads();                                                                              \
    if (tid == 0) {                                                                               \
      mbar_arrive_remote(emptyr + 8u * SM_);   /* stage-0 plane q - 1 no longer needed */         \
      if (q + G::NB1 <= q_end - 1) issue_b(q + G::NB1, BS_);                                      \
    }                                                                                             \
    /* stage 2 at plane q - 1: stage-1 planes q-2, q-1, q from ring-1 slots U-2, U-1, U */       \
    {                                                                                             \
      constexpr int T2M = ((U) + 2) % 4, T20 = ((U) + 3) % 4, T2P = (U) % 4;                       \
      const int qq = q - 1;                                                                       \
      if (q >= q0 + 2 && interior) {                                                              \
        const double* rm = ring1 + T2M * RP;                                                      \
        const double* r0 = ring1 + T20 * RP;                                                      \
        const double* rp = ring1 + T2P * RP;                                                      \
        bool cut_m = false, cut_p = false;                                                        \
        if ((FL & 1) && cp.zb > 0 && cp.local[2]) {                                               \
          const int g = cp.zg0 + pl_of(qq);                                                       \
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
        v[6] = cut_p ? 0.0 : v1;                                                                  \
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
        const double y = apply19c(bnd[B_], v);                                                    \
        const double v2 = (K2 == CK_SWEEP) ? fma(cp.omega[2] * (rr[B_] - y), bnd[B_][19], hc) : y; \
        if (qq >= z0 && qq < z1) cp.out[(int64_t)pl_of(qq) * cp.P + cxy] = v2;                    \
      }                                                                                           \
      hm = hc;                                                                                    \
      hc = v1;                                                                                    \
    }                                                                                             \
    ++q;                                                                                          \
  }
    for (int q = q0; q < q_end; itc ^= 1u) {
      RK_C19C_C(0) RK_C19C_C(1) RK_C19C_C(2) RK_C19C_C(3) RK_C19C_C(4) RK_C19C_C(5)
      RK_C19C_C(6) RK_C19C_C(7) RK_C19C_C(8) RK_C19C_C(9) RK_C19C_C(10) RK_C19C_C(11)
    }
#undef RK_C19C_C
  }
  cluster_sync_all();   // neither CTA leaves while the other may still touch its shared memory
}

}  // namespace rk
