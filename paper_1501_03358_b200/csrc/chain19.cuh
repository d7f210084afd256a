// 19-point variant of the fused preconditioned-operator chain (included by
// chain.cu).  The channel operators of BASELINE configs[1]/[3] are 19-point
// (non-orthogonal grids) with periodic x and z, and their
// preconditioned operator is again a chain of 6 stencil stages over the same
// S + 1 = 20 band arrays, so fusing stages saves ~20 W per stage.
//
// What differs from the 7-point kernels:
//  * A 19-point stage at plane q reads the previous stage's values at planes
//    q-1 and q+1 with in-plane (+-x, +-y) neighbours, not only the centre, so
//    stage s (plane tau - s at step tau) reads stage s-1's plane computed in
//    the SAME step by other threads: a barrier separates consecutive stages
//    of a step (NST - 1 barriers per step) and the stage rings hold 4 planes.
//  * The bands of a plane (20 x 8 B per cell) are 2.5x the 7-point ones, so
//    the band tiles are smaller (TX x TY = 32 x 8 by default) and stay in
//    registers from stage 0 (which loads them from shared memory) through
//    the later stages of the plane.
//  * Periodic x: every tile is staged as three x regions -- the left halo
//    columns [gx0 - HW, gx0), the interior [gx0, gx0 + TX) and the right halo
//    [gx0 + TX, gx0 + TX + HW) -- each brought by its own TMA box.  On a
//    periodic x axis the halo boxes of the first / last tile start at the
//    wrapped coordinate; otherwise they lie outside the grid and TMA
//    zero-fills them (the zero-ghost semantics of non-periodic boundaries).
//    A TMA box lands densely, so each region is its own [rows][width] array
//    and every thread computes its neighbours' addresses once.
//  * Threads: one per cell.  Warps 0 .. EY-1 own the interior columns of one
//    tile row each (32 lanes = TX columns: conflict-free, row-aligned shared
//    loads); the last warps own the 2 H halo columns of every row.
// Per-cell arithmetic (band order, four FMA chains, 1/D band) is that of
// stencil_kernel<19>, so fused and unfused paths agree bit for bit.
#pragma once

namespace rk {

template <int NST, int TX, int TY, int PD>
struct C19Geom {
  static constexpr int ST = 19, NBAND = 20;           // register set: bands + 1/D
  // arrays streamed per plane: the 19 bands (+ the 1/D band unless
  // RK_C19_INVD = 0, where 1/D = 1.0 / D is recomputed at stage 0 -- the
  // same correctly rounded value invdiag_kernel stores)
  static constexpr int NBT = RK_C19_INVD ? 20 : 19;
  static constexpr int H = NST - 1;                    // recomputed halo of stage 0
  static constexpr int EY = TY + 2 * H;                // stage-0 rows
  static constexpr int EX = TX + 2 * H;                // stage-0 columns (ring pitch)
  static constexpr int HW = (H + 2) / 2 * 2;           // halo region width: even, >= H + 1
  static constexpr int XROWS = EY + 2;                 // input tile rows (+1 y halo)
  static_assert(TX == 32, "one warp per tile row");
  static constexpr int NWM = EY;                       // interior-column warps
  static constexpr int NHALO = 2 * H * EY;             // halo-column cells
  static constexpr int NWH = (NHALO + 31) / 32;
  static constexpr int NTHR = 32 * (NWM + NWH);
  static constexpr int NB = PD + 1;                    // band / rhs slots (planes tau .. tau+PD)
  static constexpr int NXB = 8;                        // input-tile ring (planes tau-1 .. tau+6)
  __host__ __device__ static constexpr int al(int b) { return (b + 127) / 128 * 128; }
  // band slot: regions L, M, R, each [NBAND][EY][w]
  static constexpr int BL_BYTES = NBT * EY * HW * 8, BM_BYTES = NBT * EY * TX * 8;
  static constexpr int B_BYTES = 2 * BL_BYTES + BM_BYTES;
  static constexpr int RL_BYTES = EY * HW * 8, RM_BYTES = EY * TX * 8;
  static constexpr int R_BYTES = 2 * RL_BYTES + RM_BYTES;
  static constexpr int XL_BYTES = XROWS * HW * 8, XM_BYTES = XROWS * TX * 8;
  static constexpr int X_BYTES = 2 * XL_BYTES + XM_BYTES;
  // region offsets inside a slot (bytes): L at 0, M, R (16-byte aligned: TMA destinations)
  static constexpr int B_M = al(BL_BYTES), B_R = B_M + al(BM_BYTES);
  static constexpr int BSLOT = B_R + al(BL_BYTES);
  static constexpr int R_M = al(RL_BYTES), R_R = R_M + al(RM_BYTES);
  static constexpr int RSLOT = R_R + al(RL_BYTES);
  static constexpr int X_M = al(XL_BYTES), X_R = X_M + al(XM_BYTES);
  static constexpr int XSLOT = X_R + al(XL_BYTES);
  static constexpr int RBASE = NB * BSLOT;                      // rhs slots
  static constexpr int XBASE = RBASE + NB * RSLOT;              // input tiles
  static constexpr int RING_BASE = XBASE + NXB * XSLOT;         // stage rings [NST-1][4][EY][EX]
  static constexpr int RING = (NST > 1 ? NST - 1 : 1) * 4 * EY * EX * 8;
  static constexpr int BAR_BASE = RING_BASE + al(RING);
  static constexpr int SMEM = BAR_BASE + 8 * (NXB + NB) + 128;
};

// Offsets (in doubles, within one slot) of a cell in a region-split tile:
// column c relative to the tile's first interior column, row r.
template <int TX, int HW>
__device__ __forceinline__ int region_off(int c, int r, int m_off, int r_off) {
  if (c < 0) return r * HW + (c + HW);
  if (c >= TX) return r_off + r * HW + (c - TX);
  return m_off + r * TX + c;
}
template <int TX, int HW>
__device__ __forceinline__ int region_pitch(int c) {
  return (c < 0 || c >= TX) ? HW : TX;
}

// KIND of stage s; FL bit 0: block-Jacobi cuts possible, bit 1: periodic z
// (one rank, wrapped in the kernel), bit 2: several ranks -- the bands of
// planes outside [0, nz) come from the ghost-band maps mgM / mgH.
template <int NST, int TX, int TY, int PD, int K0, int K1, int K2, int FL>
__global__ void __launch_bounds__(C19Geom<NST, TX, TY, PD>::NTHR, 1)
chain19_kernel(const __grid_constant__ CUtensorMap mbM, const __grid_constant__ CUtensorMap mbH,
               const __grid_constant__ CUtensorMap mrM, const __grid_constant__ CUtensorMap mrH,
               const __grid_constant__ CUtensorMap mxM, const __grid_constant__ CUtensorMap mxH,
               const __grid_constant__ CUtensorMap mgM, const __grid_constant__ CUtensorMap mgH,
               ChainParams cp) {
  RK_PDL_ENTRY();
  RK_GATE(cp.gate);
  using G = C19Geom<NST, TX, TY, PD>;
  constexpr int H = G::H, EY = G::EY, EX = G::EX, HW = G::HW, NB = G::NB, NXB = G::NXB;
  constexpr int NBAND = G::NBAND;
  constexpr bool LOAD_R = (K0 != CK_SPMV1);
  constexpr int KIND[3] = {K0, K1, K2};
  constexpr bool pz = (FL & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BAR_BASE);
  double* ring = reinterpret_cast<double*>(smem + G::RING_BASE);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // this thread's cell: column c (relative to the interior), row ry of the stage-0 region
  int c, ry;
  bool active;
  if (warp < G::NWM) {
    c = lane;
    ry = warp;
    active = true;
  } else {
    const int e = (warp - G::NWM) * 32 + lane;   // halo cell index
    active = e < G::NHALO;
    const int ee = active ? e : 0;
    const int col = ee / EY;                     // 0 .. 2H-1
    ry = ee - col * EY;
    c = col < H ? col - H : TX + (col - H);      // -H .. -1, TX .. TX+H-1
  }
  const int nx = cp.nx, ny = cp.ny, nz = cp.nz;
  const int gx0 = (int)blockIdx.x * TX, gy0 = (int)blockIdx.y * TY - H;
  int gx = gx0 + c;
  if (cp.px) gx = gx < 0 ? gx + nx : (gx >= nx ? gx - nx : gx);
  const int gy = gy0 + ry;
  const bool inside = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
  const bool interior = active && c >= 0 && c < TX && ry >= H && ry < H + TY && inside;
  const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
  // shared-memory offsets (doubles) of the own cell in a band / rhs slot and
  // of the 3 x 3 in-plane neighbourhood in an input tile
  const int boff = region_off<TX, HW>(c, ry, G::B_M / 8, G::B_R / 8);   // band 0
  const int bstr = EY * region_pitch<TX, HW>(c);                        // band stride
  const int roff = region_off<TX, HW>(c, ry, G::R_M / 8, G::R_R / 8);
  int xo[3][3];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx)
      xo[dy + 1][dx + 1] = region_off<TX, HW>(c + dx, ry + 1 + dy, G::X_M / 8, G::X_R / 8);
  const int gofs = ry * EX + (c + H);   // own cell in a ring plane

  const int z0 = (int)blockIdx.z * cp.zc;
  const int z1 = min(nz, z0 + cp.zc);
  const int tau0 = z0 - H;
  const int tau_end = z1 + H;
  const int qfirst = tau0 - 1, qlast = tau_end;   // input planes read
  const uint32_t b_bytes = G::B_BYTES + (LOAD_R ? G::R_BYTES : 0);
  uint64_t* bbar = bars + NXB;   // band / rhs slots' barriers
  auto pl_of = [&](int q) { return pz ? (q < 0 ? q + nz : (q >= nz ? q - nz : q)) : q; };
  // x coordinates of the three region boxes (wrapped on a periodic x axis)
  int xl = gx0 - HW, xr = gx0 + TX;
  if (cp.px) {
    xl = xl < 0 ? xl + nx : xl;
    xr = xr >= nx ? xr - nx : xr;
  }
  auto issue_x = [&](int q, int xs) {   // input tile of plane q (padded vector: z = pl + GHOST)
    unsigned char* xb = smem + G::XBASE + xs * G::XSLOT;
    const int z = pl_of(q) + GHOST;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bars[xs], G::X_BYTES);
    tma_load_3d(xb, &mxH, &bars[xs], xl, gy0 - 1, z);
    tma_load_3d(xb + G::X_M, &mxM, &bars[xs], gx0, gy0 - 1, z);
    tma_load_3d(xb + G::X_R, &mxH, &bars[xs], xr, gy0 - 1, z);
  };
  // band batch q: the bands (+ 1/D) and rhs of plane q, on band slot bs's barrier
  auto issue_b = [&](int q, int bs) {
    unsigned char* bb = smem + bs * G::BSLOT;
    unsigned char* rb = smem + G::RBASE + bs * G::RSLOT;
    const int pl = pl_of(q);
    uint64_t* bar = &bbar[bs];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, b_bytes);
    if ((FL & 4) && (pl < 0 || pl >= nz)) {
      const int gz = pl < 0 ? pl + BGHOST : pl - nz + BGHOST;
      tma_load_4d(bb, &mgH, bar, xl, gy0, gz, 0);
      tma_load_4d(bb + G::B_M, &mgM, bar, gx0, gy0, gz, 0);
      tma_load_4d(bb + G::B_R, &mgH, bar, xr, gy0, gz, 0);
    } else {
      tma_load_4d(bb, &mbH, bar, xl, gy0, pl, 0);
      tma_load_4d(bb + G::B_M, &mbM, bar, gx0, gy0, pl, 0);
      tma_load_4d(bb + G::B_R, &mbH, bar, xr, gy0, pl, 0);
    }
    if (LOAD_R) {
      const int rzz = pl + cp.rz;
      tma_load_3d(rb, &mrH, bar, xl, gy0, rzz);
      tma_load_3d(rb + G::R_M, &mrM, bar, gx0, gy0, rzz);
      tma_load_3d(rb + G::R_R, &mrH, bar, xr, gy0, rzz);
    }
  };

  // Arnoldi line 10 folded in (ChainParams::xs_*): the input tiles hold w;
  // each is scaled by 1 / h in shared memory once, after its TMA lands and a
  // step before its first read (normalize_kernel's arithmetic, so every
  // value the stages read is the v_{j+1} that kernel would have stored)
  const bool xsc = (K0 == CK_SPMV1) && cp.xs_n2 != nullptr;
  double xs_inv = 1.0;
  if (xsc) {
    const double h = sqrt(*cp.xs_n2);
    const bool brk = cp.xs_in2 && !(h > 1e-14 * sqrt(*cp.xs_in2));
    xs_inv = brk ? 0.0 : 1.0 / h;
    if (cp.xs_flag && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
      *cp.xs_flag = brk ? 1.0 : 0.0;
  }
  auto scale_x = [&](int xs) {   // input-tile slot xs: regions L, M, R
    double* xb = reinterpret_cast<double*>(smem + G::XBASE + xs * G::XSLOT);
    constexpr int NL = G::XROWS * HW, NM = G::XROWS * TX;
    for (int i = tid; i < NM; i += G::NTHR) xb[G::X_M / 8 + i] *= xs_inv;
    if (tid < 2 * NL) xb[tid < NL ? tid : G::X_R / 8 + (tid - NL)] *= xs_inv;
  };
  static_assert(2 * G::XROWS * G::HW <= G::NTHR, "one halo-region value per thread");

  if (tid == 0) {
    for (int s = 0; s < NXB + NB; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // prologue: input tiles qfirst .. qfirst + 7 (plane p in slot p - qfirst),
  // bands of planes tau0 .. tau0 + PD (plane q in slot q - tau0)
  if (tid == 0) {
    for (int p = qfirst; p <= min(qfirst + NXB - 1, qlast); ++p) issue_x(p, p - qfirst);
    for (int q = tau0; q <= min(tau0 + PD, tau_end - 1); ++q) issue_b(q, q - tau0);
  }
  mbar_wait(&bars[0], 0);
  mbar_wait(&bars[1], 0);
  // RK_C19_XREG (with the carried neighbourhoods, ROT0): the scale is applied
  // to each input value as it is loaded into registers (every input value
  // stage 0 uses passes through xcm / xcc / xn / a0 / p0 / nb), not by a pass
  // over the tile in shared memory
  constexpr bool XREG = RK_C19_XREG && (RK_C19_ROT & 1) && K0 == CK_SPMV1;
  if (!XREG && xsc) {   // planes qfirst .. qfirst + 2: the tiles step tau0 reads
    scale_x(0);
    scale_x(1);
    if (qfirst + 2 <= qlast) {
      mbar_wait(&bars[2], 0);
      scale_x(2);
    }
    __syncthreads();
  }
  // Input-tile slots are compile-time: the step loop is unrolled 8 times and
  // plane tau - tau0 = 8 it + U reads tiles of planes tau-1, tau, tau+1 from
  // slots U, U+1, U+2 (mod 8; plane p lives in slot (p - qfirst) & 7), ring
  // slot U & 3 and register band set U % NST, so every input / ring access is
  // a per-thread offset register plus an immediate.  Tiles are issued 7
  // planes ahead (after step tau's barrier, plane tau + 7 into the slot of
  // plane tau - 1); the PD + 1 band slots rotate at run time (one pointer per
  // step, then immediates), bands of plane tau + PD + 1 issued after step
  // tau's barrier into plane tau's slot.
  static_assert(NXB == 8 && NST <= 2, "compile-time input slots need an 8-slot ring and NST <= 2");
  int bs0 = 0;             // band slot of plane tau
  uint32_t bpar = 0;       // its barrier parity
  const double* xbase = reinterpret_cast<const double*>(smem + G::XBASE);
  const double* bbase = reinterpret_cast<const double*>(smem);
  const double* rbase = reinterpret_cast<const double*>(smem + G::RBASE);
  constexpr int XS = G::XSLOT / 8, BSD = G::BSLOT / 8, RSD = G::RSLOT / 8, RP = EY * EX;
  const bool mwarp = warp < G::NWM;   // interior-column warp: band stride EY * TX

  double bnd[NST][NBAND];
  double rr[NST];
#pragma unroll
  for (int s = 0; s < NST; ++s) {
    rr[s] = 0.0;
#pragma unroll
    for (int d = 0; d < NBAND; ++d) bnd[s][d] = 0.0;
  }
  // own z-columns: input at planes tau-1, tau (registers); stage 0's outputs
  // at the two planes below the one it produced last
  // (XREG: x * 1.0 when the launch does not normalise -- the same value)
  const double xm = XREG ? xs_inv : 1.0;
  double xcm = xbase[xo[1][1]] * xm, xcc = xbase[XS + xo[1][1]] * xm;   // planes qfirst, tau0: slots 0, 1
  double hm = 0.0, hc = 0.0;
  // In-plane neighbourhoods carried in registers from step to step (each
  // tile / ring value is read from shared memory once per thread instead of
  // up to three times): order W, E, S, N, SW, SE, NW, NE (xo[1][0], xo[1][2],
  // xo[0][1], xo[2][1], xo[0][0], xo[0][2], xo[2][0], xo[2][2]).
  //   stage 0: a0 = input plane tau's 8 neighbours, p0 = plane tau-1's 4 edges;
  //   stage 1: a1 = stage-0 plane tau-1's 8 neighbours, p1 = plane tau-2's 4 edges.
  // RK_C19_ROT bit 0: stage 0 carries, bit 1: stage 1 carries.
  constexpr bool ROT0 = (RK_C19_ROT & 1) != 0, ROT1 = (RK_C19_ROT & 2) != 0;
  const int xn8[8] = {xo[1][0], xo[1][2], xo[0][1], xo[2][1], xo[0][0], xo[0][2], xo[2][0], xo[2][2]};
  constexpr int rn8[8] = {-1, 1, -EX, EX, -EX - 1, -EX + 1, EX - 1, EX + 1};
  double a0[8], p0[4], a1[8], p1[4];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    a0[e] = ROT0 ? xbase[XS + xn8[e]] * xm : 0.0;
    a1[e] = 0.0;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    p0[e] = ROT0 ? xbase[xn8[e]] * xm : 0.0;
    p1[e] = 0.0;
  }

  // y = sum_d a_d v_d in stencil_kernel<19>'s order: four FMA chains (band
  // d mod 4), summed as (c0 + c1) + (c2 + c3) -- half the dependent-FMA
  // latency of two chains (the "wait" stall led the PC samples)
  auto apply19 = [](const double (&a)[NBAND], const double (&v)[19]) {
    double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < 19; ++d) c[d % 4] = fma(a[d], v[d], c[d % 4]);
    return (c[0] + c[1]) + (c[2] + c[3]);
  };

#define RK_C19_STEP(U)                                                                            \
  {                                                                                               \
    if (tau >= tau_end) break;                                                                    \
    constexpr int PH = (U) % NST, XM = (U) & 7, X0 = ((U) + 1) & 7, XP = ((U) + 2) & 7;           \
    mbar_wait(&bbar[bs0], bpar);                                                                  \
    mbar_wait(&bars[XP], (U) < 6 ? par : par ^ 1u);                                               \
    double v0 = 0.0;                                                                              \
    /* every thread runs stage 0: the spare lanes of the halo warp (!active) alias halo cell 0 */ \
    /* and store the same value to the same ring entry, so no branch splits the carried registers */ \
    if (RK_C19_ALLLANES || active) {                                                              \
      /* stage 0 at plane tau: bands / rhs to registers, input neighbours from the tiles */      \
      const double* bsl = bbase + bs0 * BSD + boff;                                               \
      if (mwarp) {                                                                                \
        _Pragma("unroll") for (int d = 0; d < G::NBT; ++d) bnd[PH][d] = bsl[d * (EY * TX)];      \
      } else {                                                                                    \
        _Pragma("unroll") for (int d = 0; d < G::NBT; ++d) bnd[PH][d] = bsl[d * bstr];           \
      }                                                                                           \
      if (!RK_C19_INVD) bnd[PH][19] = bnd[PH][0] != 0.0 ? 1.0 / bnd[PH][0] : 0.0;                 \
      if (LOAD_R) rr[PH] = rbase[bs0 * RSD + roff];                                               \
      const double* tm = xbase + XM * XS;                                                         \
      const double* t0 = xbase + X0 * XS;                                                         \
      const double* tp = xbase + XP * XS;                                                         \
      bool cut_m = false, cut_p = false;                                                          \
      if ((FL & 1) && cp.zb > 0 && cp.local[0]) {                                                 \
        const int g = cp.zg0 + pl_of(tau);                                                        \
        cut_m = (g % cp.zb) == 0;                                                                 \
        cut_p = ((g + 1) % cp.zb) == 0;                                                           \
      }                                                                                           \
      const double xn = tp[xo[1][1]] * xm;                                                        \
      double nb[8];   /* plane tau+1's neighbours (all 8 when carried, else the 4 edges) */      \
      _Pragma("unroll") for (int e = 0; e < (ROT0 ? 8 : 4); ++e) nb[e] = tp[xn8[e]] * xm;       \
      double v[19];                                                                               \
      v[0] = xcc;                                                                                 \
      v[1] = ROT0 ? a0[0] : t0[xo[1][0]];                                                         \
      v[2] = ROT0 ? a0[1] : t0[xo[1][2]];                                                         \
      v[3] = ROT0 ? a0[2] : t0[xo[0][1]];                                                         \
      v[4] = ROT0 ? a0[3] : t0[xo[2][1]];                                                         \
      v[5] = cut_m ? 0.0 : xcm;                                                                   \
      v[6] = cut_p ? 0.0 : xn;                                                                    \
      v[7] = ROT0 ? a0[4] : t0[xo[0][0]];                                                         \
      v[8] = ROT0 ? a0[5] : t0[xo[0][2]];                                                         \
      v[9] = ROT0 ? a0[6] : t0[xo[2][0]];                                                         \
      v[10] = ROT0 ? a0[7] : t0[xo[2][2]];                                                        \
      v[11] = cut_m ? 0.0 : (ROT0 ? p0[2] : tm[xo[0][1]]);                                        \
      v[12] = cut_m ? 0.0 : (ROT0 ? p0[3] : tm[xo[2][1]]);                                        \
      v[13] = cut_p ? 0.0 : nb[2];                                                                \
      v[14] = cut_p ? 0.0 : nb[3];                                                                \
      v[15] = cut_m ? 0.0 : (ROT0 ? p0[0] : tm[xo[1][0]]);                                        \
      v[16] = cut_m ? 0.0 : (ROT0 ? p0[1] : tm[xo[1][2]]);                                        \
      v[17] = cut_p ? 0.0 : nb[0];                                                                \
      v[18] = cut_p ? 0.0 : nb[1];                                                                \
      if (ROT0) {                                                                                 \
        _Pragma("unroll") for (int e = 0; e < 4; ++e) p0[e] = a0[e];                              \
        _Pragma("unroll") for (int e = 0; e < 8; ++e) a0[e] = nb[e];                              \
      }                                                                                           \
      const double y = apply19(bnd[PH], v);                                                       \
      const double inv = bnd[PH][19];                                                             \
      if (K0 == CK_SPMV1) {                                                                       \
        rr[PH] = y;                                                                               \
        v0 = (cp.omega[0] * y) * inv;                                                             \
      } else if (K0 == CK_SWEEP) {                                                                \
        v0 = fma(cp.omega[0] * (rr[PH] - y), inv, xcc);                                           \
      } else {                                                                                    \
        v0 = y;                                                                                   \
      }                                                                                           \
      if (interior && tau >= z0 && tau < z1 && (pz || tau < nz)) {                                \
        const int64_t nn = (int64_t)pl_of(tau) * cp.P + cxy;                                      \
        if (K0 == CK_SPMV1 && cp.out_t) cp.out_t[nn] = y;                                         \
        if (xsc && cp.xs_out) cp.xs_out[nn] = xcc;   /* v_{j+1} at plane tau */                   \
        if (NST == 1) cp.out[nn] = v0;                                                            \
        if (NST == 2 && cp.out_mid) cp.out_mid[nn] = v0;                                          \
      }                                                                                           \
      if (NST > 1) ring[((U) & 3) * RP + gofs] = v0;   /* ring slot (tau - tau0) & 3 */          \
      xcm = xcc;                                                                                  \
      xcc = xn;                                                                                   \
    }                                                                                             \
    /* normalisation folded in: plane tau+2's tile (slot (U+3)&7), first read at step tau+1 */    \
    if (!XREG && xsc && tau + 2 <= qlast) {                                                       \
      mbar_wait(&bars[((U) + 3) & 7], (U) < 5 ? par : par ^ 1u);                                  \
      scale_x(((U) + 3) & 7);                                                                     \
    }                                                                                             \
    __syncthreads();                                                                              \
    /* the slots of plane tau-1's tile and plane tau's bands / rhs are free */                    \
    if (tid == 0) {                                                                               \
      if (tau + 7 <= qlast) issue_x(tau + 7, XM);                                                 \
      if (tau + PD + 1 <= tau_end - 1) issue_b(tau + PD + 1, bs0);                                \
    }                                                                                             \
    if constexpr (NST == 2) {                                                                     \
      /* stage 1 at plane q = tau - 1: stage 0 at planes q-1, q, q+1 from ring slots           */ \
      /* (U-2)&3, (U-1)&3, U&3 (own column from registers), bands / rhs of q from set PH ^ 1    */ \
      constexpr int R = (PH + 1) % 2, RM = ((U) + 2) & 3, R0 = ((U) + 3) & 3, RQ = (U) & 3;       \
      double vs = 0.0;                                                                            \
      const int q = tau - 1;                                                                      \
      double nr[8];   /* stage-0 plane tau's neighbours (carried: read once, every step) */      \
      if (ROT1 && interior) {                                                                     \
        const double* rp = ring + RQ * RP + gofs;                                                 \
        _Pragma("unroll") for (int e = 0; e < 8; ++e) nr[e] = rp[rn8[e]];                         \
      }                                                                                           \
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
        v[1] = ROT1 ? a1[0] : r0[-1];                                                             \
        v[2] = ROT1 ? a1[1] : r0[1];                                                              \
        v[3] = ROT1 ? a1[2] : r0[-EX];                                                            \
        v[4] = ROT1 ? a1[3] : r0[EX];                                                             \
        v[5] = cut_m ? 0.0 : hm;                                                                  \
        v[6] = cut_p ? 0.0 : v0;                                                                  \
        v[7] = ROT1 ? a1[4] : r0[-EX - 1];                                                        \
        v[8] = ROT1 ? a1[5] : r0[-EX + 1];                                                        \
        v[9] = ROT1 ? a1[6] : r0[EX - 1];                                                         \
        v[10] = ROT1 ? a1[7] : r0[EX + 1];                                                        \
        v[11] = cut_m ? 0.0 : (ROT1 ? p1[2] : rm[-EX]);                                           \
        v[12] = cut_m ? 0.0 : (ROT1 ? p1[3] : rm[EX]);                                            \
        v[13] = cut_p ? 0.0 : (ROT1 ? nr[2] : rp[-EX]);                                           \
        v[14] = cut_p ? 0.0 : (ROT1 ? nr[3] : rp[EX]);                                            \
        v[15] = cut_m ? 0.0 : (ROT1 ? p1[0] : rm[-1]);                                            \
        v[16] = cut_m ? 0.0 : (ROT1 ? p1[1] : rm[1]);                                             \
        v[17] = cut_p ? 0.0 : (ROT1 ? nr[0] : rp[-1]);                                            \
        v[18] = cut_p ? 0.0 : (ROT1 ? nr[1] : rp[1]);                                             \
        const double y = apply19(bnd[R], v);                                                      \
        vs = (K1 == CK_SWEEP) ? fma(cp.omega[1] * (rr[R] - y), bnd[R][19], hc) : y;               \
        if (q >= z0 && q < z1) cp.out[(int64_t)pl_of(q) * cp.P + cxy] = vs;                       \
      }                                                                                           \
      if (ROT1 && interior) {                                                                     \
        _Pragma("unroll") for (int e = 0; e < 4; ++e) p1[e] = a1[e];                              \
        _Pragma("unroll") for (int e = 0; e < 8; ++e) a1[e] = nr[e];                              \
      }                                                                                           \
      hm = hc;                                                                                    \
      hc = v0;                                                                                    \
    }                                                                                             \
    if (++bs0 == NB) {                                                                            \
      bs0 = 0;                                                                                    \
      bpar ^= 1u;                                                                                 \
    }                                                                                             \
    ++tau;                                                                                        \
  }

  uint32_t par = 0;   // completion parity of the slots' current round
  for (int tau = tau0; tau < tau_end; par ^= 1u) {
    RK_C19_STEP(0)
    RK_C19_STEP(1)
    RK_C19_STEP(2)
    RK_C19_STEP(3)
    RK_C19_STEP(4)
    RK_C19_STEP(5)
    RK_C19_STEP(6)
    RK_C19_STEP(7)
  }
#undef RK_C19_STEP
}

}  // namespace rk
