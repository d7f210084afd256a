// Two-cells-per-thread variant of the fused chain (included by chain.cu).
//
// Same schedule, shared-memory rings, TMA feed and per-cell arithmetic as
// chain_kernel (so the results are bit-identical), but every thread owns an
// x-pair of cells (2c, 2c+1) of its row: bands, 1/D, rhs and the y
// neighbours of the pair come in 16-byte shared loads, the pair's x
// neighbours are each other's centres plus two 8-byte loads, the ring /
// global stores are 16 bytes, and the pair's own z-column (input at planes
// tau-1, tau; each stage's output at the two previous planes) stays in
// registers, so shared memory only serves the in-plane neighbours.  Per cell this halves the load and integer
// instructions of the one-cell kernel (whose step was issue-latency bound,
// DESIGN.md §7) at half the thread count.  Requires an even halo (NST = 3)
// so that every pair is either interior or halo; x tile offsets are even,
// which keeps all 16-byte accesses aligned.
#pragma once

namespace rk {

// FL bit 0: block-Jacobi cuts may apply (cp.zb > 0 and a local stage);
// bit 1: periodic z.  Launches without them compile the checks out.
template <int ST, int NST, int TX, int TY, int PD, int K0, int K1, int K2, int PH, int FL>
struct ChainStepX2 {
  using G = ChainGeom<ST, NST, TX, TY, PD>;
  static constexpr int EX = G::EX, EY = G::EY, XX = G::XX, SX = G::SX, RPL = EY * EX;

  static __device__ __forceinline__ double2 ld2(const double* p) {
    return *reinterpret_cast<const double2*>(p);
  }
  static __device__ __forceinline__ void st2(double* p, double2 v) {
    *reinterpret_cast<double2*>(p) = v;
  }

  // y = sum_d a_d x_d for the pair, in the one-cell kernel's order: two FMA
  // chains (even / odd d), summed at the end.  Neighbour order of the 7-point
  // canonical layout: 0 centre, 1 -x, 2 +x, 3 -y, 4 +y, 5 -z, 6 +z.
  static __device__ __forceinline__ double2 apply7(const double2 (&a)[ST], double2 c, double l,
                                                   double r, double2 ym, double2 yp, double2 zm,
                                                   double2 zp) {
    const double v0[7] = {c.x, l, c.y, ym.x, yp.x, zm.x, zp.x};
    const double v1[7] = {c.y, c.x, r, ym.y, yp.y, zm.y, zp.y};
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
#pragma unroll
    for (int d = 0; d < ST; ++d) {
      const double ad0 = a[d].x, ad1 = a[d].y;
      if (d % 2 == 0) {
        a0 = fma(ad0, v0[d], a0);
        a1 = fma(ad1, v1[d], a1);
      } else {
        b0 = fma(ad0, v0[d], b0);
        b1 = fma(ad1, v1[d], b1);
      }
    }
    return make_double2(a0 + b0, a1 + b1);
  }

  // stage 0's shared-memory operands of plane tau: the bands / 1/D / rhs go
  // to this phase's registers, the input tile's in-plane neighbours of the
  // pair and the pair at tau+1 (from the next tile) to X0
  struct X0 {
    double l, r;
    double2 ym, yp, xnext;
  };
  static __device__ __forceinline__ X0 load0(const unsigned char* sb, const double* x0, const double* xp,
                                             double2 (&bnd)[3][ST], double2 (&rr)[3], double2 (&inv)[3],
                                             int boff) {
    constexpr bool LOAD_R = (K0 != CK_SPMV1);
    const double* bs = reinterpret_cast<const double*>(sb) + boff;
#pragma unroll
    for (int d = 0; d < ST; ++d) bnd[PH][d] = ld2(bs + d * EY * SX);
    if (RK_CHAIN_TMA_INVD) {
      inv[PH] = ld2(bs + ST * EY * SX);   // 1/D (0 outside the grid: TMA zero fill)
    } else {
      inv[PH].x = bnd[PH][0].x != 0.0 ? 1.0 / bnd[PH][0].x : 0.0;
      inv[PH].y = bnd[PH][0].y != 0.0 ? 1.0 / bnd[PH][0].y : 0.0;
    }
    if (LOAD_R) rr[PH] = ld2(reinterpret_cast<const double*>(sb + G::R_OFF) + boff);
    X0 n;
    n.l = x0[-1];
    n.r = x0[2];
    n.ym = ld2(x0 - XX);
    n.yp = ld2(x0 + XX);
    n.xnext = ld2(xp);
    return n;
  }

  // xc / xm: this thread's input pair at planes tau and tau-1 (registers,
  // z-column reuse); the pair at tau+1 (n.xnext) becomes xc
  static __device__ __forceinline__ double2 compute0(bool st_ok, int pl_tau, double2& xc, double2& xm,
                                                     double* ring, double2 (&bnd)[3][ST], double2 (&rr)[3],
                                                     double2 (&inv)[3], int64_t cxy, int roff,
                                                     const ChainParams& cp, const X0& n) {
    bool cut_m = false, cut_p = false;   // block-Jacobi local sweep (R17)
    if ((FL & 1) && cp.zb > 0 && cp.local[0]) {
      const int g = cp.zg0 + pl_tau;
      cut_m = (g % cp.zb) == 0;
      cut_p = ((g + 1) % cp.zb) == 0;
    }
    const double2 c = xc;
    const double2 zm = cut_m ? make_double2(0.0, 0.0) : xm;
    const double2 zp = cut_p ? make_double2(0.0, 0.0) : n.xnext;
    xm = xc;
    xc = n.xnext;
    const double2 y = apply7(bnd[PH], c, n.l, n.r, n.ym, n.yp, zm, zp);
    double2 val;
    if (K0 == CK_SPMV1) {
      rr[PH] = y;
      val = make_double2((cp.omega[0] * y.x) * inv[PH].x, (cp.omega[0] * y.y) * inv[PH].y);
    } else if (K0 == CK_SWEEP) {
      val = make_double2(fma(cp.omega[0] * (rr[PH].x - y.x), inv[PH].x, c.x),
                         fma(cp.omega[0] * (rr[PH].y - y.y), inv[PH].y, c.y));
    } else {
      val = y;
    }
    if (st_ok) {
      const int64_t nn = (int64_t)pl_tau * cp.P + cxy;
      if (K0 == CK_SPMV1 && cp.out_t) st2(cp.out_t + nn, y);
      if (NST == 1) st2(cp.out + nn, val);
      if (NST == 2 && cp.out_mid) st2(cp.out_mid + nn, val);
    }
    if (NST > 1) st2(ring + PH * RPL + roff, val);
    return val;
  }

  static __device__ __forceinline__ double2 stage0(bool st_ok, int pl_tau, const unsigned char* sb,
                                                   const double* x0, const double* xp,
                                                   double2& xc, double2& xm, double* ring,
                                                   double2 (&bnd)[3][ST], double2 (&rr)[3],
                                                   double2 (&inv)[3], int64_t cxy, int boff,
                                                   int roff, const ChainParams& cp) {
    const X0 n = load0(sb, x0, xp, bnd, rr, inv, boff);
    return compute0(st_ok, pl_tau, xc, xm, ring, bnd, rr, inv, cxy, roff, cp, n);
  }

  // hc / hm: stage S-1's outputs for this thread at planes q and q-1
  // (registers, written in the two previous steps); up: at plane q+1 (this step)
  template <int S>
  static __device__ __forceinline__ double2 stage(bool st_ok, int pl_q, double* ring,
                                                  double2 (&bnd)[3][ST], double2 (&rr)[3],
                                                  double2 (&inv)[3], int64_t cxy, int roff,
                                                  double2 hc, double2 hm, double2 up,
                                                  const ChainParams& cp) {
    static_assert(ST == 7, "single-barrier chain steps need a 7-point stencil");
    constexpr int KIND[3] = {K0, K1, K2};
    constexpr int R = (PH - S + 3) % 3;
    const double* rb = ring + (S - 1) * 3 * RPL + roff;
    const double* r0 = rb + R * RPL;
    bool cut_m = false, cut_p = false;   // block-Jacobi local sweep (R17)
    if ((FL & 1) && cp.zb > 0 && cp.local[S]) {
      const int g = cp.zg0 + pl_q;
      cut_m = (g % cp.zb) == 0;
      cut_p = ((g + 1) % cp.zb) == 0;
    }
    const double2 c = hc;
    const double l = r0[-1], r = r0[2];
    const double2 ym = ld2(r0 - EX), yp = ld2(r0 + EX);
    const double2 zm = cut_m ? make_double2(0.0, 0.0) : hm;
    const double2 zp = cut_p ? make_double2(0.0, 0.0) : up;
    const double2 y = apply7(bnd[R], c, l, r, ym, yp, zm, zp);
    const double2 val = (KIND[S] == CK_SWEEP)
                            ? make_double2(fma(cp.omega[S] * (rr[R].x - y.x), inv[R].x, c.x),
                                           fma(cp.omega[S] * (rr[R].y - y.y), inv[R].y, c.y))
                            : y;
    if (st_ok) {
      const int64_t nq = (int64_t)pl_q * cp.P + cxy;
      if (S == NST - 1) st2(cp.out + nq, val);
      else if (S == NST - 2 && cp.out_mid) st2(cp.out_mid + nq, val);
    }
    if (S < NST - 1) st2(ring + (S * 3 + R) * RPL + roff, val);
    return val;
  }
};

// FL bit 2: several ranks -- the bands of planes outside [0, nz) come from
// the ghost-band map (the neighbours' planes, librk's op->gbands).
template <int ST, int NST, int TX, int TY, int PD, int K0, int K1, int K2, int FL>
__global__ void __launch_bounds__((TX + 2 * (NST - 1)) * (TY + 2 * (NST - 1)) / 2, 1)
chain_kernel_x2(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_r,
                const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_gb,
                ChainParams cp) {
  RK_PDL_ENTRY();
  RK_GATE(cp.gate);
  using G = ChainGeom<ST, NST, TX, TY, PD>;
  constexpr int HALO = G::HALO, EX = G::EX, XX = G::XX, NXB = G::NXB, NB = G::NB;
  constexpr int SX = G::SX, PADB = G::PADB, PADX = G::PADX;
  constexpr bool LOAD_R = (K0 != CK_SPMV1);
  static_assert(HALO % 2 == 0 && EX % 2 == 0 && PADB % 2 == 0 && (1 + PADX) % 2 == 0 && XX % 2 == 0,
                "x-pairs need even offsets");
  extern __shared__ __align__(128) unsigned char smem[];
  double* ring = reinterpret_cast<double*>(smem + G::RING_BASE);   // [NST-1][3][EY][EX]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BAR_BASE);

  const int tx = 2 * (int)threadIdx.x, ty = threadIdx.y;   // first cell of the pair
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nx = cp.nx, ny = cp.ny, nz = cp.nz;
  constexpr bool pz = (FL & 2) != 0;   // periodic z (the host picks FL from cp.pz)
  const int gx0 = (int)blockIdx.x * TX - HALO, gy0 = (int)blockIdx.y * TY - HALO;
  const int gx = gx0 + tx, gy = gy0 + ty;
  // nx even and gx even: both cells of a pair are inside or outside together
  const bool inside = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
  const bool interior = tx >= HALO && tx < HALO + TX && ty >= HALO && ty < HALO + TY;
  const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
  const int z0 = (int)blockIdx.z * cp.zc;
  const int z1 = min(nz, z0 + cp.zc);
  const int tau0 = z0 - HALO;
  const int qfirst = tau0 - 1;
  const int qlast = z1 + HALO;
  // last batch to issue: every issued batch is waited for before the CTA
  // exits (no bulk copy may land in shared memory after it is released)
  const int qiss = RK_CHAIN_XLEAD ? qlast - 1 : qlast;
  const uint32_t tx_bytes = G::B_BYTES + (LOAD_R ? G::R_BYTES : 0) + G::X_BYTES;
  const int xoff = (ty + 1) * XX + tx + 1 + PADX;
  const int boff = ty * SX + tx + PADB;
  const int roff = ty * EX + tx;
  auto pl_of = [&](int q) { return pz ? (q < 0 ? q + nz : (q >= nz ? q - nz : q)) : q; };
  auto xtile = [&](int xs) {
    return reinterpret_cast<const double*>(smem + G::X_BASE + xs * G::XSLOT) + xoff;
  };
  // Batch q (one mbarrier, on the input tile's slot): the bands / rhs of
  // plane q and, with RK_CHAIN_XLEAD, the input tile of plane q + 1 (else of
  // plane q).  Step tau waits for the batch holding tile tau + 1; with the
  // input tile one plane ahead that batch was issued PD steps earlier
  // instead of PD - 1 (the bands of plane tau + 1 are not needed until the
  // next step), so a TMA round trip gets two steps to land.
  auto issue = [&](int q, int xs, int bs) {
    unsigned char* bbase = smem + bs * G::BSLOT;
    unsigned char* xbase = smem + G::X_BASE + xs * G::XSLOT;
    const int pl = pl_of(q);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bars[xs], tx_bytes);
    if ((FL & 4) && (pl < 0 || pl >= nz))
      tma_load_4d(bbase, &map_gb, &bars[xs], gx0 - PADB, gy0, pl < 0 ? pl + BGHOST : pl - nz + BGHOST, 0);
    else
      tma_load_4d(bbase, &map_b, &bars[xs], gx0 - PADB, gy0, pl, 0);
    if (LOAD_R) tma_load_3d(bbase + G::R_OFF, &map_r, &bars[xs], gx0 - PADB, gy0, pl + cp.rz);
    tma_load_3d(xbase, &map_x, &bars[xs], gx0 - 1 - PADX, gy0 - 1,
                (RK_CHAIN_XLEAD ? pl_of(q + 1) : pl) + GHOST);
  };

  if (tid == 0) {
    for (int s = 0; s < NXB; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    if (RK_CHAIN_MIDSYNC) {
      // tiles qfirst and tau0 alone, then batches tau0 .. tau0 + PD - 1 (the
      // bands of qfirst are never used); batch tau0 + PD follows the barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[0], G::X_BYTES);
      tma_load_3d(smem + G::X_BASE, &map_x, &bars[0], gx0 - 1 - PADX, gy0 - 1, pl_of(qfirst) + GHOST);
      mbar_expect_tx(&bars[1], G::X_BYTES);
      tma_load_3d(smem + G::X_BASE + G::XSLOT, &map_x, &bars[1], gx0 - 1 - PADX, gy0 - 1,
                  pl_of(qfirst + 1) + GHOST);
      for (int q = qfirst + 1; q <= min(qfirst + PD, qiss); ++q)
        issue(q, (q + 1 - qfirst) % NXB, (q - qfirst - 1) % NB);
    } else if (RK_CHAIN_XLEAD) {
      // the first tile alone, then batches qfirst .. qfirst + PD
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[0], G::X_BYTES);
      tma_load_3d(smem + G::X_BASE, &map_x, &bars[0], gx0 - 1 - PADX, gy0 - 1, pl_of(qfirst) + GHOST);
      for (int q = qfirst; q <= min(qfirst + PD, qiss); ++q)
        issue(q, (q + 1 - qfirst) % NXB, (q - qfirst) % NB);
    } else {
      for (int q = qfirst; q <= min(qfirst + PD, qlast); ++q) issue(q, (q - qfirst) % NXB, (q - qfirst) % NB);
    }
  }
  mbar_wait(&bars[0], 0);
  if (RK_CHAIN_XLEAD || qfirst + 1 <= qlast) mbar_wait(&bars[1], 0);
  int xsm = 0, xs0 = 1, xsp = 2 % NXB;
  uint32_t parp = 0;
  int bs0 = RK_CHAIN_MIDSYNC ? 0 : 1 % NB;
  int xsi = (PD + 1 + RK_CHAIN_XLEAD) % NXB, bsi = (PD + 1) % NB;
  auto adv = [](int& v, int n) { v = (v + 1 == n) ? 0 : v + 1; };

  double2 bnd[3][ST], rr[3], inv[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    rr[s] = inv[s] = make_double2(0.0, 0.0);
#pragma unroll
    for (int d = 0; d < ST; ++d) bnd[s][d] = make_double2(0.0, 0.0);
  }
  // z-column registers: input pair at planes tau, tau-1 (tiles of slots 1, 0
  // at tau0) and the stage outputs of the two previous steps
  double2 xc = *reinterpret_cast<const double2*>(xtile(1)), xm = *reinterpret_cast<const double2*>(xtile(0));
  if (RK_CHAIN_XLEAD) __syncthreads();   // slot 0 (tile qfirst) is refilled at the first step
  if (RK_CHAIN_MIDSYNC && tid == 0 && tau0 + PD <= qiss)
    issue(tau0 + PD, (tau0 + PD + 1 - qfirst) % NXB, PD % NB);
  const double2 zero2 = make_double2(0.0, 0.0);
  double2 h1c = zero2, h1m = zero2, h2c = zero2, h2m = zero2;
  const int tau_end = z1 + HALO;
#define RK_CHAIN2_STEP(PHV)                                                                        \
  {                                                                                                \
    if (tau >= tau_end) break;                                                                     \
    if (!RK_CHAIN_COMPUTEONLY && tid == 0 && tau + PD <= qiss) issue(tau + PD, xsi, bsi);          \
    if (!RK_CHAIN_COMPUTEONLY && tau + 1 <= qlast) mbar_wait(&bars[xsp], parp);                    \
    using SP = ChainStepX2<ST, NST, TX, TY, PD, K0, K1, K2, PHV, FL>;                                  \
    if (RK_CHAIN_LOADONLY) {                                                                       \
      __syncthreads();                                                                             \
      xsm = xs0;                                                                                   \
      xs0 = xsp;                                                                                   \
      adv(xsp, NXB);                                                                               \
      if (xsp == 0) parp ^= 1u;                                                                    \
      adv(bs0, NB);                                                                                \
      adv(xsi, NXB);                                                                               \
      adv(bsi, NB);                                                                                \
      ++tau;                                                                                       \
      continue;                                                                                    \
    }                                                                                              \
    const double2 v0 = SP::stage0(interior && tau >= z0 && tau < z1 && (pz || tau < nz),          \
                                  pl_of(tau), smem + bs0 * G::BSLOT, xtile(xs0), xtile(xsp), xc,   \
                                  xm, ring, bnd, rr, inv, cxy, boff, roff, cp);                    \
    if constexpr (NST >= 2) {                                                                      \
      double2 v1 = zero2;                                                                          \
      if (tau >= tau0 + 2) {                                                                       \
        const int q = tau - 1;                                                                     \
        v1 = SP::template stage<1>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv,    \
                                   cxy, roff, h1c, h1m, v0, cp);                                   \
      }                                                                                            \
      if constexpr (NST >= 3) {                                                                    \
        if (tau >= tau0 + 4) {                                                                     \
          const int q = tau - 2;                                                                   \
          SP::template stage<2>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv, cxy, \
                                roff, h2c, h2m, v1, cp);                                           \
        }                                                                                          \
        h2m = h2c;                                                                                 \
        h2c = v1;                                                                                  \
      }                                                                                            \
      h1m = h1c;                                                                                   \
      h1c = v0;                                                                                    \
    }                                                                                              \
    __syncthreads();                                                                               \
    xsm = xs0;                                                                                     \
    xs0 = xsp;                                                                                     \
    adv(xsp, NXB);                                                                                 \
    if (xsp == 0) parp ^= 1u;                                                                      \
    adv(bs0, NB);                                                                                  \
    adv(xsi, NXB);                                                                                 \
    adv(bsi, NB);                                                                                  \
    ++tau;                                                                                         \
  }
// RK_CHAIN_MIDSYNC: one barrier per step placed after stage 0's shared-memory
// loads; right after it the slots of plane tau's bands and tile are free and
// batch tau + PD + 1 is issued into them (a TMA lead of ~PD + 1 steps with
// the same slots).  The barrier also orders the previous step's ring writes
// before stages 1-2 read them, and every ring slot written in this step was
// last read two barriers earlier.
#define RK_CHAIN2_STEP_MS(PHV)                                                                     \
  {                                                                                                \
    if (tau >= tau_end) break;                                                                     \
    if (!RK_CHAIN_COMPUTEONLY && tau + 1 <= qlast) mbar_wait(&bars[xsp], parp);                    \
    using SP = ChainStepX2<ST, NST, TX, TY, PD, K0, K1, K2, PHV, FL>;                                  \
    const typename SP::X0 n0 = SP::load0(smem + bs0 * G::BSLOT, xtile(xs0), xtile(xsp), bnd, rr,   \
                                         inv, boff);                                               \
    __syncthreads();                                                                               \
    if (!RK_CHAIN_COMPUTEONLY && tid == 0 && tau + PD + 1 <= qiss) issue(tau + PD + 1, xs0, bs0);  \
    const double2 v0 = SP::compute0(interior && tau >= z0 && tau < z1 && (pz || tau < nz),        \
                                    pl_of(tau), xc, xm, ring, bnd, rr, inv, cxy, roff, cp, n0);    \
    if constexpr (NST >= 2) {                                                                      \
      double2 v1 = zero2;                                                                          \
      if (tau >= tau0 + 2) {                                                                       \
        const int q = tau - 1;                                                                     \
        v1 = SP::template stage<1>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv,    \
                                   cxy, roff, h1c, h1m, v0, cp);                                   \
      }                                                                                            \
      if constexpr (NST >= 3) {                                                                    \
        if (tau >= tau0 + 4) {                                                                     \
          const int q = tau - 2;                                                                   \
          SP::template stage<2>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv, cxy, \
                                roff, h2c, h2m, v1, cp);                                           \
        }                                                                                          \
        h2m = h2c;                                                                                 \
        h2c = v1;                                                                                  \
      }                                                                                            \
      h1m = h1c;                                                                                   \
      h1c = v0;                                                                                    \
    }                                                                                              \
    xs0 = xsp;                                                                                     \
    adv(xsp, NXB);                                                                                 \
    if (xsp == 0) parp ^= 1u;                                                                      \
    adv(bs0, NB);                                                                                  \
    ++tau;                                                                                         \
  }
  if constexpr (RK_CHAIN_MIDSYNC) {
    for (int tau = tau0; tau < tau_end;) {
      RK_CHAIN2_STEP_MS(0)
      RK_CHAIN2_STEP_MS(1)
      RK_CHAIN2_STEP_MS(2)
    }
  } else {
    for (int tau = tau0; tau < tau_end;) {
      RK_CHAIN2_STEP(0)
      RK_CHAIN2_STEP(1)
      RK_CHAIN2_STEP(2)
    }
  }
#undef RK_CHAIN2_STEP_MS
#undef RK_CHAIN2_STEP
}

}  // namespace rk
