// Temporally blocked preconditioned-operator chain (K1 + K2 fused), fed by TMA.
//
// The left-preconditioned operator of rGCROT (t = A v, then the Jacobi(5+1)
// sweeps z <- z + w D^-1 (t - A z)) and the right-
// preconditioned application of rBiCGStab (p_hat = M^-1 p by the sweeps, then
// v = A p_hat) are chains of 6 stencil stages over the SAME bands.  One stage
// per launch streams the S bands from HBM six times (~(S+3) W per stage).
// Here NST consecutive stages run in one launch:
//  * the grid tiles x-y (TX x TY interior + an (NST-1)-cell halo that is
//    recomputed) and chunks z; each CTA marches through its z range;
//  * stage s computes plane tau - s at step tau (a wavefront in z) and keeps
//    the three most recent planes of its output in a shared-memory ring that
//    stage s+1 reads;
//  * thread 0 streams, TWO planes ahead, the band tile, the sweep right-hand
//    side tile and the input tile (+1 halo) of each plane into a shared-memory
//    slot ring with cp.async.bulk.tensor (TMA), completion tracked by one
//    mbarrier per slot; out-of-grid boxes are zero-filled by TMA, which is
//    exactly the zero-ghost semantics of non-periodic boundaries.
// Every band coefficient therefore crosses HBM once per NST stages: ~(S + 4)
// W per launch instead of NST (S + 3) W.  The per-cell arithmetic (FMA order,
// the division by D) is that of stencil_kernel, so the fused and unfused
// paths agree bit for bit.
//
// Scope: 7-point operators whose x and y axes are not periodic (the porous
// configs c1, c3, c5) on one rank; everything else uses the unfused path.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rk_internal.h"

// 1/D: recomputed from the diagonal band (1.0 / D is correctly rounded, so
// the bits equal librk's precomputed 1/D band used by the unfused kernels);
// RK_CHAIN_TMA_INVD = 1 streams that band instead (one more array per plane).
// RK_CHAIN_XLEAD = 1: the x-pair kernel's TMA batches carry the input tile one
// plane ahead of the bands (chain_x2.cuh); 0: the same plane.
// RK_CHAIN_MIDSYNC = 1 (needs RK_CHAIN_XLEAD): the x-pair kernel's barrier sits
// after stage 0's shared-memory loads and the next batch is issued right
// after it, one plane further ahead (chain_x2.cuh).
#ifndef RK_CHAIN_MIDSYNC
#define RK_CHAIN_MIDSYNC 1
#endif
#ifndef RK_CHAIN_XLEAD
#define RK_CHAIN_XLEAD 1
#endif
#if RK_CHAIN_MIDSYNC && !RK_CHAIN_XLEAD
#error "RK_CHAIN_MIDSYNC needs RK_CHAIN_XLEAD (the batches carry the next plane's tile)"
#endif
#ifndef RK_CHAIN_TMA_INVD
#define RK_CHAIN_TMA_INVD 1
#endif
#ifndef RK_C19_ROT
#define RK_C19_ROT 1    // 19-point chain: in-plane neighbourhoods carried in registers (bit 0 stage 0, bit 1 stage 1)
#endif
#ifndef RK_C19_ALLLANES
#define RK_C19_ALLLANES 1   // 19-point chain: stage 0 unconditional in every lane (no branch around the carried registers)
#endif
#ifndef RK_C19_XREG
#define RK_C19_XREG 1   // 19-point chain, folded normalisation: scale input values in registers (1) or the tile in shared memory (0)
#endif
#ifndef RK_C19_INVD
#define RK_C19_INVD 0   // 19-point chain: 1/D recomputed (0) or streamed as a 20th band (1)
#endif
#ifndef RK_CHAIN_COMPUTEONLY
#define RK_CHAIN_COMPUTEONLY 0  // experiments: 1 = no TMA after the prologue (stale data)
#endif
#ifndef RK_CHAIN_LOADONLY
#define RK_CHAIN_LOADONLY 0   // experiments: 1 = TMA traffic only, no stage arithmetic
#endif

namespace rk {

template <int ST>
__host__ __device__ constexpr void coffs(int d, int& dx, int& dy, int& dz) {
  constexpr int DX[19] = {0, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1};
  constexpr int DY[19] = {0, 0, 0, -1, 1, 0, 0, -1, -1, 1, 1, -1, 1, -1, 1, 0, 0, 0, 0};
  constexpr int DZ[19] = {0, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, -1, 1, 1, -1, -1, 1, 1};
  dx = DX[d];
  dy = DY[d];
  dz = DZ[d];
}

// Tile geometry.  TX x TY interior cells per CTA plus an (NST-1)-cell halo
// that is recomputed; PD = TMA prefetch distance in planes (plane tau + PD is
// issued at step tau, so the data of plane tau + 1 -- waited for at step tau
// -- was issued PD - 1 steps earlier).
// TMA box starts must be 16-byte aligned in the innermost (x) dimension, so
// every box starts at an even x and the shared-memory rows carry PAD cells.
// Shared memory: NB = PD + 1 band/rhs buffers (plane q's bands are read into
// registers by stage 0 at step q), NXB = PD + 2 input-tile buffers (plane q's
// tile is read at steps q-1 .. q+1; one mbarrier each, which also carries
// the band/rhs bytes of that plane), and the (NST-1) x 3-plane stage rings.
template <int ST, int NST, int TX, int TY, int PD>
struct ChainGeom {
  static constexpr int HALO = NST - 1;
  static constexpr int EX = TX + 2 * HALO, EY = TY + 2 * HALO;        // stage tile (threads)
  static constexpr int NTHR = EX * EY;
  static constexpr int PADB = HALO % 2;                               // band/rhs box starts at gx0 - PADB
  static constexpr int SX = (EX + PADB + 1) / 2 * 2;                  // band/rhs smem row (even)
  static constexpr int PADX = (HALO + 1) % 2;                         // input box starts at gx0 - 1 - PADX
  static constexpr int XX = (EX + 2 + PADX + 1) / 2 * 2, XY = EY + 2; // input tile (+1 halo)
  static constexpr int NB = PD + 1, NXB = PD + 2;
  static constexpr int NBAND = ST + (RK_CHAIN_TMA_INVD ? 1 : 0);     // bands (+ 1/D)
  static constexpr int B_BYTES = NBAND * EY * SX * 8;
  static constexpr int R_BYTES = EY * SX * 8;
  static constexpr int X_BYTES = XY * XX * 8;
  __host__ __device__ static constexpr int al(int b) { return (b + 127) / 128 * 128; }
  static constexpr int BSLOT = al(B_BYTES) + al(R_BYTES);             // bands + rhs of one plane
  static constexpr int R_OFF = al(B_BYTES);
  static constexpr int XSLOT = al(X_BYTES);
  static constexpr int X_BASE = NB * BSLOT;
  // guard zones around the rings: edge threads of the branch-free stages read
  // one row / column beyond their plane (values nobody uses)
  static constexpr int GUARD = al((EX + 2) * 8);
  static constexpr int RING_BASE = X_BASE + NXB * XSLOT + GUARD;
  static constexpr int RING = (NST > 1 ? NST - 1 : 1) * 3 * EY * EX * 8;
  static constexpr int BAR_BASE = RING_BASE + al(RING) + GUARD;
  static constexpr int SMEM = BAR_BASE + 8 * NXB + 128;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Bounded wait: a TMA that never lands (a descriptor error) traps the kernel
// (a reported launch failure) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0; !mbar_try(b, parity); ++it)
    if (it > (1u << 26)) __trap();
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// One z-step of the chain for loop phase PH = (tau - tau0) mod 3: register
// sets (bands / rhs / 1/D of the planes stages 0..NST-1 work on) and ring
// slots rotate with PH at compile time.  The code is branch-free per cell:
// TMA zero-fills every band and input value outside the grid (x/y) and
// outside [0, nz) (non-periodic z), and the guarded reciprocal 1/D = 0
// there, so such cells evaluate to exactly 0 -- the zero-ghost value --
// without tests.  Threads outside a stage's shrinking valid region compute
// values nobody reads.
template <int ST, int NST, int TX, int TY, int PD, int K0, int K1, int K2, int PH>
struct ChainStep {
  using G = ChainGeom<ST, NST, TX, TY, PD>;
  static constexpr int EX = G::EX, EY = G::EY, XX = G::XX, SX = G::SX, RPL = EY * EX;
  // stage 0 at plane tau: bands / rhs from the band slot `sb`, input
  // neighbours from the x tiles of planes tau-1, tau, tau+1
  static __device__ __forceinline__ double stage0(bool st_ok, int pl_tau, const unsigned char* sb,
                                                  const double* xm, const double* x0,
                                                  const double* xp, double* ring,
                                                  double (&bnd)[3][ST], double (&rr)[3],
                                                  double (&inv)[3], int64_t cxy, int boff, int roff,
                                                  const ChainParams& cp) {
    constexpr bool LOAD_R = (K0 != CK_SPMV1);
    const double* bs = reinterpret_cast<const double*>(sb) + boff;
#pragma unroll
    for (int d = 0; d < ST; ++d) bnd[PH][d] = bs[d * EY * SX];
    if (LOAD_R) rr[PH] = reinterpret_cast<const double*>(sb + G::R_OFF)[boff];
    if (RK_CHAIN_TMA_INVD) inv[PH] = bs[ST * EY * SX];   // 1/D (0 outside the grid: zero fill)
    else inv[PH] = bnd[PH][0] != 0.0 ? 1.0 / bnd[PH][0] : 0.0;
    // block-Jacobi local sweep (R17): no coupling across z-block boundaries
    bool cut_m = false, cut_p = false;
    if (cp.zb > 0 && cp.local[0]) {
      const int g = cp.zg0 + pl_tau;
      cut_m = (g % cp.zb) == 0;
      cut_p = ((g + 1) % cp.zb) == 0;
    }
    double ya = 0.0, yb = 0.0, xc = 0.0;
#pragma unroll
    for (int d = 0; d < ST; ++d) {
      int dx = 0, dy = 0, dz = 0;
      coffs<ST>(d, dx, dy, dz);
      const double* xt = dz < 0 ? xm : (dz > 0 ? xp : x0);
      const double xv = (dz < 0 && cut_m) || (dz > 0 && cut_p) ? 0.0 : xt[dy * XX + dx];
      if (d == 0) xc = xv;
      if (d % 2 == 0) ya = fma(bnd[PH][d], xv, ya);
      else yb = fma(bnd[PH][d], xv, yb);
    }
    const double y = ya + yb;
    double val;
    if (K0 == CK_SPMV1) {
      rr[PH] = y;
      val = (cp.omega[0] * y) * inv[PH];
    } else if (K0 == CK_SWEEP) {
      val = fma(cp.omega[0] * (rr[PH] - y), inv[PH], xc);
    } else {
      val = y;
    }
    if (st_ok) {
      const int64_t n = (int64_t)pl_tau * cp.P + cxy;
      if (K0 == CK_SPMV1 && cp.out_t) cp.out_t[n] = y;
      if (NST == 1) cp.out[n] = val;
      if (NST == 2 && cp.out_mid) cp.out_mid[n] = val;
    }
    if (NST > 1) ring[PH * RPL + roff] = val;
    return val;
  }

  // stage s at plane q = tau - s (register set / ring slot R of plane q).
  // `up` is stage s-1's value at plane q+1 for this thread's own cell,
  // computed earlier in the SAME step; every other input (planes q and q-1)
  // was written to the ring in earlier steps.  A 7-point stencil reaches
  // plane q+1 only through its centre (0,0,+1), so a step needs a single
  // __syncthreads at its end.
  template <int S>
  static __device__ __forceinline__ double stage(bool st_ok, int pl_q, double* ring,
                                                 double (&bnd)[3][ST], double (&rr)[3],
                                                 double (&inv)[3], int64_t cxy, int roff, double up,
                                                 const ChainParams& cp) {
    static_assert(ST == 7, "single-barrier chain steps need a 7-point stencil");
    constexpr int KIND[3] = {K0, K1, K2};
    constexpr int R = (PH - S + 3) % 3;
    const double* rb = ring + (S - 1) * 3 * RPL + roff;
    const double* rm = rb + ((R + 2) % 3) * RPL;
    const double* r0 = rb + R * RPL;
    bool cut_m = false, cut_p = false;       // block-Jacobi local sweep (R17)
    if (cp.zb > 0 && cp.local[S]) {
      const int g = cp.zg0 + pl_q;
      cut_m = (g % cp.zb) == 0;
      cut_p = ((g + 1) % cp.zb) == 0;
    }
    double ya = 0.0, yb = 0.0, zc = 0.0;
#pragma unroll
    for (int d = 0; d < ST; ++d) {
      int dx = 0, dy = 0, dz = 0;
      coffs<ST>(d, dx, dy, dz);
      const double zv = dz > 0 ? (cut_p ? 0.0 : up) : (dz < 0 ? (cut_m ? 0.0 : rm[0]) : r0[dy * EX + dx]);
      if (d == 0) zc = zv;
      if (d % 2 == 0) ya = fma(bnd[R][d], zv, ya);
      else yb = fma(bnd[R][d], zv, yb);
    }
    const double y = ya + yb;
    const double val = (KIND[S] == CK_SWEEP) ? fma(cp.omega[S] * (rr[R] - y), inv[R], zc) : y;
    if (st_ok) {
      const int64_t nq = (int64_t)pl_q * cp.P + cxy;
      if (S == NST - 1) cp.out[nq] = val;
      else if (S == NST - 2 && cp.out_mid) cp.out_mid[nq] = val;
    }
    if (S < NST - 1) ring[(S * 3 + R) * RPL + roff] = val;
    return val;
  }
};

template <int ST, int NST, int TX, int TY, int PD, int K0, int K1, int K2>
__global__ void __launch_bounds__((TX + 2 * (NST - 1)) * (TY + 2 * (NST - 1)), 1)
chain_kernel(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_r,
             const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_gb,
             ChainParams cp) {
  RK_PDL_ENTRY();
  RK_GATE(cp.gate);
  using G = ChainGeom<ST, NST, TX, TY, PD>;
  constexpr int HALO = G::HALO, EX = G::EX, XX = G::XX, NXB = G::NXB, NB = G::NB;
  constexpr int SX = G::SX, PADB = G::PADB, PADX = G::PADX;
  constexpr bool LOAD_R = (K0 != CK_SPMV1);
  extern __shared__ __align__(128) unsigned char smem[];
  double* ring = reinterpret_cast<double*>(smem + G::RING_BASE);   // [NST-1][3][EY][EX]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BAR_BASE);

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * EX + tx;
  const int nx = cp.nx, ny = cp.ny, nz = cp.nz;
  const bool pz = cp.pz != 0;
  const int gx0 = (int)blockIdx.x * TX - HALO, gy0 = (int)blockIdx.y * TY - HALO;
  const int gx = gx0 + tx, gy = gy0 + ty;
  const bool inside = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
  const bool interior = tx >= HALO && tx < HALO + TX && ty >= HALO && ty < HALO + TY;
  const int64_t cxy = inside ? (int64_t)gy * nx + gx : 0;
  const int z0 = (int)blockIdx.z * cp.zc;
  const int z1 = min(nz, z0 + cp.zc);
  const int tau0 = z0 - HALO;
  const int qfirst = tau0 - 1;                  // first plane loaded (stage 0 needs x at tau-1)
  const int qlast = z1 + HALO;                  // last plane loaded (x at tau+1, last step)
  const uint32_t tx_bytes = G::B_BYTES + (LOAD_R ? G::R_BYTES : 0) + G::X_BYTES;
  const int xoff = (ty + 1) * XX + tx + 1 + PADX;    // own cell in an input tile
  const int boff = ty * SX + tx + PADB;              // own cell in a band / rhs tile
  const int roff = ty * EX + tx;                     // own cell in a ring plane
  // planes outside [0, nz) wrap on a periodic z axis (|overhang| <= HALO + 1
  // < nz) and are zero-filled by TMA otherwise
  auto pl_of = [&](int q) { return pz ? (q < 0 ? q + nz : (q >= nz ? q - nz : q)) : q; };
  auto xtile = [&](int xs) {
    return reinterpret_cast<const double*>(smem + G::X_BASE + xs * G::XSLOT) + xoff;
  };

  // thread 0: all bytes of plane q (bands, rhs, input tile) land on the
  // mbarrier of q's input-tile slot xs; the bands / rhs go to band slot bs
  auto issue = [&](int q, int xs, int bs) {
    unsigned char* bbase = smem + bs * G::BSLOT;
    unsigned char* xbase = smem + G::X_BASE + xs * G::XSLOT;
    const int pl = pl_of(q);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bars[xs], tx_bytes);
    if (cp.ghost && (pl < 0 || pl >= nz))   // several ranks: the neighbours' band planes
      tma_load_4d(bbase, &map_gb, &bars[xs], gx0 - PADB, gy0, pl < 0 ? pl + BGHOST : pl - nz + BGHOST, 0);
    else
      tma_load_4d(bbase, &map_b, &bars[xs], gx0 - PADB, gy0, pl, 0);
    if (LOAD_R) tma_load_3d(bbase + G::R_OFF, &map_r, &bars[xs], gx0 - PADB, gy0, pl + cp.rz);
    // the input vector is padded: plane pl lives at z-coordinate pl + GHOST
    tma_load_3d(xbase, &map_x, &bars[xs], gx0 - 1 - PADX, gy0 - 1, pl + GHOST);
  };

  if (tid == 0) {
    for (int s = 0; s < NXB; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // prologue: planes qfirst .. qfirst + PD (step tau0 issues tau0 + PD);
  // plane q uses x slot (q - qfirst) % NXB, band slot (q - qfirst) % NB and
  // barrier parity ((q - qfirst) / NXB) & 1
  if (tid == 0)
    for (int q = qfirst; q <= min(qfirst + PD, qlast); ++q) issue(q, (q - qfirst) % NXB, (q - qfirst) % NB);
  mbar_wait(&bars[0], 0);
  if (qfirst + 1 <= qlast) mbar_wait(&bars[1], 0);
  // running slot state (advanced once per step; no divisions in the loop)
  int xsm = 0, xs0 = 1, xsp = 2 % NXB;          // x slots of planes tau-1, tau, tau+1
  uint32_t parp = 0;                             // barrier parity of plane tau+1
  int bs0 = 1 % NB;                              // band slot of plane tau
  int xsi = (PD + 1) % NXB, bsi = (PD + 1) % NB; // slots of plane tau + PD
  auto adv = [](int& v, int n) { v = (v + 1 == n) ? 0 : v + 1; };

  double bnd[3][ST], rr[3], inv[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    rr[s] = 0.0;
    inv[s] = 0.0;
#pragma unroll
    for (int d = 0; d < ST; ++d) bnd[s][d] = 0.0;
  }
  const int tau_end = z1 + HALO;
#define RK_CHAIN_STEP(PHV)                                                                         \
  {                                                                                                \
    if (tau >= tau_end) break;                                                                     \
    if (!RK_CHAIN_COMPUTEONLY && tid == 0 && tau + PD <= qlast) issue(tau + PD, xsi, bsi);         \
    if (!RK_CHAIN_COMPUTEONLY && tau + 1 <= qlast) mbar_wait(&bars[xsp], parp);                    \
    using SP = ChainStep<ST, NST, TX, TY, PD, K0, K1, K2, PHV>;                                    \
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
    const double v0 = SP::stage0(interior && tau >= z0 && tau < z1 && (pz || tau < nz),           \
                                 pl_of(tau), smem + bs0 * G::BSLOT, xtile(xsm), xtile(xs0),        \
                                 xtile(xsp), ring, bnd, rr, inv, cxy, boff, roff, cp);             \
    if constexpr (NST >= 2) {                                                                      \
      double v1 = 0.0;                                                                             \
      if (tau >= tau0 + 2) {                                                                       \
        const int q = tau - 1;                                                                     \
        v1 = SP::template stage<1>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv,    \
                                   cxy, roff, v0, cp);                                             \
      }                                                                                            \
      if constexpr (NST >= 3) {                                                                    \
        if (tau >= tau0 + 4) {                                                                     \
          const int q = tau - 2;                                                                   \
          SP::template stage<2>(interior && q >= z0 && q < z1, pl_of(q), ring, bnd, rr, inv, cxy, \
                                roff, v1, cp);                                                     \
        }                                                                                          \
      }                                                                                            \
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
  for (int tau = tau0; tau < tau_end;) {
    RK_CHAIN_STEP(0)
    RK_CHAIN_STEP(1)
    RK_CHAIN_STEP(2)
  }
#undef RK_CHAIN_STEP
}

}  // namespace rk

#include "chain_x2.cuh"
#include "chain19.cuh"

namespace rk {

// ------------------------------------------------------------------- host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // resolved once, thread-safely (ranks of an in-process group launch from
  // several host threads)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    RK_REQUIRE(p && q == cudaDriverEntryPointSuccess, RK_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

void encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box) {
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank,
                           const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RK_REQUIRE(r == CUDA_SUCCESS, RK_ECUDA, "cuTensorMapEncodeTiled failed");
}

// z chunks for a one-CTA-per-SM kernel with `tiles` x-y tiles: the chunk
// count c (chunks of >= 16 planes) maximising the wave efficiency
// tiles c / (slots ceil(tiles c / slots)) times the share of steps that are
// not wavefront prologue, zc / (zc + 2 halo + 1).
int pick_chunks(int tiles, int slots, int nzl, int halo) {
  int best = 1;
  double bv = -1.0;
  for (int c = 1; c <= std::max(1, nzl / 16); ++c) {
    const int zc = (nzl + c - 1) / c;
    const int ctas = tiles * ((nzl + zc - 1) / zc);
    const int waves = (ctas + slots - 1) / slots;
    const double v = (double)ctas / ((double)slots * waves) * zc / (zc + 2.0 * halo + 1.0);
    if (v > bv + 1e-9) {
      bv = v;
      best = c;
    }
  }
  return best;
}

// The sweeps' right-hand side: the caller's unpadded vector on one rank;
// on several ranks a padded vector whose ghost planes chain_run filled
// (cp.rz = GHOST: plane pl at z-coordinate pl + GHOST).
void encode_rhs(const rk_op* op, const ChainParams& cp, CUtensorMap* m, cuuint32_t bx, cuuint32_t by) {
  const cuuint64_t nx = op->g.nx, ny = op->g.ny, nz = op->g.nz_local;
  cuuint64_t str[2] = {nx * 8, nx * ny * 8};
  cuuint32_t box[3] = {bx, by, 1};
  if (cp.r && cp.rz) {
    cuuint64_t dims[3] = {nx, ny, nz + 2 * GHOST};
    encode(m, cp.r - GHOST * op->P, 3, dims, str, box);
  } else {
    cuuint64_t dims[3] = {nx, ny, nz};
    encode(m, cp.r ? cp.r : cp.bands, 3, dims, str, box);
  }
}

template <int ST, int NST, int TX, int TY, int PD, int K0, int K1, int K2, int X2>
void launch_one(rk_op* op, ChainParams cp, dim3 grid) {
  using G = ChainGeom<ST, NST, TX, TY, PD>;
  static_assert(G::SMEM <= 232448, "chain tile exceeds 227 KB of shared memory");
  using KernFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          ChainParams);
  using KernFn2 = KernFn;
  KernFn kern = nullptr;
  KernFn2 kern2 = nullptr;
  int fl = 0;   // x-pair kernel flavour: block-Jacobi cuts (1), periodic z (2), ghost bands (4)
  if constexpr (X2 != 0) {
    bool cuts = false;
    for (int s = 0; s < NST; ++s) cuts = cuts || (cp.zb > 0 && cp.local[s]);
    fl = (cuts ? 1 : 0) | (cp.pz ? 2 : 0) | (cp.ghost ? 4 : 0);
    switch (fl) {
      case 0: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 0>; break;
      case 1: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 1>; break;
      case 2: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 2>; break;
      case 3: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 3>; break;
      case 4: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 4>; break;
      default: kern2 = chain_kernel_x2<ST, NST, TX, TY, PD, K0, K1, K2, 5>; break;
    }
  } else {
    kern = chain_kernel<ST, NST, TX, TY, PD, K0, K1, K2>;
  }
  const void* kp = X2 ? (const void*)kern2 : (const void*)kern;
  const int nthr = X2 ? G::NTHR / 2 : G::NTHR;
  // resident CTAs per SM of this instantiation; the shared-memory attribute
  // is per device, so it is set (and the occupancy cached) per context
  int occ = 0;
  {
    auto it = op->ctx->occ_cache.find(kp);
    if (it == op->ctx->occ_cache.end()) {
      RK_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
      RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kp, nthr, G::SMEM));
      occ = std::max(1, occ);
      op->ctx->occ_cache[kp] = occ;
    } else {
      occ = it->second;
    }
  }
  // z chunks (>= 16 planes, to amortise the 2 (NST-1)-plane wavefront
  // prologue) chosen for wave efficiency: 128^3 -> 32 tiles x 4 chunks (one
  // wave of 128 CTAs), 512^3 -> 512 tiles x 2 chunks (6.9 waves of 148)
  const int nzl = (int)op->g.nz_local;
  const int tiles = (int)(grid.x * grid.y);
  const int chunks = pick_chunks(tiles, op->ctx->sms * occ, nzl, NST - 1);
  const int zc = std::max(1, std::min((nzl + chunks - 1) / chunks, nzl));
  cp.zc = zc;
  grid.z = (unsigned)((nzl + zc - 1) / zc);
  const cuuint64_t nx = op->g.nx, ny = op->g.ny, nz = op->g.nz_local;
  CUtensorMap mb, mr, mx, mg;
  {
    cuuint64_t dims[4] = {nx, ny, nz, (cuuint64_t)G::NBAND};       // bands (then 1/D)
    cuuint64_t str[3] = {nx * 8, nx * ny * 8, (cuuint64_t)op->N * 8};
    cuuint32_t box[4] = {(cuuint32_t)G::SX, (cuuint32_t)G::EY, 1, (cuuint32_t)G::NBAND};
    encode(&mb, cp.bands, 4, dims, str, box);
    if (cp.ghost) {   // the neighbours' band planes (op->gbands)
      cuuint64_t gd[4] = {nx, ny, 2 * BGHOST, (cuuint64_t)G::NBAND};
      cuuint64_t gs[3] = {nx * 8, nx * ny * 8, (cuuint64_t)(2 * BGHOST) * nx * ny * 8};
      encode(&mg, op->gbands, 4, gd, gs, box);
    } else {
      mg = mb;
    }
  }
  encode_rhs(op, cp, &mr, (cuuint32_t)G::SX, (cuuint32_t)G::EY);
  {
    cuuint64_t dims[3] = {nx, ny, nz + 2 * GHOST};         // padded: GHOST ghost planes each side
    cuuint64_t str[2] = {nx * 8, nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)G::XX, (cuuint32_t)G::XY, 1};
    encode(&mx, cp.xin - GHOST * op->P, 3, dims, str, box);
  }
  dim3 blk(X2 ? G::EX / 2 : G::EX, G::EY);
  // PDL lets the next grid's CTAs become resident early; next to the chain
  // (one 200 KB-smem CTA per SM) that measured 9 % slower at c3, so by
  // default neither the chain nor its successor overlaps (RK_PDL_MODE)
  rk_ctx* ctx = op->ctx;
  // mode 0: chain and successor overlap; 1: chain does not; 2: neither;
  // 3: the chain overlaps its predecessor, its successor does not
  const bool allow = ctx->pdl && (ctx->pdl_mode == 0 || ctx->pdl_mode == 3) && !ctx->pdl_skip_next;
  ctx->pdl_skip_next = ctx->pdl_mode >= 2;
  launch_pdl_if(ctx, allow, X2 ? kern2 : kern, grid, blk, G::SMEM, mb, mr, mx, mg, cp);
}

template <int NST, int TX, int TY, int PD, int X2 = 0>
void chain_dispatch(rk_op* op, const int* k, const ChainParams& cp, dim3 grid) {
  if constexpr (NST == 3) {
    if (k[0] == CK_SPMV1 && k[1] == CK_SWEEP && k[2] == CK_SWEEP)
      return launch_one<7, 3, TX, TY, PD, CK_SPMV1, CK_SWEEP, CK_SWEEP, X2>(op, cp, grid);
    if (k[0] == CK_SWEEP && k[1] == CK_SWEEP && k[2] == CK_SWEEP)
      return launch_one<7, 3, TX, TY, PD, CK_SWEEP, CK_SWEEP, CK_SWEEP, X2>(op, cp, grid);
    if (k[0] == CK_SWEEP && k[1] == CK_SWEEP && k[2] == CK_SPMV)
      return launch_one<7, 3, TX, TY, PD, CK_SWEEP, CK_SWEEP, CK_SPMV, X2>(op, cp, grid);
  } else if constexpr (NST == 2) {
    if (k[0] == CK_SPMV1 && k[1] == CK_SWEEP)
      return launch_one<7, 2, TX, TY, PD, CK_SPMV1, CK_SWEEP, 0, X2>(op, cp, grid);
    if (k[0] == CK_SWEEP && k[1] == CK_SWEEP)
      return launch_one<7, 2, TX, TY, PD, CK_SWEEP, CK_SWEEP, 0, X2>(op, cp, grid);
    if (k[0] == CK_SWEEP && k[1] == CK_SPMV)
      return launch_one<7, 2, TX, TY, PD, CK_SWEEP, CK_SPMV, 0, X2>(op, cp, grid);
  } else {
    if (k[0] == CK_SPMV1) return launch_one<7, 1, TX, TY, PD, CK_SPMV1, 0, 0, X2>(op, cp, grid);
    if (k[0] == CK_SWEEP) return launch_one<7, 1, TX, TY, PD, CK_SWEEP, 0, 0, X2>(op, cp, grid);
    return launch_one<7, 1, TX, TY, PD, CK_SPMV, 0, 0, X2>(op, cp, grid);
  }
  throw Error(RK_EINVAL, "unsupported chain stage combination");
}

// Tile configurations (interior TX x TY, prefetch distance PD).  RK_CHAIN_CFG
// (read per launch; experiments only) selects one by index.  Measured at
// 128^3 / 256^3 (scripts/micro/chain_bench.cu, r01): 32x16 pd2 is fastest;
// smaller tiles (more CTAs per SM, deeper prefetch) lose to their larger
// recomputed halo.
struct TileCfg {
  int tx, ty, pd;
};
constexpr TileCfg CFGS[] = {{32, 16, 2}, {32, 8, 2}, {16, 8, 2}, {16, 8, 3}, {16, 16, 2}, {32, 16, 2}};
constexpr int NCFG = sizeof(CFGS) / sizeof(CFGS[0]);
constexpr int DEFAULT_CFG = 5;   // x-pairs with register z-columns (chain_x2.cuh)

int cfg_index() {
  const char* e = std::getenv("RK_CHAIN_CFG");
  const int i = e ? std::atoi(e) : DEFAULT_CFG;
  return (i >= 0 && i < NCFG) ? i : DEFAULT_CFG;
}

template <int NST>
void chain_dispatch_cfg(int ci, rk_op* op, const int* k, const ChainParams& cp, dim3 grid) {
  switch (ci) {
    case 0: return chain_dispatch<NST, 32, 16, 2>(op, k, cp, grid);
    case 1: return chain_dispatch<NST, 32, 8, 2>(op, k, cp, grid);
    case 2: return chain_dispatch<NST, 16, 8, 2>(op, k, cp, grid);
    case 3: return chain_dispatch<NST, 16, 8, 3>(op, k, cp, grid);
    case 4: return chain_dispatch<NST, 16, 16, 2>(op, k, cp, grid);
    default:   // x-pairs (chain_x2.cuh); needs an even halo
      if constexpr (NST == 3) return chain_dispatch<NST, 32, 16, 2, 1>(op, k, cp, grid);
      else return chain_dispatch<NST, 32, 16, 2>(op, k, cp, grid);
  }
}

// ------------------------------------------------------- 19-point chain
// Tile of the 19-point chain (chain19.cuh): 32 x TY19 interior cells, TMA
// prefetch distance PD19.
constexpr int TY19 = 8, PD19 = 2, NST19 = 2;

template <int NST, int TX, int TY, int PD, int K0, int K1, int K2>
void launch19(rk_op* op, ChainParams cp) {
  using G = C19Geom<NST, TX, TY, PD>;
  static_assert(G::SMEM <= 232448, "19-point chain tile exceeds 227 KB of shared memory");
  using KernFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          ChainParams);
  bool cuts = false;
  for (int s = 0; s < NST; ++s) cuts = cuts || (cp.zb > 0 && cp.local[s]);
  const int fl = (cuts ? 1 : 0) | (cp.pz ? 2 : 0) | (cp.ghost ? 4 : 0);
  KernFn kern;
  switch (fl) {
    case 0: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 0>; break;
    case 1: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 1>; break;
    case 2: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 2>; break;
    case 3: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 3>; break;
    case 4: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 4>; break;
    default: kern = chain19_kernel<NST, TX, TY, PD, K0, K1, K2, 5>; break;
  }
  rk_ctx* ctx = op->ctx;
  int occ = 0;
  {
    auto it = ctx->occ_cache.find((const void*)kern);
    if (it == ctx->occ_cache.end()) {
      RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
      RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NTHR, G::SMEM));
      occ = std::max(1, occ);
      ctx->occ_cache[(const void*)kern] = occ;
    } else {
      occ = it->second;
    }
  }
  const int nzl = (int)op->g.nz_local;
  dim3 grid((unsigned)(op->g.nx / TX), (unsigned)(op->g.ny / TY), 1);
  const int chunks = pick_chunks((int)(grid.x * grid.y), ctx->sms * occ, nzl, G::H);
  const int zc = (nzl + chunks - 1) / chunks;
  cp.zc = zc;
  grid.z = (unsigned)((nzl + zc - 1) / zc);
  const cuuint64_t nx = op->g.nx, ny = op->g.ny, nz = op->g.nz_local;
  CUtensorMap mbM, mbH, mrM, mrH, mxM, mxH, mgM, mgH;
  {
    cuuint64_t dims[4] = {nx, ny, nz, (cuuint64_t)G::NBT};
    cuuint64_t str[3] = {nx * 8, nx * ny * 8, (cuuint64_t)op->N * 8};
    cuuint32_t boxM[4] = {(cuuint32_t)TX, (cuuint32_t)G::EY, 1, (cuuint32_t)G::NBT};
    cuuint32_t boxH[4] = {(cuuint32_t)G::HW, (cuuint32_t)G::EY, 1, (cuuint32_t)G::NBT};
    encode(&mbM, cp.bands, 4, dims, str, boxM);
    encode(&mbH, cp.bands, 4, dims, str, boxH);
    if (cp.ghost) {   // the neighbours' band planes (op->gbands)
      cuuint64_t gd[4] = {nx, ny, 2 * BGHOST, (cuuint64_t)G::NBT};
      cuuint64_t gs[3] = {nx * 8, nx * ny * 8, (cuuint64_t)(2 * BGHOST) * nx * ny * 8};
      encode(&mgM, op->gbands, 4, gd, gs, boxM);
      encode(&mgH, op->gbands, 4, gd, gs, boxH);
    } else {
      mgM = mbM;
      mgH = mbH;
    }
  }
  encode_rhs(op, cp, &mrM, (cuuint32_t)TX, (cuuint32_t)G::EY);
  encode_rhs(op, cp, &mrH, (cuuint32_t)G::HW, (cuuint32_t)G::EY);
  {
    cuuint64_t dims[3] = {nx, ny, nz + 2 * GHOST};   // padded: GHOST ghost planes each side
    cuuint64_t str[2] = {nx * 8, nx * ny * 8};
    cuuint32_t boxM[3] = {(cuuint32_t)TX, (cuuint32_t)G::XROWS, 1};
    cuuint32_t boxH[3] = {(cuuint32_t)G::HW, (cuuint32_t)G::XROWS, 1};
    encode(&mxM, cp.xin - GHOST * op->P, 3, dims, str, boxM);
    encode(&mxH, cp.xin - GHOST * op->P, 3, dims, str, boxH);
  }
  const bool allow = ctx->pdl && (ctx->pdl_mode == 0 || ctx->pdl_mode == 3) && !ctx->pdl_skip_next;
  ctx->pdl_skip_next = ctx->pdl_mode >= 2;
  launch_pdl_if(ctx, allow, kern, grid, dim3(G::NTHR), G::SMEM, mbM, mbH, mrM, mrH, mxM, mxH, mgM, mgH,
                cp);
}

void chain19_dispatch(rk_op* op, int nst, const int* k, const ChainParams& cp) {
  constexpr int TX = 32, TY = TY19, PD = PD19;
  if (nst == 2) {
    if (k[0] == CK_SPMV1 && k[1] == CK_SWEEP) return launch19<2, TX, TY, PD, CK_SPMV1, CK_SWEEP, 0>(op, cp);
    if (k[0] == CK_SWEEP && k[1] == CK_SWEEP) return launch19<2, TX, TY, PD, CK_SWEEP, CK_SWEEP, 0>(op, cp);
    if (k[0] == CK_SWEEP && k[1] == CK_SPMV) return launch19<2, TX, TY, PD, CK_SWEEP, CK_SPMV, 0>(op, cp);
  } else if (nst == 1) {
    if (k[0] == CK_SPMV1) return launch19<1, TX, TY, PD, CK_SPMV1, 0, 0>(op, cp);
    if (k[0] == CK_SWEEP) return launch19<1, TX, TY, PD, CK_SWEEP, 0, 0>(op, cp);
    return launch19<1, TX, TY, PD, CK_SPMV, 0, 0>(op, cp);
  }
  throw Error(RK_EINVAL, "unsupported 19-point chain stage combination");
}

}  // namespace

int chain_max_stages(const rk_op* op) {
  if (op->no_chain) return 0;
  // several ranks: the chain input's NST-deep halo comes from one exchange
  // per launch (chain_run), the bands' from op->gbands
  if (op->ctx->nranks != 1 && (op->gbands == nullptr || op->g.nz_local < 16)) return 0;
  if (op->S == 19) {
    // chain19.cuh: x-region boxes wrap a periodic x axis; y must not be periodic
    if (op->g.periodic_mask & 2) return 0;
    if (op->g.nx % 32 != 0 || op->g.ny % TY19 != 0 || op->g.nz_local < 16) return 0;
    if (!op->force_chain && (double)(op->S + 3) * 8.0 * (double)op->N <= (double)op->ctx->l2_bytes)
      return 0;
    return NST19;
  }
  if (op->S != 7) return 0;
  if (op->g.periodic_mask & 3) return 0;                    // TMA boxes do not wrap in x/y
  const TileCfg tc = CFGS[cfg_index()];
  if (op->g.nx % tc.tx != 0 || op->g.ny % tc.ty != 0 || op->g.nx % 2 != 0) return 0;
  if (op->g.nz_local < 16) return 0;
  // While the bands and the sweep vectors fit in L2 the one-stage-per-launch
  // path re-reads them from L2, not HBM, and wins (64^3: 46 vs 63 us per
  // M^-1); the chain pays off once a stage's traffic exceeds L2.
  if (!op->force_chain && (double)(op->S + 3) * 8.0 * (double)op->N <= (double)op->ctx->l2_bytes)
    return 0;
  return 3;
}

void chain_launch(rk_op* op, int nst, const int* kinds, const double* omegas, const double* xin,
                  const double* r, double* out_t, double* out_mid, double* out, const int* local,
                  int zb, const XScale* xs) {
  rk_ctx* ctx = op->ctx;
  const int ci = cfg_index();
  const TileCfg tc = CFGS[ci];
  ChainParams cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.bands = op->bands;
  cp.N = op->N;
  cp.P = op->P;
  cp.nx = (int)op->g.nx;
  cp.ny = (int)op->g.ny;
  cp.nz = (int)op->g.nz_local;
  cp.px = (op->S == 19 && (op->g.periodic_mask & 1)) ? 1 : 0;   // only the 19-point kernel wraps x
  cp.py = 0;
  cp.pz = op->wrapz;   // periodic z on one rank wraps in the kernel; on several, halos
  cp.ghost = op->ctx->nranks > 1 ? 1 : 0;
  cp.rz = op->ctx->nranks > 1 ? GHOST : 0;
  cp.xin = xin;
  cp.r = r;
  cp.out_t = out_t;
  cp.out_mid = out_mid;
  cp.out = out;
  for (int s = 0; s < nst; ++s) cp.omega[s] = omegas[s];
  cp.zb = zb;
  cp.zg0 = (int)op->g.z0;
  cp.gate = ctx->gate;
  for (int s = 0; s < nst; ++s) cp.local[s] = local ? local[s] : 0;
  if (xs) {
    RK_REQUIRE(op->S == 19 && kinds[0] == CK_SPMV1 && xs->n2 && xs->out, RK_EINVAL,
               "input normalisation needs the 19-point chain with stage 0 = A v");
    cp.xs_n2 = xs->n2;
    cp.xs_in2 = xs->in2;
    cp.xs_out = xs->out;
    cp.xs_flag = xs->flag;
  }
  dim3 grid((unsigned)(op->g.nx / tc.tx), (unsigned)(op->g.ny / tc.ty), 1);   // z: launch_one
  // algorithmic bytes: bands once + stage-0 input + rhs (if any) + outputs (the
  // 1/D array is an implementation choice -- flops for bytes -- and not counted)
  const double words = op->S + 1 + ((kinds[0] != CK_SPMV1) ? 1 : 0) + 1 + (out_t ? 1 : 0) +
                       (out_mid ? 1 : 0) + (xs ? 1 : 0);
  Launch L(ctx, op->S == 19 ? "chain19" : "chain", 8.0 * op->N * words);
  if (op->S == 19) chain19_dispatch(op, nst, kinds, cp);
  else if (nst == 3) chain_dispatch_cfg<3>(ci, op, kinds, cp, grid);
  else if (nst == 2) chain_dispatch_cfg<2>(ci, op, kinds, cp, grid);
  else chain_dispatch_cfg<1>(ci, op, kinds, cp, grid);
  L.done();
}

bool chain_scales_input(const rk_op* op) { return op->S == 19 && chain_max_stages(op) > 0; }

void chain_run(rk_op* op, const std::vector<int>& kinds, const std::vector<double>& om,
               const double* xin, const double* r, double* out_t, double* out_mid, double* out,
               double* za, double* zb, const std::vector<int>& local, int zbs, const XScale* xs) {
  const int n = (int)kinds.size();
  // TMA tensor maps need 16-byte aligned bases and the x-pair stores 16-byte
  // aligned outputs; a caller's misaligned vector (rk_precond_apply accepts
  // any pointer) takes the unfused path, which handles any alignment
  auto al16 = [](const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; };
  const bool aligned = al16(xin - GHOST * op->P) && al16(r) && al16(out_t) && al16(out_mid) && al16(out);
  const int nmax = aligned ? chain_max_stages(op) : 0;
  RK_REQUIRE(!xs || (nmax > 0 && op->S == 19 && kinds[0] == CK_SPMV1 && al16(xs->out)), RK_EINVAL,
             "input normalisation needs the fused 19-point chain");
  std::vector<int> loc(n, 0);
  for (int q = 0; q < n && q < (int)local.size(); ++q) loc[q] = local[q];
  double* bufs[2] = {za, zb};
  if (xin == za) std::swap(bufs[0], bufs[1]);
  const double* rhs = kinds[0] == CK_SPMV1 ? out_t : r;
  if (nmax == 0) {
    const double* cur = xin;
    for (int q = 0; q < n; ++q) {
      double* dst = (q == n - 1) ? out : ((q == n - 2 && out_mid) ? out_mid : bufs[q % 2]);
      if (kinds[q] == CK_SPMV1) stencil(op, SM_SPMV_SWEEP1, cur, nullptr, out_t, dst, om[q], nullptr);
      else if (kinds[q] == CK_SWEEP)
        stencil(op, SM_SWEEP, cur, rhs, dst, nullptr, om[q], nullptr, loc[q] ? zbs : 0);
      else stencil(op, SM_SPMV, cur, nullptr, dst, nullptr, 0.0, nullptr);
      cur = dst;
    }
    return;
  }
  const int g = (n + nmax - 1) / nmax;
  const double* cur = xin;
  int a = 0;
  int rhs_depth = 0;   // ghost planes of rhs already exchanged in this call (it does not change
                       // after the launch that produces it)
  for (int i = 0; i < g; ++i) {
    const int len = n / g + (i < n % g ? 1 : 0);
    const bool last = (i == g - 1);
    double* dst = last ? out : bufs[i % 2];
    // several ranks: the launch reads its input len planes and the sweeps'
    // right-hand side len - 1 planes beyond the slab (stage 0 recomputes the
    // halo planes the later stages need)
    // (input and right-hand-side halos of one launch in one collective launch)
    comm_group_begin(op->ctx);
    halo(op, cur, len);
    if (kinds[a] != CK_SPMV1 && rhs && len - 1 > rhs_depth) {
      halo(op, rhs, len - 1);
      rhs_depth = len - 1;
    }
    comm_group_end(op->ctx);
    chain_launch(op, len, kinds.data() + a, om.data() + a, cur, rhs,
                 (kinds[a] == CK_SPMV1) ? out_t : nullptr, last ? out_mid : nullptr, dst,
                 loc.data() + a, zbs, i == 0 ? xs : nullptr);
    cur = dst;
    a += len;
  }
}

}  // namespace rk
