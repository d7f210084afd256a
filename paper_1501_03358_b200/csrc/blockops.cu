// sm_100a block kernels of librk: K3 block dot, K4 block update, normalise,
// K5 linear combinations, projection, K8 rotation (tall-skinny, HBM-bound).
#include "kcommon.cuh"

namespace rk {


// ----------------------------------------------------------------- K3
// g_c = Q_c^T w for c < ncol (block dot, "[C V_j]^T w").  NC accumulators
// per thread; every column is streamed once, w once.
template <int NC, int VEC>
__global__ void __launch_bounds__(256) bdot_kernel(ColPtrs Q, int ncol, const double* __restrict__ w,
                                                   int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
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
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
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

// ------------------------------------------------ K3 / K4, tiled (VEC = 2)
// Column-chunk order: a CTA owns a tile of TILE = 512 RV rows; each thread
// holds its RV double2 of w in registers and streams the columns through
// the tile G at a time (G x RV independent 16-byte loads in flight).  Every
// warp reads 512-byte runs of one column at a time, which keeps DRAM pages
// open far better than interleaving all columns per row (measured at c3:
// 4.8 -> 7.0 TB/s for the block dot, 5.4 -> 6.8 TB/s for the update;
// scripts/micro/bdot_bench.cu).  The rows past the last whole tile are
// handled by a row-interleaved tail loop.  Columns are padded to a
// multiple of GRP by the host (duplicate pointers: surplus dot accumulators
// are never stored, surplus update coefficients are 0), so every group is
// loaded whole -- one basic block per group keeps all G x RV loads in flight
// ahead of the FMAs (a remainder branch let the compiler sink them).
constexpr int TRV = 2, TG = 4, TILE_ROWS = 512 * TRV;

#ifndef RK_BDOT_RV
#define RK_BDOT_RV 4
#define RK_BDOT_G 2
#endif
constexpr int DRV = RK_BDOT_RV, DG = RK_BDOT_G;

template <int NC, int BT>
__global__ void __launch_bounds__(BT) bdot_tile_kernel(ColPtrs Q, int ncol, const double* __restrict__ w,
                                                        int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  constexpr int RV = DRV, G = DG, TILE_ROWS = 2 * BT * DRV;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int64_t ntile = N / TILE_ROWS;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = t * TILE_ROWS + 2 * threadIdx.x;
    double2 wv[RV];
#pragma unroll
    for (int v = 0; v < RV; ++v) wv[v] = __ldg(reinterpret_cast<const double2*>(w + r0 + 2 * BT * v));
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double2 q[G][RV];
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const Vec<2> a = ldv_stream<2>(Q.p[c + u] + r0 + 2 * BT * v);
            q[u][v] = make_double2(a.v[0], a.v[1]);
          }
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            acc[c + u] = fma(q[u][v].x, wv[v].x, acc[c + u]);
            acc[c + u] = fma(q[u][v].y, wv[v].y, acc[c + u]);
          }
      }
    }
  }
  // tail rows (N even: VEC = 2 is only chosen for even N)
  for (int64_t r = ntile * TILE_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    const Vec<2> wv = ldv_ro<2>(w + r);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < ncol) {
        const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
        acc[c] = fma(a.v[0], wv.v[0], acc[c]);
        acc[c] = fma(a.v[1], wv.v[1], acc[c]);
      }
  }
  block_reduce_store<NC>(acc, ncol, ra);
}

// Bulk-copy-fed variant of bdot_tile_kernel (same column-chunk order and
// summation order per thread, one CTA per SM): the w rows and column chunks
// of a CTA's 2048-row tiles stream through a ring of BS shared-memory slots
// of 16 KB filled by 1-D cp.async.bulk, so the bytes in flight per SM are set
// by the ring (128 KB), not by the register budget that caps the tile
// kernel at 2 CTAs/SM (read-only streaming needs ~128 KB in flight per SM to
// reach the HBM ceiling; scripts/micro/read_bw.cu).
namespace {
__device__ __forceinline__ uint32_t bk_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ bool bk_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bk_smem(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
}  // namespace

constexpr int BK_ROWS = 2048, BK_SLOTS = 8, BK_BYTES = BK_ROWS * 8;
// columns per two-right-hand-side bulk launch (2 x 40 accumulators per thread
// at one CTA per SM; wider [C V_j] is split into balanced launches, each
// re-reading w and v)
#ifndef RK_BK_MAXC2
#define RK_BK_MAXC2 40
#endif
constexpr int BK_MAXC2 = RK_BK_MAXC2;
constexpr size_t BK_SMEM = (size_t)BK_SLOTS * BK_BYTES + BK_SLOTS * sizeof(uint64_t);
// ring slots of the bulk block update (read-modify-write of w)
#ifndef RK_BU_SLOTS
#define RK_BU_SLOTS 8
#endif
constexpr int BU_SLOTS = RK_BU_SLOTS;
constexpr size_t BU_SMEM = (size_t)BU_SLOTS * BK_BYTES + BU_SLOTS * sizeof(uint64_t);

// NR = 1: Q^T w; NR = 2: [Q^T w, Q^T v] (values NC.. for v, as bdot2_tile_kernel)
template <int NC, int NR>
__global__ void __launch_bounds__(256, 1) bdot_bulk_kernel(ColPtrs Q, int ncol, const double* __restrict__ w,
                                                           const double* __restrict__ v, int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  extern __shared__ __align__(128) unsigned char bk_sm[];
  double2* ring = reinterpret_cast<double2*>(bk_sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(bk_sm + (size_t)BK_SLOTS * BK_BYTES);
  constexpr int RV = BK_ROWS / 512;   // double2 per thread per tile
  double acc[NR * NC];
#pragma unroll
  for (int c = 0; c < NR * NC; ++c) acc[c] = 0.0;
  const int64_t ntile = N / BK_ROWS;
  const int64_t mytiles = ntile > blockIdx.x ? (ntile - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int per = ncol + NR;                        // items per tile: w (, v), Q_0 .. Q_{ncol-1}
  const int64_t nitem = mytiles * per;
  // items in order: per tile (blockIdx.x, + gridDim.x, ...) w (, v), then
  // Q_0 .. Q_{ncol-1}; thread 0 walks them with a cursor (no division on the
  // issue path, which sits between two barriers)
  int ic = -NR;
  int64_t irow = (int64_t)blockIdx.x * BK_ROWS;
  auto issue = [&](int64_t, int slot) {
    const double* src = (ic < 0 ? (ic + NR == 0 ? w : v) : Q.p[ic]) + irow;
    if (++ic == ncol) {
      ic = -NR;
      irow += (int64_t)gridDim.x * BK_ROWS;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bk_smem(bar + slot)),
                 "r"(BK_BYTES)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            bk_smem(ring + (size_t)slot * (BK_ROWS / 2))),
        "l"(src), "r"(BK_BYTES), "r"(bk_smem(bar + slot))
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < BK_SLOTS; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bk_smem(bar + q)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < BK_SLOTS && q < nitem; ++q) issue(q, q);
  }
  __syncthreads();
  int slot = 0;
  uint32_t phase = 0;
  int64_t it = 0;
  // consume item `it` in `slot`; refill the slot with item it + BK_SLOTS
  auto next = [&]() {
    __syncthreads();   // every thread is done with the slot
    if (threadIdx.x == 0 && it + BK_SLOTS < nitem) issue(it + BK_SLOTS, slot);
    ++it;
    if (++slot == BK_SLOTS) {
      slot = 0;
      phase ^= 1;
    }
  };
#pragma unroll 1
  for (int64_t lt = 0; lt < mytiles; ++lt) {
    double2 wv[NR][RV];
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      while (!bk_try(bar + slot, phase)) {
      }
      const double2* sl = ring + (size_t)slot * (BK_ROWS / 2);
#pragma unroll
      for (int u = 0; u < RV; ++u) wv[h][u] = sl[threadIdx.x + 256 * u];
      next();
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c < ncol) {
        while (!bk_try(bar + slot, phase)) {
        }
        const double2* qs = ring + (size_t)slot * (BK_ROWS / 2);
#pragma unroll
        for (int u = 0; u < RV; ++u) {
          const double2 q = qs[threadIdx.x + 256 * u];
#pragma unroll
          for (int h = 0; h < NR; ++h) {
            acc[h * NC + c] = fma(q.x, wv[h][u].x, acc[h * NC + c]);
            acc[h * NC + c] = fma(q.y, wv[h][u].y, acc[h * NC + c]);
          }
        }
        next();
      }
    }
  }
  // tail rows (N even)
  for (int64_t r = ntile * BK_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    Vec<2> wt[NR];
    wt[0] = ldv_ro<2>(w + r);
    if (NR == 2) wt[NR - 1] = ldv_ro<2>(v + r);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < ncol) {
        const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          acc[h * NC + c] = fma(a.v[0], wt[h].v[0], acc[h * NC + c]);
          acc[h * NC + c] = fma(a.v[1], wt[h].v[1], acc[h * NC + c]);
        }
      }
  }
  block_reduce_store<NR * NC>(acc, NR == 1 ? ncol : NR * NC, ra);
}

// Two right-hand sides: [Q^T w, Q^T v] in one read of Q (the Gram-corrected
// CGS2 of reading R19 needs Q_j^T v_j, the lagged Gram row of the newest basis
// vector, next to the projection coefficients Q_j^T w).  Values 0..NC-1 go to
// out (w), NC.. to out2 (v); only the first ncol of each are stored.
template <int NC>
__global__ void __launch_bounds__(256) bdot2_tile_kernel(ColPtrs Q, int ncol, const double* __restrict__ w,
                                                         const double* __restrict__ v, int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  constexpr int RV = 2, G = 2, BT = 256, TILE_ROWS = 2 * BT * RV;
  double acc[2 * NC];
#pragma unroll
  for (int c = 0; c < 2 * NC; ++c) acc[c] = 0.0;
  const int64_t ntile = N / TILE_ROWS;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = t * TILE_ROWS + 2 * threadIdx.x;
    double2 wv[RV], vv[RV];
#pragma unroll
    for (int u = 0; u < RV; ++u) {
      wv[u] = __ldg(reinterpret_cast<const double2*>(w + r0 + 2 * BT * u));
      vv[u] = __ldg(reinterpret_cast<const double2*>(v + r0 + 2 * BT * u));
    }
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double2 q[G][RV];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int u = 0; u < RV; ++u) {
            const Vec<2> a = ldv_stream<2>(Q.p[c + g] + r0 + 2 * BT * u);
            q[g][u] = make_double2(a.v[0], a.v[1]);
          }
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int u = 0; u < RV; ++u) {
            acc[c + g] = fma(q[g][u].x, wv[u].x, acc[c + g]);
            acc[c + g] = fma(q[g][u].y, wv[u].y, acc[c + g]);
            acc[NC + c + g] = fma(q[g][u].x, vv[u].x, acc[NC + c + g]);
            acc[NC + c + g] = fma(q[g][u].y, vv[u].y, acc[NC + c + g]);
          }
      }
    }
  }
  for (int64_t r = ntile * TILE_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    const Vec<2> wv = ldv_ro<2>(w + r), vv = ldv_ro<2>(v + r);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < ncol) {
        const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
        acc[c] = fma(a.v[0], wv.v[0], acc[c]);
        acc[c] = fma(a.v[1], wv.v[1], acc[c]);
        acc[NC + c] = fma(a.v[0], vv.v[0], acc[NC + c]);
        acc[NC + c] = fma(a.v[1], vv.v[1], acc[NC + c]);
      }
  }
  block_reduce_store<2 * NC>(acc, 2 * NC, ra);
}

// The Gram-corrected CGS2 update (reading R19): every CTA forms, in shared
// memory, h = 2 g - G g from the projection coefficients g = Q^T w and the
// Gram matrix G = Q^T Q of the basis Q = [C, v_0 .. v_j] (C-block = I; the
// rows of v_0 .. v_j are the lagged dots grow[k + i][0 .. k + i], row stride
// MAXCOL), then streams w <- w - Q h (+ ||w||^2) like bupd_tile_kernel.
// CTA 0 stores h (the Hessenberg / B column) to hout.
template <int NC>
__global__ void __launch_bounds__(256) bupd_gram_kernel(ColPtrs Q, int ncol, int k, const double* __restrict__ g,
                                                        const double* __restrict__ grow, double* __restrict__ hout,
                                                        double* __restrict__ w, int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  constexpr int RV = TRV, G = TG;
  __shared__ double gs[NC], hs[NC];
  for (int c = threadIdx.x; c < NC; c += blockDim.x) gs[c] = c < ncol ? g[c] : 0.0;
  __syncthreads();
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    double h = 0.0;
    if (c < ncol) {
      double gg = 0.0;
      for (int l = 0; l < ncol; ++l) {
        double Gcl;
        if (c < k && l < k) Gcl = (c == l) ? 1.0 : 0.0;
        else if (c >= l) Gcl = grow[(int64_t)c * MAXCOL + l];
        else Gcl = grow[(int64_t)l * MAXCOL + c];
        gg = fma(Gcl, gs[l], gg);
      }
      h = 2.0 * gs[c] - gg;
    }
    hs[c] = h;
    if (blockIdx.x == 0 && c < ncol) hout[c] = h;
  }
  __syncthreads();
  const volatile double* hv = hs;
  double acc[1] = {0.0};
  const int64_t ntile = N / TILE_ROWS;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = t * TILE_ROWS + 2 * threadIdx.x;
    double2 wv[RV];
#pragma unroll
    for (int u = 0; u < RV; ++u) wv[u] = *reinterpret_cast<const double2*>(w + r0 + 512 * u);
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double hc[G];
#pragma unroll
        for (int u = 0; u < G; ++u) hc[u] = hv[c + u];
        double2 q[G][RV];
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int vv = 0; vv < RV; ++vv) {
            const Vec<2> a = ldv_stream<2>(Q.p[c + u] + r0 + 512 * vv);
            q[u][vv] = make_double2(a.v[0], a.v[1]);
          }
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int vv = 0; vv < RV; ++vv) {
            wv[vv].x = fma(-hc[u], q[u][vv].x, wv[vv].x);
            wv[vv].y = fma(-hc[u], q[u][vv].y, wv[vv].y);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < RV; ++u) {
      *reinterpret_cast<double2*>(w + r0 + 512 * u) = wv[u];
      acc[0] = fma(wv[u].x, wv[u].x, acc[0]);
      acc[0] = fma(wv[u].y, wv[u].y, acc[0]);
    }
  }
  for (int64_t r = ntile * TILE_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    double2 wn = *reinterpret_cast<const double2*>(w + r);
#pragma unroll 1
    for (int c = 0; c < ncol; ++c) {
      const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
      wn.x = fma(-hs[c], a.v[0], wn.x);
      wn.y = fma(-hs[c], a.v[1], wn.y);
    }
    *reinterpret_cast<double2*>(w + r) = wn;
    acc[0] = fma(wn.x, wn.x, acc[0]);
    acc[0] = fma(wn.y, wn.y, acc[0]);
  }
  block_reduce_store<1>(acc, 1, ra);
}

// Bulk-copy-fed form of bupd_gram_kernel for large N (one CTA per SM): the
// w rows and the column chunks of the CTA's 2048-row tiles stream through
// the bdot_bulk ring (8 x 16 KB, cp.async.bulk + mbarrier), the h prologue
// runs while the first items are in flight, and the new w rows are stored
// from registers.  Every element's update w - h_0 q_0 - h_1 q_1 - ... is
// the tile kernel's FMA chain in the same column order (bit-identical w and
// h); only ||w||^2 is summed in another order.  grow == nullptr: a plain
// block update with h = gs g (the recycle projection r -= C xi, x += U xi);
// hout nullable; ra.out == nullptr: no ||w||^2.
__global__ void __launch_bounds__(256, 1) bupd_gram_bulk_kernel(ColPtrs Q, int ncol, int k,
                                                                const double* __restrict__ g,
                                                                const double* __restrict__ grow,
                                                                double gs_scale,
                                                                double* __restrict__ hout, double* w,
                                                                int64_t N, RedArgs ra) {
  RK_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char bk_sm[];
  double2* ring = reinterpret_cast<double2*>(bk_sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(bk_sm + (size_t)BU_SLOTS * BK_BYTES);
  __shared__ double gs[MAXCOL], hs[MAXCOL];
  constexpr int RV = BK_ROWS / 512;
  const int64_t ntile = N / BK_ROWS;
  const int64_t mytiles = ntile > blockIdx.x ? (ntile - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int per = ncol + 1;   // items per tile: w, Q_0 .. Q_{ncol-1}
  const int64_t nitem = mytiles * per;
  int ic = -1;
  int64_t irow = (int64_t)blockIdx.x * BK_ROWS;
  auto issue = [&](int slot) {
    const double* src = (ic < 0 ? w : Q.p[ic]) + irow;
    if (++ic == ncol) {
      ic = -1;
      irow += (int64_t)gridDim.x * BK_ROWS;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bk_smem(bar + slot)),
                 "r"(BK_BYTES)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            bk_smem(ring + (size_t)slot * (BK_ROWS / 2))),
        "l"(src), "r"(BK_BYTES), "r"(bk_smem(bar + slot))
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < BU_SLOTS; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bk_smem(bar + q)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < BU_SLOTS && q < nitem; ++q) issue(q);
  }
  // h = 2 g - G g (bupd_gram_kernel's prologue, same FMA order)
  for (int c = threadIdx.x; c < MAXCOL; c += blockDim.x) gs[c] = c < ncol ? g[c] : 0.0;
  __syncthreads();
  for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
    double h;
    if (grow) {
      double gg = 0.0;
      for (int l = 0; l < ncol; ++l) {
        double Gcl;
        if (c < k && l < k) Gcl = (c == l) ? 1.0 : 0.0;
        else if (c >= l) Gcl = grow[(int64_t)c * MAXCOL + l];
        else Gcl = grow[(int64_t)l * MAXCOL + c];
        gg = fma(Gcl, gs[l], gg);
      }
      h = 2.0 * gs[c] - gg;
    } else {
      h = gs_scale * gs[c];
    }
    hs[c] = h;
    if (hout && blockIdx.x == 0) hout[c] = h;
  }
  __syncthreads();
  int slot = 0;
  uint32_t phase = 0;
  int64_t it = 0;
  auto next = [&]() {
    __syncthreads();   // every thread is done with the slot
    if (threadIdx.x == 0 && it + BU_SLOTS < nitem) issue(slot);
    ++it;
    if (++slot == BU_SLOTS) {
      slot = 0;
      phase ^= 1;
    }
  };
  double acc[1] = {0.0};
  int64_t row0 = (int64_t)blockIdx.x * BK_ROWS;
#pragma unroll 1
  for (int64_t lt = 0; lt < mytiles; ++lt, row0 += (int64_t)gridDim.x * BK_ROWS) {
    double2 wv[RV];
    while (!bk_try(bar + slot, phase)) {
    }
    {
      const double2* sl = ring + (size_t)slot * (BK_ROWS / 2);
#pragma unroll
      for (int u = 0; u < RV; ++u) wv[u] = sl[threadIdx.x + 256 * u];
    }
    next();
#pragma unroll 1
    for (int c = 0; c < ncol; ++c) {
      const double hc = hs[c];
      while (!bk_try(bar + slot, phase)) {
      }
      const double2* qs = ring + (size_t)slot * (BK_ROWS / 2);
#pragma unroll
      for (int u = 0; u < RV; ++u) {
        const double2 q = qs[threadIdx.x + 256 * u];
        wv[u].x = fma(-hc, q.x, wv[u].x);
        wv[u].y = fma(-hc, q.y, wv[u].y);
      }
      next();
    }
#pragma unroll
    for (int u = 0; u < RV; ++u) {
      *reinterpret_cast<double2*>(w + row0 + 2 * (threadIdx.x + 256 * u)) = wv[u];
      acc[0] = fma(wv[u].x, wv[u].x, acc[0]);
      acc[0] = fma(wv[u].y, wv[u].y, acc[0]);
    }
  }
  for (int64_t r = ntile * BK_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    double2 wn = *reinterpret_cast<const double2*>(w + r);
#pragma unroll 1
    for (int c = 0; c < ncol; ++c) {
      const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
      wn.x = fma(-hs[c], a.v[0], wn.x);
      wn.y = fma(-hs[c], a.v[1], wn.y);
    }
    *reinterpret_cast<double2*>(w + r) = wn;
    acc[0] = fma(wn.x, wn.x, acc[0]);
    acc[0] = fma(wn.y, wn.y, acc[0]);
  }
  if (ra.out) block_reduce_store<1>(acc, 1, ra);
}

// gsh[c] = gs g_c with g_c the deferred block-dot sums; CTA 0 stores g_c
template <int NC>
__device__ __forceinline__ void coef_from_partials(const CoefIn& cin, int ncol, double gs, double* gsh) {
  block_sum_partials<NC>(cin.part, cin.G, ncol, gsh);
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    if (c < ncol && blockIdx.x == 0) cin.store[c] = gsh[c];
    gsh[c] = c < ncol ? gs * gsh[c] : 0.0;
  }
}

template <int NC, int ND>
__global__ void __launch_bounds__(256) bupd_tile_kernel(ColPtrs Q, int ncol, const double* __restrict__ g,
                                                        double gs, double* __restrict__ w, int64_t N,
                                                        const double* d0, const double* d1,
                                                        const double* d2, RedArgs ra, CoefIn cin) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  constexpr int RV = TRV, G = TG;
  __shared__ double gsh[NC];
  if (cin.part) {
    coef_from_partials<NC>(cin, ncol, gs, gsh);
  } else {
    for (int c = threadIdx.x; c < NC; c += blockDim.x) gsh[c] = c < ncol ? gs * g[c] : 0.0;
  }
  __syncthreads();
  // volatile: re-read per group instead of hoisting NC coefficients into
  // registers for the whole tile loop (which cost occupancy)
  const volatile double* gshv = gsh;
  double acc[ND > 0 ? ND : 1];
#pragma unroll
  for (int q = 0; q < (ND > 0 ? ND : 1); ++q) acc[q] = 0.0;
  const double* dv[3] = {d0, d1, d2};
  auto dots = [&](const double* row, const double2& wn) {
#pragma unroll
    for (int q = 0; q < ND; ++q) {
      double2 o = wn;
      if (dv[q]) {
        const Vec<2> a = ldv_ro<2>(dv[q] + (row - w));
        o = make_double2(a.v[0], a.v[1]);
      }
      acc[q] = fma(o.x, wn.x, acc[q]);
      acc[q] = fma(o.y, wn.y, acc[q]);
    }
  };
  const int64_t ntile = N / TILE_ROWS;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = t * TILE_ROWS + 2 * threadIdx.x;
    double2 wv[RV];
#pragma unroll
    for (int v = 0; v < RV; ++v) wv[v] = *reinterpret_cast<const double2*>(w + r0 + 512 * v);
    // padded columns (host duplicates, coefficient 0) are loaded whole
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double gc[G];
#pragma unroll
        for (int u = 0; u < G; ++u) gc[u] = gshv[c + u];
        double2 q[G][RV];
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const Vec<2> a = ldv_stream<2>(Q.p[c + u] + r0 + 512 * v);
            q[u][v] = make_double2(a.v[0], a.v[1]);
          }
#pragma unroll
        for (int u = 0; u < G; ++u) {
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            wv[v].x = fma(-gc[u], q[u][v].x, wv[v].x);
            wv[v].y = fma(-gc[u], q[u][v].y, wv[v].y);
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      *reinterpret_cast<double2*>(w + r0 + 512 * v) = wv[v];
      dots(w + r0 + 512 * v, wv[v]);
    }
  }
  for (int64_t r = ntile * TILE_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < N;
       r += 2 * (int64_t)gridDim.x * blockDim.x) {
    double2 wn = *reinterpret_cast<const double2*>(w + r);
#pragma unroll 1
    for (int c = 0; c < ncol; ++c) {   // rolled: keeps the tail out of the register budget
      const Vec<2> a = ldv_stream<2>(Q.p[c] + r);
      wn.x = fma(-gsh[c], a.v[0], wn.x);
      wn.y = fma(-gsh[c], a.v[1], wn.y);
    }
    *reinterpret_cast<double2*>(w + r) = wn;
    dots(w + r, wn);
  }
  if constexpr (ND > 0) block_reduce_store<(ND > 0 ? ND : 1)>(acc, ND, ra);
}

// rBiCGStab lines 7a + 8 fused (one rank, reading R20): the block dot before
// this kernel produced the per-CTA partials of [C, r~]^T v (k + 1 values);
// every CTA sums them (eta = C^T v, r~^T v), forms
//   sigma = r~^T v - (C^T r~)^T eta  (= r~^T (v - C eta); ctr = C^T r~ is
//   computed once per solve) and alpha = rho / sigma,
// then streams v <- v - C eta (bupd_tile_kernel's order and FMAs) and, with
// the new v rows still in registers, bicg_s: s = r - alpha v, z = w_l s / D,
// ||s||^2.  CTA 0 stores eta and sigma.
template <int NC>
__global__ void __launch_bounds__(256) bproj_s_kernel(ColPtrs Q, int k, double* __restrict__ v, int64_t N,
                                                      CoefIn cin, const double* __restrict__ ctr,
                                                      const double* __restrict__ r, double* __restrict__ s,
                                                      double* __restrict__ z, const double* __restrict__ D,
                                                      double wl, BiIter* cur, RedArgs ra) {
  RK_PDL_ENTRY();
  RK_GATE(ra.gate);
  constexpr int RV = TRV, G = TG;
  __shared__ double gsh[NC];
  __shared__ double sig_alpha[2];
  block_sum_partials<NC>(cin.part, cin.G, k + 1, gsh);
  if (threadIdx.x == 0) {
    double corr = 0.0;
    for (int c = 0; c < k; ++c) corr = fma(ctr[c], gsh[c], corr);
    const double sigma = gsh[k] - corr;
    sig_alpha[0] = sigma;
    sig_alpha[1] = cur->rho / sigma;
    if (blockIdx.x == 0) cur->sigma = sigma;
  }
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < k; c += blockDim.x) cin.store[c] = gsh[c];
  __syncthreads();
  if (threadIdx.x == 0) gsh[k] = 0.0;   // r~ is not an update column
  for (int c = k + 1 + threadIdx.x; c < NC; c += blockDim.x) gsh[c] = 0.0;
  __syncthreads();
  const double alpha = sig_alpha[1];
  const volatile double* gshv = gsh;
  double acc[1] = {0.0};
  auto epi = [&](int64_t n, const double2& vn) {
    const double2 rn = *reinterpret_cast<const double2*>(r + n);
    double2 sn, zn;
    sn.x = rn.x - alpha * vn.x;
    sn.y = rn.y - alpha * vn.y;
    acc[0] = fma(sn.x, sn.x, acc[0]);
    acc[0] = fma(sn.y, sn.y, acc[0]);
    zn = sn;
    if (D) {
      const Vec<2> dn = ldv_stream<2>(D + n);
      zn.x = (wl * sn.x) * dn.v[0];
      zn.y = (wl * sn.y) * dn.v[1];
    }
    *reinterpret_cast<double2*>(s + n) = sn;
    *reinterpret_cast<double2*>(z + n) = zn;
  };
  const int64_t ntile = N / TILE_ROWS;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = t * TILE_ROWS + 2 * threadIdx.x;
    double2 wv[RV];
#pragma unroll
    for (int u = 0; u < RV; ++u) wv[u] = *reinterpret_cast<const double2*>(v + r0 + 512 * u);
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < k) {
        double gc[G];
#pragma unroll
        for (int u = 0; u < G; ++u) gc[u] = gshv[c + u];
        double2 q[G][RV];
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int vv = 0; vv < RV; ++vv) {
            const Vec<2> a = ldv_stream<2>(Q.p[c + u] + r0 + 512 * vv);
            q[u][vv] = make_double2(a.v[0], a.v[1]);
          }
#pragma unroll
        for (int u = 0; u < G; ++u) {
#pragma unroll
          for (int vv = 0; vv < RV; ++vv) {
            wv[vv].x = fma(-gc[u], q[u][vv].x, wv[vv].x);
            wv[vv].y = fma(-gc[u], q[u][vv].y, wv[vv].y);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RV; ++u) {
      *reinterpret_cast<double2*>(v + r0 + 512 * u) = wv[u];
      epi(r0 + 512 * u, wv[u]);
    }
  }
  for (int64_t n = ntile * TILE_ROWS + 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); n < N;
       n += 2 * (int64_t)gridDim.x * blockDim.x) {
    double2 wn = *reinterpret_cast<const double2*>(v + n);
#pragma unroll 1
    for (int c = 0; c < k; ++c) {
      const Vec<2> a = ldv_stream<2>(Q.p[c] + n);
      wn.x = fma(-gsh[c], a.v[0], wn.x);
      wn.y = fma(-gsh[c], a.v[1], wn.y);
    }
    *reinterpret_cast<double2*>(v + n) = wn;
    epi(n, wn);
  }
  block_reduce_store<1>(acc, 1, ra);
}

// v_{j+1} = w / h_{j+1,j} (as w * (1 / h)), with the happy-breakdown test
// h <= 1e-14 ||A_hat v_j|| (reading D18): on breakdown v_{j+1} = 0 and *flag = 1.
template <int VEC>
__global__ void __launch_bounds__(256) normalize_kernel(double* __restrict__ w, int64_t N,
                                                        const double* nrm2, const double* nin2,
                                                        double* flag) {
  RK_PDL_ENTRY();
  // four grid-stride elements per thread in flight (the one-load loop kept
  // ~32 KB per SM in flight: 5.0 TB/s at c4); the first four are loaded
  // before the norm arrives
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Vec<VEC> v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (e + u * stride < NE) v[u] = ldv<VEC>(w + (e + u * stride) * VEC);
  const double h = sqrt(*nrm2);
  bool brk = false;
  if (nin2) brk = !(h > 1e-14 * sqrt(*nin2));
  // v = w * (1 / h): one division per thread (the fused chain19 launch that
  // folds line 10 in applies the same product, so both paths store the same v)
  const double inv = brk ? 0.0 : 1.0 / h;
  for (; e < NE; e += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e + u * stride < NE) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) v[u].v[t] = v[u].v[t] * inv;
        stv<VEC>(w + (e + u * stride) * VEC, v[u]);
      }
    }
    const int64_t en = e + U * stride;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (en + u * stride < NE) v[u] = ldv<VEC>(w + (en + u * stride) * VEC);
  }
  if (flag && blockIdx.x == 0 && threadIdx.x == 0) *flag = brk ? 1.0 : 0.0;
}

// ----------------------------------------------------------------- K5
// out_o = scale_o * sum_c Q_c coef[o][c]  (+ out_o if acc_o), o < nout.
template <int NC, int VEC>
__global__ void __launch_bounds__(256) lincomb_kernel(ColPtrs Q, int ncol, const double* __restrict__ coef,
                                                      int nout, LcOut lo, int64_t N) {
  RK_PDL_ENTRY();
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
  RK_PDL_ENTRY();
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
__global__ void __launch_bounds__(256) rotate_kernel(ColPtrs Qc, int k, int kout, const double* __restrict__ T,
                                                     int64_t N) {
  RK_PDL_ENTRY();
  __shared__ double ts[NC * NC];
  for (int t = threadIdx.x; t < k * kout; t += blockDim.x) ts[t] = T[t];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += stride) {
    double in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < k) in[c] = Qc.p[c][n];
#pragma unroll
    for (int o = 0; o < NC; ++o) {
      if (o < kout) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c < k) s = fma(in[c], ts[o * k + c], s);
        const_cast<double*>(Qc.p[o])[n] = s;
      }
    }
  }
}


// The same rotation with T in the kernel's parameter space (constant bank,
// up to 18 KB of parameters: CUDA >= 12.1 on sm_70+): every T entry is a
// compile-time operand of its FMA -- the shared-memory form spent one LDS per
// FMA (1.5 TB/s at c4, k = 31); stride NC (t[o * NC + c] = T(c, o)); the
// same FMA order as rotate_kernel (bit-identical).
template <int NC>
struct TMat {
  double t[NC * NC];
};
template <int NC, int VEC>
__global__ void __launch_bounds__(256) rotate_cb_kernel(ColPtrs Qc, int k, int kout,
                                                        const __grid_constant__ TMat<NC> T, int64_t N) {
  RK_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NE = N / VEC;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NE; e += stride) {
    const int64_t n = e * VEC;
    // columns c >= k are column 0 again with T(c, o) = 0 (host padding): the
    // FMA chain needs no per-term predicate (x * 0 adds an exact zero)
    Vec<VEC> in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = ldv<VEC>(Qc.p[c] + n);
#pragma unroll
    for (int o = 0; o < NC; ++o) {
      if (o < kout) {
        Vec<VEC> s;
#pragma unroll
        for (int t = 0; t < VEC; ++t) s.v[t] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int t = 0; t < VEC; ++t) s.v[t] = fma(in[c].v[t], T.t[o * NC + c], s.v[t]);
        stv<VEC>(const_cast<double*>(Qc.p[o]) + n, s);
      }
    }
  }
}

// =================================================================== host
namespace {
// one CTA per SM (the ring fills the shared memory), grid = #SMs
template <typename... KArgs, typename... Args>
int launch_bulk_smem(rk_ctx* ctx, size_t smem, void (*kern)(KArgs...), Args&&... args) {
  auto it = ctx->occ_cache.find((const void*)kern);
  if (it == ctx->occ_cache.end()) {
    RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ctx->occ_cache[(const void*)kern] = 1;
  }
  launch_pdl(ctx, kern, dim3(ctx->sms), dim3(256), smem, std::forward<Args>(args)...);
  return ctx->sms;
}
template <typename... KArgs, typename... Args>
int launch_bulk(rk_ctx* ctx, void (*kern)(KArgs...), Args&&... args) {
  return launch_bulk_smem(ctx, BK_SMEM, kern, std::forward<Args>(args)...);
}
}  // namespace
// One block-dot launch over <= 40 columns; returns its grid (the number of
// per-CTA partials of every value).
static int bdot_launch(rk_ctx* ctx, const std::vector<const double*>& cols, const double* w,
                       int64_t N, RedArgs ra) {
  const int ncol = (int)cols.size();
  const int nc = nc_round(ncol);
  const int vec = pick_vec(N, {w}, cols);
  ColPtrs Q = make_cols_padded(cols, nc);
  const int64_t work = N / vec;
  // bulk-copy path: 16-byte aligned columns and even N (vec == 2), a tile per
  // SM, >= 4 columns (measured at N = 2^21: equal to the register-tile
  // kernel at 20 columns, -5 % at 8, -17 % at 40; slower for 1-2 columns)
  const bool bulk = vec == 2 && (ctx->bdot_bulk == 2 ||
                                 (ctx->bdot_bulk == 1 && ncol >= 4 && N >= (int64_t)BK_ROWS * ctx->sms));
  int grid = 0;
#define RK_BDOT(NCV)                                                                          \
  if (bulk)                                                                                         \
    grid = launch_bulk(ctx, bdot_bulk_kernel<NCV, 1>, Q, ncol, w, (const double*)nullptr, N, ra);   \
  else if (vec == 2)                                                                                \
    grid = launch_k(ctx, bdot_tile_kernel<NCV, 256>, work / DRV, dim3(256), Q, ncol, w, N, ra);     \
  else grid = launch_k(ctx, bdot_kernel<NCV, 1>, work, dim3(256), Q, ncol, w, N, ra);
  switch (nc) {
    case 8: RK_BDOT(8); break;
    case 16: RK_BDOT(16); break;
    case 24: RK_BDOT(24); break;
    case 32: RK_BDOT(32); break;
    default: RK_BDOT(40); break;
  }
#undef RK_BDOT
  return grid;
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
    Launch L(ctx, "bdot", 8.0 * N * (ncol + 1));
    bdot_launch(ctx, cols, w, N, red_args(ctx, out + off));
    L.done();
  }
  allreduce(ctx, out, total);   // one collective for all column chunks
}

void bproject(rk_ctx* ctx, const std::vector<const double*>& cols, double* w, int64_t N,
              double* eta, const std::vector<const double*>& dots, double* red_out, bool reduce) {
  const int ncol = (int)cols.size();
  const int nd = (int)dots.size();
  const bool defer = ctx->defer_coef && ctx->nranks == 1 && ncol >= 1 && ncol <= 40 && nd <= 3 &&
                     pick_vec(N, {w, nd > 0 ? dots[0] : nullptr, nd > 1 ? dots[1] : nullptr,
                                  nd > 2 ? dots[2] : nullptr}, cols) == 2;
  if (!defer) {
    bdot(ctx, cols, w, N, eta);
    bupd(ctx, cols, eta, 1.0, w, N, dots, red_out, CoefIn{}, reduce);
    return;
  }
  RedArgs ra = red_args(ctx, nullptr);
  ra.partials = ctx->dpartials;
  ra.defer = 1;
  Launch L(ctx, "bdot", 8.0 * N * (ncol + 1));
  CoefIn cin;
  cin.G = bdot_launch(ctx, cols, w, N, ra);
  L.done();
  cin.part = ctx->dpartials;
  cin.store = eta;
  bupd(ctx, cols, eta, 1.0, w, N, dots, red_out, cin, reduce);
}

bool bicg_proj_s(rk_op* op, const std::vector<const double*>& C, double* v, const double* rtl,
                 const double* ctr, double* eta, const double* r, double* s, double* z, double wl,
                 bool jacobi, BiIter* cur, double* stage) {
  rk_ctx* ctx = op->ctx;
  const int64_t N = op->N;
  const int k = (int)C.size();
  const double* D = jacobi ? op->invd() : nullptr;
  const bool one = ctx->nranks == 1;
  if ((one && !ctx->defer_coef) || k < 1 || k + 1 > 40 || pick_vec(N, {v, rtl, r, s, z, D}, C) != 2)
    return false;
  std::vector<const double*> cols(C);
  cols.push_back(rtl);
  CoefIn cin;
  cin.store = eta;
  if (one) {   // deferred: bproj_s sums the block dot's per-CTA partials
    RedArgs ra = red_args(ctx, nullptr);
    ra.partials = ctx->dpartials;
    ra.defer = 1;
    Launch L(ctx, "bdot", 8.0 * N * (k + 2));
    cin.G = bdot_launch(ctx, cols, v, N, ra);
    L.done();
    cin.part = ctx->dpartials;
  } else {     // finalised, one all-reduce of [C^T v, r~^T v], read as G = 1 partials
    Launch L(ctx, "bdot", 8.0 * N * (k + 2));
    bdot_launch(ctx, cols, v, N, red_args(ctx, stage));
    L.done();
    allreduce(ctx, stage, k + 1);
    cin.part = stage;
    cin.G = 1;
  }
  const int nc = nc_round(k + 1);
  ColPtrs Q = make_cols_padded(C, nc_round(k));
  RedArgs rs = red_args(ctx, &cur->ss);
  Launch L2(ctx, "bupd", 8.0 * N * (k + 2 + 3 + (jacobi ? 1 : 0)));
  switch (nc) {
#define RK_BPS(NCV)                                                                                  \
  case NCV:                                                                                          \
    launch_k(ctx, bproj_s_kernel<NCV>, N / (2 * TRV), dim3(256), Q, k, v, N, cin, ctr, r, s, z, D, wl, \
             cur, rs);                                                                               \
    break;
    RK_BPS(8)
    RK_BPS(16)
    RK_BPS(24)
    RK_BPS(32)
    default: RK_BPS(40)
#undef RK_BPS
  }
  L2.done();
  return true;
}

void bupd(rk_ctx* ctx, const std::vector<const double*>& cols, const double* g, double gscale,
          double* w, int64_t N, const std::vector<const double*>& dots, double* red_out,
          CoefIn cin, bool reduce) {
  const int ncol = (int)cols.size();
  const int nd = (int)dots.size();
  RK_REQUIRE(nd <= 3, RK_EINVAL, "bupd: at most 3 dots");
  RK_REQUIRE(ncol <= MAXCOL, RK_EINVAL, "too many columns in a block product");
  const int nc = nc_round(ncol);
  const int vec = pick_vec(N, {w, nd > 0 ? dots[0] : nullptr, nd > 1 ? dots[1] : nullptr,
                               nd > 2 ? dots[2] : nullptr}, cols);
  RedArgs ra = nd ? red_args(ctx, red_out) : RedArgs{nullptr, nullptr, nullptr};
  ra.gate = ctx->gate;
  RK_REQUIRE(!cin.part || (vec == 2 && nc <= 40), RK_ESTATE, "deferred coefficients need the tiled update");
  ColPtrs Q = make_cols_padded(cols, nc);
  const double* d[3] = {nullptr, nullptr, nullptr};
  for (int q = 0; q < nd; ++q) d[q] = dots[q];
  double words = ncol + 2;
  for (int q = 0; q < nd; ++q) words += dots[q] ? 1 : 0;
  const int64_t work = N / vec;
  Launch L(ctx, "bupd", 8.0 * N * words);
#define RK_BUPD(NCV, NDV)                                                                      \
  if (vec == 2)                                                                                \
    launch_k(ctx, bupd_tile_kernel<NCV, NDV>, work / TRV, dim3(256), Q, ncol, g, gscale, w, N,  \
             d[0], d[1], d[2], ra, cin);                                                       \
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
  if (nd && reduce) allreduce(ctx, red_out, nd);
}

void bdot2(rk_ctx* ctx, const std::vector<const double*>& cols_all, const double* w, const double* v,
           int64_t N, double* out_w, double* out_v) {
  const int total = (int)cols_all.size();
  RK_REQUIRE(total <= MAXCOL + 1, RK_EINVAL, "too many columns in a block product");
  const bool tiled = pick_vec(N, {w, v}, cols_all) == 2;
  if (!tiled) {   // odd sizes / misaligned: two single-RHS block dots
    bdot(ctx, cols_all, w, N, out_w);
    bdot(ctx, cols_all, v, N, out_v);
    return;
  }
  // bulk-copy path: launches of up to BK_MAXC2 columns, balanced (71
  // columns: 2 x 36; each launch re-reads w and v, 2 W), else <= 24 columns
  // per tiled launch
  if (ctx->bdot_bulk == 2 ||
      (ctx->bdot_bulk == 1 && total >= 4 && N >= (int64_t)BK_ROWS * ctx->sms)) {
    const int nch = (total + BK_MAXC2 - 1) / BK_MAXC2;
    const int per = (total + nch - 1) / nch;
    for (int off = 0; off < total; off += per) {
      const int ncol = std::min(per, total - off);
      std::vector<const double*> cols(cols_all.begin() + off, cols_all.begin() + off + ncol);
      const int nc = nc_round(ncol);
      RedArgs ra = red_args(ctx, out_w + off);
      ra.out2 = out_v + off;
      ra.split = nc;
      ra.valid = ncol;
      ColPtrs Q = make_cols_padded(cols, nc);
      Launch L(ctx, "bdot", 8.0 * N * (ncol + 2));
      switch (nc) {
        case 8: launch_bulk(ctx, bdot_bulk_kernel<8, 2>, Q, ncol, w, v, N, ra); break;
        case 16: launch_bulk(ctx, bdot_bulk_kernel<16, 2>, Q, ncol, w, v, N, ra); break;
        case 24: launch_bulk(ctx, bdot_bulk_kernel<24, 2>, Q, ncol, w, v, N, ra); break;
        case 32: launch_bulk(ctx, bdot_bulk_kernel<32, 2>, Q, ncol, w, v, N, ra); break;
        default: launch_bulk(ctx, bdot_bulk_kernel<40, 2>, Q, ncol, w, v, N, ra); break;
      }
      L.done();
    }
    // one collective for all column chunks (out_w / out_v are contiguous over the chunks)
    allreduce2(ctx, out_w, total, out_v, total);
    return;
  }
  for (int off = 0; off < total; off += 24) {
    std::vector<const double*> cols(cols_all.begin() + off, cols_all.begin() + std::min(total, off + 24));
    const int ncol = (int)cols.size();
    const int nc = nc_round(ncol);
    RedArgs ra = red_args(ctx, out_w + off);
    ra.out2 = out_v + off;
    ra.split = nc;
    ra.valid = ncol;
    ColPtrs Q = make_cols_padded(cols, nc);
    Launch L(ctx, "bdot", 8.0 * N * (ncol + 2));
    switch (nc) {
      case 8: launch_k(ctx, bdot2_tile_kernel<8>, N / 4, dim3(256), Q, ncol, w, v, N, ra); break;
      case 16: launch_k(ctx, bdot2_tile_kernel<16>, N / 4, dim3(256), Q, ncol, w, v, N, ra); break;
      default: launch_k(ctx, bdot2_tile_kernel<24>, N / 4, dim3(256), Q, ncol, w, v, N, ra); break;
    }
    L.done();
  }
  allreduce2(ctx, out_w, total, out_v, total);
}

void bupd_gram(rk_ctx* ctx, const std::vector<const double*>& cols, int k, const double* g,
               const double* grow, double* hout, double* w, int64_t N, double* red_out) {
  const int ncol = (int)cols.size();
  RK_REQUIRE(ncol <= MAXCOL, RK_EINVAL, "too many columns in a block product");
  RK_REQUIRE(pick_vec(N, {w}, cols) == 2, RK_EUNSUPPORTED, "bupd_gram needs even N, aligned columns");
  const int nc = nc_round(ncol);
  ColPtrs Q = make_cols_padded(cols, nc);
  RedArgs ra = red_args(ctx, red_out);
  Launch L(ctx, "bupd", 8.0 * N * (ncol + 2));
  // bulk-copy form at large N (>= 16 ring tiles per SM: the ring's fill and
  // drain are amortised); RK_BUPD_BULK: 0 never, 2 always
  if (ctx->bupd_bulk == 2 || (ctx->bupd_bulk == 1 && N >= (int64_t)BK_ROWS * ctx->sms * 16)) {
    launch_bulk_smem(ctx, BU_SMEM, bupd_gram_bulk_kernel, Q, ncol, k, g, grow, 1.0, hout, w, N, ra);
    L.done();
    allreduce(ctx, red_out, 1);
    return;
  }
#define RK_BG(NCV) launch_k(ctx, bupd_gram_kernel<NCV>, N / (2 * TRV), dim3(256), Q, ncol, k, g, grow, hout, w, N, ra)
  switch (nc) {
    case 8: RK_BG(8); break;
    case 16: RK_BG(16); break;
    case 24: RK_BG(24); break;
    case 32: RK_BG(32); break;
    case 40: RK_BG(40); break;
    case 48: RK_BG(48); break;
    case 56: RK_BG(56); break;
    case 64: RK_BG(64); break;
    case 72: RK_BG(72); break;
    default: RK_BG(80); break;
  }
#undef RK_BG
  L.done();
  allreduce(ctx, red_out, 1);
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
  // large N: two bulk-copy block updates in column-chunk order (r -= C xi
  // with ||r||^2, then x += U xi) -- the row-interleaved kernel below reads
  // the 2k columns with poor DRAM page locality (4.4 TB/s at c4)
  if (vec == 2 && ctx->bupd_bulk != 0 &&
      (ctx->bupd_bulk == 2 || N >= (int64_t)BK_ROWS * ctx->sms * 16)) {
    Launch L(ctx, "proj", 8.0 * N * (k * (x ? 2 : 1) + 2 + (x ? 2 : 0)));
    launch_bulk_smem(ctx, BU_SMEM, bupd_gram_bulk_kernel, Cp, k, 0, xi, (const double*)nullptr, 1.0, (double*)nullptr, r, N,
                ra);
    if (x) {
      RedArgs none = red_args(ctx, nullptr);
      launch_bulk_smem(ctx, BU_SMEM, bupd_gram_bulk_kernel, Up, k, 0, xi, (const double*)nullptr, -1.0, (double*)nullptr, x,
                  N, none);
    }
    L.done();
    allreduce(ctx, red_out, 1);
    return;
  }
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

namespace {
template <int NC>
void launch_rotate_cb(rk_ctx* ctx, ColPtrs Q, int k, int kout, const double* Th, int64_t N, bool vec2) {
  for (int c = k; c < NC; ++c) Q.p[c] = Q.p[0];
  TMat<NC> tm;
  memset(&tm, 0, sizeof(tm));
  for (int o = 0; o < kout; ++o)
    for (int c = 0; c < k; ++c) tm.t[o * NC + c] = Th[(size_t)o * k + c];
  // two cells per thread while the k inputs fit the registers
  if constexpr (NC <= 32) {
    if (vec2) {
      launch_k(ctx, rotate_cb_kernel<NC, 2>, N / 2, dim3(256), Q, k, kout, tm, N);
      return;
    }
  }
  launch_k(ctx, rotate_cb_kernel<NC, 1>, N, dim3(256), Q, k, kout, tm, N);
}
}  // namespace

void rotate(rk_ctx* ctx, const std::vector<double*>& cols, const double* T, int64_t N, int kout,
            const double* T_host) {
  const int k = (int)cols.size();
  if (k == 0) return;
  if (kout < 0) kout = k;
  RK_REQUIRE(kout >= 1 && kout <= k, RK_EINVAL, "rotate: 1 <= kout <= k");
  const int nc = nc_bucket(k);
  ColPtrs Q;
  memset(&Q, 0, sizeof(Q));
  for (int c = 0; c < k; ++c) Q.p[c] = cols[c];
  Launch L(ctx, "rotate", 8.0 * N * (k + kout));
  if (T_host) {
    std::vector<const double*> cc(cols.begin(), cols.end());
    const bool vec2 = pick_vec(N, {}, cc) == 2;
    switch (nc) {
      case 8: launch_rotate_cb<8>(ctx, Q, k, kout, T_host, N, vec2); break;
      case 16: launch_rotate_cb<16>(ctx, Q, k, kout, T_host, N, vec2); break;
      case 32: launch_rotate_cb<32>(ctx, Q, k, kout, T_host, N, vec2); break;
      default: launch_rotate_cb<48>(ctx, Q, k, kout, T_host, N, vec2); break;
    }
    L.done();
    return;
  }
  switch (nc) {
    case 8: launch_k(ctx, rotate_kernel<8>, N, dim3(256), Q, k, kout, T, N); break;
    case 16: launch_k(ctx, rotate_kernel<16>, N, dim3(256), Q, k, kout, T, N); break;
    case 32: launch_k(ctx, rotate_kernel<32>, N, dim3(256), Q, k, kout, T, N); break;
    default: launch_k(ctx, rotate_kernel<48>, N, dim3(256), Q, k, kout, T, N); break;
  }
  L.done();
}

}  // namespace rk
