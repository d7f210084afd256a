// Shared device helpers and launch utilities of the librk kernel translation
// units (stencil.cu, blockops.cu, bicg.cu).  Not part of the ABI.
//
// Every librk kernel is HBM-bound fp64 work on the CUDA cores (0.1-0.3
// flop/B, SURVEY §8(a) "Tensor cores"):
//  * coalesced x-fastest rows, 16-byte loads wherever the data allows;
//  * streaming (ld.global.nc.L1::no_allocate) loads for data read once per
//    launch (bands, basis columns);
//  * grids sized from each instantiation's occupancy: SMs x resident CTAs,
//    grid-stride loops;
//  * deterministic two-stage reductions (per-CTA partials + fixed-order
//    finalisation by the last CTA; no floating-point atomics).
#pragma once
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
  if (ra.defer) return;   // the consuming kernel sums the partials (CoefIn)
#ifdef RK_EXP_NO_FINAL   // experiment only: per-CTA partials, no cross-CTA finalisation
  return;
#endif
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(ra.counter, 1u) == (unsigned)(G - 1));
  __syncthreads();
  if (last) {
    __threadfence();
    if constexpr (NV > 8) {
      // many values (block dot products): one warp per value, each lane with
      // 4 independent partial sums
      for (int q = warp; q < nv; q += nwarps) {
        const double* p = ra.partials + (int64_t)q * G;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int c = lane;
        for (; c + 96 < G; c += 128) {
          s0 += __ldcg(p + c);
          s1 += __ldcg(p + c + 32);
          s2 += __ldcg(p + c + 64);
          s3 += __ldcg(p + c + 96);
        }
        for (; c < G; c += 32) s0 += __ldcg(p + c);
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
          if (q < ra.split) {
            if (q < ra.valid) ra.out[q] = s;
          } else if (q - ra.split < ra.valid) {
            ra.out2[q - ra.split] = s;
          }
        }
      }
    } else {
      // few values (norms, the rBiCGStab scalars): every thread loads its
      // partials of all values at once (nv loads in flight per round, G /
      // nthreads rounds), then one more block reduction per value -- fewer
      // dependent L2 round trips on the critical path; a fixed order, so the
      // result is still deterministic (measured: -1 to -2 us per launch)
      double a[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) a[q] = 0.0;
      for (int c = tid; c < G; c += nthreads) {
#pragma unroll
        for (int q = 0; q < NV; ++q)
          if (q < nv) a[q] += __ldcg(ra.partials + (int64_t)q * G + c);
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (q < nv) {
          double s = a[q];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
          if (lane == 0) sm[q][warp] = s;   // sm is free: every thread passed the barrier above
        }
      }
      __syncthreads();
      for (int q = warp; q < nv; q += nwarps) {
        double s = lane < nwarps ? sm[q][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
          if (q < ra.split) {
            if (q < ra.valid) ra.out[q] = s;
          } else if (q - ra.split < ra.valid) {
            ra.out2[q - ra.split] = s;
          }
        }
      }
    }
    if (tid == 0) atomicExch(ra.counter, 0u);
  }
}


// Deferred finalisation (one rank): the consumer of a reduction sums its
// per-CTA partials part[q * G + b] (b < G) itself, in a fixed order that every
// CTA repeats (thread t sums partials t, t + 256, ...; a warp shuffle tree;
// the 8 warp sums in order), instead of the producer's last CTA doing it
// behind a fence and an atomic.  256-thread CTAs; dst (shared) gets the nv
// sums; ends with a barrier.
template <int NV>
__device__ __forceinline__ void block_sum_partials(const double* part, int G, int nv, double* dst) {
  __shared__ double wsum[NV][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c0 = 0; c0 < NV; c0 += 8) {
    if (c0 < nv) {
      constexpr int U = NV < 8 ? NV : 8;
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = 0.0;
      for (int b = threadIdx.x; b < G; b += 256) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u < nv) a[u] += __ldcg(part + (int64_t)(c0 + u) * G + b);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a[u] += __shfl_down_sync(0xffffffffu, a[u], o);
        if (lane == 0 && c0 + u < NV) wsum[c0 + u][warp] = a[u];
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += wsum[c][q];
    dst[c] = s;
  }
  __syncthreads();
}

// Columns are processed in groups of 8 with unguarded loads (the host pads
// the last group with a duplicate pointer and zero coefficients), so every
// thread keeps 8 x VEC loads in flight per group.
constexpr int GRP = 8;

// =================================================================== host
namespace {


// Grid = min(work / CTA, SMs x resident CTAs of this instantiation).
template <typename... KArgs, typename... Args>
int launch_k(rk_ctx* ctx, void (*kern)(KArgs...), int64_t work_threads, dim3 blk,
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
  launch_pdl(ctx, kern, dim3(grid), blk, 0, std::forward<Args>(args)...);
  return grid;
}

inline RedArgs red_args(rk_ctx* ctx, double* out) {
  RedArgs ra;
  ra.partials = ctx->partials;
  ra.counter = ctx->counter;
  ra.out = out;
  ra.gate = ctx->gate;
  return ra;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// VEC = 2 iff N is even and every pointer is 16-byte aligned.
inline int pick_vec(int64_t N, std::initializer_list<const void*> ps,
             const std::vector<const double*>& cols = {}) {
  if (N & 1) return 1;
  for (auto p : ps)
    if (p && !aligned16(p)) return 1;
  for (auto p : cols)
    if (p && !aligned16(p)) return 1;
  return 2;
}

// Pad to a multiple of GRP with the first column of the last group.
inline ColPtrs make_cols_padded(const std::vector<const double*>& v, int nc) {
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

}  // namespace

}  // namespace rk
