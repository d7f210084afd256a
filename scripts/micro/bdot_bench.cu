// Microbenchmark: block-dot / block-update variants at c3 / c4 sizes (not part of librk).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o bdot_bench bdot_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct ColPtrs { const double* p[80]; };

__device__ __forceinline__ double2 ldst(const double* p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  for (uint32_t n = 0; !ok; ++n) {
    if (n > (1u << 26)) __trap();
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// ---------------- V0: row-wise, groups of 8 columns (current librk)
template <int NC>
__global__ void __launch_bounds__(256) bdot_v0(ColPtrs Q, int ncol, const double* __restrict__ w, int64_t N, double* out) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N / 2; e += stride) {
    const int64_t r = e * 2;
    const double2 wv = __ldg(reinterpret_cast<const double2*>(w + r));
#pragma unroll
    for (int g = 0; g < NC / 8; ++g) {
      if (g * 8 < ncol) {
        double2 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = ldst(Q.p[g * 8 + u] + r);
#pragma unroll
        for (int u = 0; u < 8; ++u) { acc[g * 8 + u] = fma(q[u].x, wv.x, acc[g * 8 + u]); acc[g * 8 + u] = fma(q[u].y, wv.y, acc[g * 8 + u]); }
      }
    }
  }
  double s = 0; 
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;  // keep live
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------- V2: column-chunk, w in registers (R rows per thread), 4 columns unrolled
template <int NC, int RV>
__global__ void __launch_bounds__(256) bdot_v2(ColPtrs Q, int ncol, const double* __restrict__ w, int64_t N, double* out) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int64_t tile = 256 * 2 * RV;  // rows per CTA tile
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < N; t0 += (int64_t)gridDim.x * tile) {
    double2 wv[RV];
#pragma unroll
    for (int v = 0; v < RV; ++v) wv[v] = __ldg(reinterpret_cast<const double2*>(w + t0 + (v * 256 + threadIdx.x) * 2));
#pragma unroll
    for (int c = 0; c < NC; c += 2) {
      if (c < ncol) {
        double2 q0[RV], q1[RV];
#pragma unroll
        for (int v = 0; v < RV; ++v) q0[v] = ldst(Q.p[c] + t0 + (v * 256 + threadIdx.x) * 2);
#pragma unroll
        for (int v = 0; v < RV; ++v) q1[v] = ldst(Q.p[c + 1] + t0 + (v * 256 + threadIdx.x) * 2);
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          acc[c] = fma(q0[v].x, wv[v].x, acc[c]); acc[c] = fma(q0[v].y, wv[v].y, acc[c]);
          acc[c + 1] = fma(q1[v].x, wv[v].x, acc[c + 1]); acc[c + 1] = fma(q1[v].y, wv[v].y, acc[c + 1]);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c];
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------- V3: TMA bulk pipeline. 8 consumer warps + 1 producer warp.
// Tile = TR rows (TR*8 bytes per column); stage ring of ST tiles.
template <int NC, int TR, int ST>
__global__ void __launch_bounds__(288, 1) bdot_v3(ColPtrs Q, int ncol, const double* __restrict__ w, int64_t N, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = reinterpret_cast<double*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * TR * 8);
  uint64_t* empty = full + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = N / TR;
  const int per = ncol + 1;
  if (warp == 8) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int c = 0; c < per; ++c, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1;
          if (it >= ST) mbar_wait(&empty[s], ph ^ 1);
          mbar_expect(&full[s], TR * 8);
          const double* src = (c == 0 ? w : Q.p[c - 1]) + t * TR;
          bulk_g2s(ring + (size_t)s * TR, src, TR * 8, &full[s]);
        }
      }
    }
    return;
  }
  constexpr int RPT = TR / 256;  // rows per consumer thread
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  uint32_t it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double wv[RPT];
    {
      const int s = it % ST; const uint32_t ph = (it / ST) & 1;
      mbar_wait(&full[s], ph);
      const double* b = ring + (size_t)s * TR + threadIdx.x * 2;
#pragma unroll
      for (int v = 0; v < RPT; v += 2) { double2 d = *reinterpret_cast<const double2*>(b + v * 256); wv[v] = d.x; wv[v + 1] = d.y; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++it;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c < ncol) {
        const int s = it % ST; const uint32_t ph = (it / ST) & 1;
        mbar_wait(&full[s], ph);
        const double* b = ring + (size_t)s * TR + threadIdx.x * 2;
#pragma unroll
        for (int v = 0; v < RPT; v += 2) { double2 d = *reinterpret_cast<const double2*>(b + v * 256); acc[c] = fma(d.x, wv[v], acc[c]); acc[c] = fma(d.y, wv[v + 1], acc[c]); }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++it;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c];
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------- bupd V0 (current): w -= sum g_c Q_c
template <int NC>
__global__ void __launch_bounds__(256) bupd_v0(ColPtrs Q, int ncol, const double* __restrict__ g, double* __restrict__ w, int64_t N) {
  __shared__ double gsh[NC];
  for (int c = threadIdx.x; c < NC; c += blockDim.x) gsh[c] = c < ncol ? g[c] : 0.0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N / 2; e += stride) {
    const int64_t r = e * 2;
    double2 wv = *reinterpret_cast<double2*>(w + r);
#pragma unroll
    for (int gi = 0; gi < NC / 8; ++gi) {
      if (gi * 8 < ncol) {
        double2 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = ldst(Q.p[gi * 8 + u] + r);
#pragma unroll
        for (int u = 0; u < 8; ++u) { wv.x = fma(-gsh[gi * 8 + u], q[u].x, wv.x); wv.y = fma(-gsh[gi * 8 + u], q[u].y, wv.y); }
      }
    }
    *reinterpret_cast<double2*>(w + r) = wv;
  }
}

// ---------------- bupd V3: TMA pipeline (w tile + column tiles), direct stores
template <int NC, int TR, int ST>
__global__ void __launch_bounds__(288, 1) bupd_v3(ColPtrs Q, int ncol, const double* __restrict__ g, double* __restrict__ w, int64_t N) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = reinterpret_cast<double*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * TR * 8);
  uint64_t* empty = full + ST;
  __shared__ double gsh[NC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < NC; c += blockDim.x) gsh[c] = c < ncol ? g[c] : 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = N / TR;
  const int per = ncol + 1;
  if (warp == 8) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int c = 0; c < per; ++c, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1;
          if (it >= ST) mbar_wait(&empty[s], ph ^ 1);
          mbar_expect(&full[s], TR * 8);
          const double* src = (c == 0 ? w : Q.p[c - 1]) + t * TR;
          bulk_g2s(ring + (size_t)s * TR, src, TR * 8, &full[s]);
        }
      }
    }
    return;
  }
  constexpr int RPT = TR / 256;
  uint32_t it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double wv[RPT];
    {
      const int s = it % ST; const uint32_t ph = (it / ST) & 1;
      mbar_wait(&full[s], ph);
      const double* b = ring + (size_t)s * TR + threadIdx.x * 2;
#pragma unroll
      for (int v = 0; v < RPT; v += 2) { double2 d = *reinterpret_cast<const double2*>(b + v * 256); wv[v] = d.x; wv[v + 1] = d.y; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++it;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c < ncol) {
        const int s = it % ST; const uint32_t ph = (it / ST) & 1;
        mbar_wait(&full[s], ph);
        const double* b = ring + (size_t)s * TR + threadIdx.x * 2;
        const double gc = gsh[c];
#pragma unroll
        for (int v = 0; v < RPT; v += 2) { double2 d = *reinterpret_cast<const double2*>(b + v * 256); wv[v] = fma(-gc, d.x, wv[v]); wv[v + 1] = fma(-gc, d.y, wv[v + 1]); }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++it;
      }
    }
    double* dst = w + t * TR + threadIdx.x * 2;
#pragma unroll
    for (int v = 0; v < RPT; v += 2) *reinterpret_cast<double2*>(dst + v * 256) = make_double2(wv[v], wv[v + 1]);
  }
}


// ---------------- V4: column-chunk, w in registers, G columns per group
template <int NC, int RV, int G>
__global__ void __launch_bounds__(256) bdot_v4(ColPtrs Q, int ncol, const double* __restrict__ w, int64_t N, double* out) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int64_t tile = 256 * 2 * RV;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < N; t0 += (int64_t)gridDim.x * tile) {
    double2 wv[RV];
#pragma unroll
    for (int v = 0; v < RV; ++v) wv[v] = __ldg(reinterpret_cast<const double2*>(w + t0 + (v * 256 + threadIdx.x) * 2));
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double2 q[G][RV];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int v = 0; v < RV; ++v) q[g][v] = ldst(Q.p[c + g] + t0 + (v * 256 + threadIdx.x) * 2);
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int v = 0; v < RV; ++v) { acc[c + g] = fma(q[g][v].x, wv[v].x, acc[c + g]); acc[c + g] = fma(q[g][v].y, wv[v].y, acc[c + g]); }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c];
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------- bupd V2: column-chunk, w tile in registers, G columns per group
template <int NC, int RV, int G>
__global__ void __launch_bounds__(256) bupd_v2(ColPtrs Q, int ncol, const double* __restrict__ g, double* __restrict__ w, int64_t N) {
  __shared__ double gsh[NC];
  for (int c = threadIdx.x; c < NC; c += blockDim.x) gsh[c] = c < ncol ? g[c] : 0.0;
  __syncthreads();
  const int64_t tile = 256 * 2 * RV;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < N; t0 += (int64_t)gridDim.x * tile) {
    double2 wv[RV];
#pragma unroll
    for (int v = 0; v < RV; ++v) wv[v] = *reinterpret_cast<const double2*>(w + t0 + (v * 256 + threadIdx.x) * 2);
#pragma unroll
    for (int c = 0; c < NC; c += G) {
      if (c < ncol) {
        double2 q[G][RV];
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
          for (int v = 0; v < RV; ++v) q[gg][v] = ldst(Q.p[c + gg] + t0 + (v * 256 + threadIdx.x) * 2);
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
          for (int v = 0; v < RV; ++v) { wv[v].x = fma(-gsh[c + gg], q[gg][v].x, wv[v].x); wv[v].y = fma(-gsh[c + gg], q[gg][v].y, wv[v].y); }
      }
    }
#pragma unroll
    for (int v = 0; v < RV; ++v) *reinterpret_cast<double2*>(w + t0 + (v * 256 + threadIdx.x) * 2) = wv[v];
  }
}

__global__ void rd_kernel(const double* __restrict__ a, int64_t N, double* out) {
  double s = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N / 2; e += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ldst(a + 2 * e); s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
__global__ void cp_kernel(const double* __restrict__ a, double* __restrict__ b, int64_t N) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N / 2; e += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(b)[e] = ldst(a + 2 * e);
}
__global__ void fill(double* a, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = v * (1 + (i % 7));
}

template <typename F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc > 2 && atoi(argv[2]) > 24) { printf("ncol must be <= 24 (template NC)\n"); return 1; }
  const int64_t N = argc > 1 ? atoll(argv[1]) : (1 << 21);
  const int ncol = argc > 2 ? atoi(argv[2]) : 20;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double*> cols(ncol + 1);
  for (auto& p : cols) { CK(cudaMalloc(&p, N * 8)); fill<<<1024, 256>>>(p, N, 1e-3); }
  double *w, *out, *g; CK(cudaMalloc(&w, N * 8)); CK(cudaMalloc(&out, 1 << 20)); CK(cudaMalloc(&g, 80 * 8));
  fill<<<1024, 256>>>(w, N, 1.0); fill<<<1, 80>>>(g, 80, 1e-6);
  CK(cudaDeviceSynchronize());
  ColPtrs Q; for (int c = 0; c < 80; ++c) Q.p[c] = cols[c % ncol];
  const double W = 8.0 * N;
  printf("N=%lld ncol=%d sms=%d\n", (long long)N, ncol, sms);
  auto rep = [&](const char* name, float ms, double words) { printf("%-34s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, words * W / (ms * 1e-3) / 1e9); };
  rep("read 1 vec", timeit([&] { rd_kernel<<<sms * 8, 256>>>(cols[0], N, out); }), 1);
  rep("copy 1 vec", timeit([&] { cp_kernel<<<sms * 8, 256>>>(cols[0], cols[1], N); }), 2);
  // V0
  for (int occ : {2, 3, 4}) {
    char nm[64]; snprintf(nm, 64, "bdot_v0<24> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v0<24><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
  }
  for (int occ : {2, 3, 4}) {
    char nm[64]; snprintf(nm, 64, "bdot_v2<24,2> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v2<24, 2><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
    snprintf(nm, 64, "bdot_v2<24,4> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v2<24, 4><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
  }
  {
    constexpr int TR = 1024, ST = 24;
    const int smem = ST * TR * 8 + 2 * ST * 8;
    CK(cudaFuncSetAttribute(bdot_v3<24, TR, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    rep("bdot_v3<24,1024,24> tma", timeit([&] { bdot_v3<24, TR, ST><<<sms, 288, smem>>>(Q, ncol, w, N, out); }), ncol + 1);
  }
  {
    constexpr int TR = 2048, ST = 12;
    const int smem = ST * TR * 8 + 2 * ST * 8;
    CK(cudaFuncSetAttribute(bdot_v3<24, TR, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    rep("bdot_v3<24,2048,12> tma", timeit([&] { bdot_v3<24, TR, ST><<<sms, 288, smem>>>(Q, ncol, w, N, out); }), ncol + 1);
  }
  {
    constexpr int TR = 512, ST = 24;
    const int smem = ST * TR * 8 + 2 * ST * 8;
    CK(cudaFuncSetAttribute(bdot_v3<24, TR, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    rep("bdot_v3<24,512,24> tma 2/SM", timeit([&] { bdot_v3<24, TR, ST><<<sms * 2, 288, smem>>>(Q, ncol, w, N, out); }), ncol + 1);
  }
  for (int occ : {2, 3, 4}) {
    char nm[64]; snprintf(nm, 64, "bupd_v0<24> grid %dx", occ);
    rep(nm, timeit([&] { bupd_v0<24><<<sms * occ, 256>>>(Q, ncol, g, w, N); }), ncol + 2);
  }
  {
    constexpr int TR = 1024, ST = 24;
    const int smem = ST * TR * 8 + 2 * ST * 8;
    CK(cudaFuncSetAttribute(bupd_v3<24, TR, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    rep("bupd_v3<24,1024,24> tma", timeit([&] { bupd_v3<24, TR, ST><<<sms, 288, smem>>>(Q, ncol, g, w, N); }), ncol + 2);
  }
  {
    constexpr int TR = 512, ST = 24;
    const int smem = ST * TR * 8 + 2 * ST * 8;
    CK(cudaFuncSetAttribute(bupd_v3<24, TR, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    rep("bupd_v3<24,512,24> tma 2/SM", timeit([&] { bupd_v3<24, TR, ST><<<sms * 2, 288, smem>>>(Q, ncol, g, w, N); }), ncol + 2);
  }
  for (int occ : {2, 3, 4, 6}) {
    char nm[64];
    snprintf(nm, 64, "bdot_v4<24,4,2> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v4<24, 4, 2><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
    snprintf(nm, 64, "bdot_v4<24,4,4> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v4<24, 4, 4><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
    snprintf(nm, 64, "bdot_v4<24,8,1> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v4<24, 8, 1><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
    snprintf(nm, 64, "bdot_v4<24,2,4> grid %dx", occ);
    rep(nm, timeit([&] { bdot_v4<24, 2, 4><<<sms * occ, 256>>>(Q, ncol, w, N, out); }), ncol + 1);
    snprintf(nm, 64, "bupd_v2<24,4,2> grid %dx", occ);
    rep(nm, timeit([&] { bupd_v2<24, 4, 2><<<sms * occ, 256>>>(Q, ncol, g, w, N); }), ncol + 2);
    snprintf(nm, 64, "bupd_v2<24,4,1> grid %dx", occ);
    rep(nm, timeit([&] { bupd_v2<24, 4, 1><<<sms * occ, 256>>>(Q, ncol, g, w, N); }), ncol + 2);
    snprintf(nm, 64, "bupd_v2<24,2,4> grid %dx", occ);
    rep(nm, timeit([&] { bupd_v2<24, 2, 4><<<sms * occ, 256>>>(Q, ncol, g, w, N); }), ncol + 2);
    snprintf(nm, 64, "bupd_v2<24,8,1> grid %dx", occ);
    rep(nm, timeit([&] { bupd_v2<24, 8, 1><<<sms * occ, 256>>>(Q, ncol, g, w, N); }), ncol + 2);
  }
  printf("done\n");
  return 0;
}
