// Read-only HBM bandwidth ceiling on this GPU (not part of librk): what a
// streaming reduction (the bdot pattern) can reach, with plain 16-byte
// loads (several in flight per thread) and with 1-D bulk copies into a
// shared-memory ring.  Prints GB/s of bytes read.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void __launch_bounds__(256) ld_sum(const double2* __restrict__ a, int64_t n2, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) { double2 v = __ldg(a + i); acc += v.x + v.y; }
  if (acc == 12345.678) out[0] = acc;
}

// contiguous-chunk variant: each CTA owns a contiguous range (the column-chunk order)
template <int U>
__global__ void __launch_bounds__(256) ld_sum_chunk(const double2* __restrict__ a, int64_t n2, int64_t chunk, double* out) {
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * chunk; base < n2; base += (int64_t)gridDim.x * chunk) {
    const int64_t end = base + chunk < n2 ? base + chunk : n2;
    for (int64_t i = base + threadIdx.x; i < end; i += U * 256) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (i + u * 256 < end) ? __ldg(a + i + u * 256) : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int BYTES>
__global__ void __launch_bounds__(256) bulk_sum(const double* __restrict__ a, int64_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* buf = reinterpret_cast<double*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + STAGES * BYTES);
  constexpr int DPS = BYTES / 8;
  const int64_t nblk = n / DPS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t blk, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar + s)), "r"(BYTES));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(buf + s * DPS)),
                 "l"(a + blk * DPS), "r"(BYTES), "r"(smem_u32(bar + s))
                 : "memory");
  };
  int64_t blk = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s)
      if (blk + (int64_t)s * gridDim.x < nblk) issue(blk + (int64_t)s * gridDim.x, s);
  double acc = 0.0;
  uint32_t phase = 0;
  int s = 0;
  for (; blk < nblk; blk += gridDim.x) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(bar + s)), "r"(phase));
    const double2* b2 = reinterpret_cast<const double2*>(buf + s * DPS);
    for (int q = threadIdx.x; q < DPS / 2; q += 256) { double2 v = b2[q]; acc += v.x + v.y; }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t nb = blk + (int64_t)STAGES * gridDim.x;
      if (nb < nblk) issue(nb, s);
    }
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t)50 << 20;   // doubles (400 MB)
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *a, *out; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(a, 0, n * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* nm, auto f) {
    for (int i = 0; i < 3; ++i) f();
    CK(cudaEventRecord(e0));
    const int R = 20;
    for (int i = 0; i < R; ++i) f();
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
    CK(cudaGetLastError());
    printf("%-40s %8.1f us %7.0f GB/s\n", nm, ms * 1e3, n * 8.0 / (ms * 1e-3) / 1e9);
  };
  char nm[96];
  for (int occ : {2, 4, 8}) {
    snprintf(nm, 96, "ld_sum<4> grid %dx", occ);
    timeit(nm, [&] { ld_sum<4><<<sms * occ, 256>>>((const double2*)a, n / 2, out); });
    snprintf(nm, 96, "ld_sum<8> grid %dx", occ);
    timeit(nm, [&] { ld_sum<8><<<sms * occ, 256>>>((const double2*)a, n / 2, out); });
  }
  for (int occ : {2, 4}) {
    const int64_t chunk = 2048;
    snprintf(nm, 96, "ld_sum_chunk<8> 2048 grid %dx", occ);
    timeit(nm, [&] { ld_sum_chunk<8><<<sms * occ, 256>>>((const double2*)a, n / 2, chunk, out); });
  }
  {
    constexpr int ST = 4, BY = 32768;
    auto k = bulk_sum<ST, BY>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * BY + 64));
    for (int occ : {1, 2}) {
      snprintf(nm, 96, "bulk_sum<4,32K> grid %dx", occ);
      timeit(nm, [&] { k<<<sms * occ, 256, ST * BY + 64>>>(a, n, out); });
    }
  }
  {
    constexpr int ST = 6, BY = 16384;
    auto k = bulk_sum<ST, BY>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * BY + 64));
    for (int occ : {1, 2}) {
      snprintf(nm, 96, "bulk_sum<6,16K> grid %dx", occ);
      timeit(nm, [&] { k<<<sms * occ, 256, ST * BY + 64>>>(a, n, out); });
    }
  }
  // copy for reference (read+write)
  double* b; CK(cudaMalloc(&b, n * 8));
  {
    const int R = 20;
    for (int i = 0; i < 3; ++i) cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
    printf("%-40s %8.1f us %7.0f GB/s (read+write)\n", "cudaMemcpy D2D", ms * 1e3, 2 * n * 8.0 / (ms * 1e-3) / 1e9);
  }
  printf("done\n");
  return 0;
}
