// Standalone probe of the TMA + mbarrier sequence used by chain.cu
// (nvcc -gencode arch=compute_100a,code=sm_100a scripts/tma_probe.cu -lcuda).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap m, double* out, int c0, int c1, int c2, int variant) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  double* dst = reinterpret_cast<double*>(smem);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = 36 * 12 * 8;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes) : "memory");
    if (variant == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(dst)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(su(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(dst)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(su(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
  }
  uint32_t ok = 0;
  for (int it = 0; it < (1 << 20) && !ok; ++it)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok) : "r"(su(bar)), "r"(0) : "memory");
  if (threadIdx.x == 0) out[36 * 12] = ok;
  for (int i = threadIdx.x; i < 36 * 12; i += blockDim.x) out[i] = dst[i];
}

int main() {
  const int nx = 64, ny = 64, nz = 8;
  std::vector<double> h((size_t)nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 8 * 1024);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap m;
  cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 8, nx * ny * 8};
  cuuint32_t box[3] = {36, 12, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  for (int variant = 0; variant < 2; ++variant) {
    for (int c0 : {0, -2}) {
      probe<<<1, 128, 8192 + 128>>>(m, o, c0, -2, 3, variant);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> ho(36 * 12 + 1);
      cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
      // expected value at box (i, j): x = c0 + i, y = -2 + j, z = 3
      int bad = 0;
      for (int j = 0; j < 12; ++j) for (int i = 0; i < 36; ++i) {
        int x = c0 + i, y = -2 + j; double ex = (x >= 0 && x < nx && y >= 0 && y < ny) ? h[(size_t)3 * nx * ny + y * nx + x] : 0.0;
        if (ho[j * 36 + i] != ex) ++bad;
      }
      printf("variant %d c0 %d: err=%s done=%g mismatches=%d\n", variant, c0, cudaGetErrorString(e), ho[36 * 12], bad);
    }
  }
  return 0;
}
