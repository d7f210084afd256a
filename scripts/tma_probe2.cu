// Probe 2: chain.cu's per-plane issue (4D band box + 2 x 3D boxes on one mbarrier).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int EX = 36, EY = 12, XX = 38, XY = 14, ST = 7;
constexpr int B_BYTES = ST * EY * EX * 8, R_BYTES = EY * EX * 8, X_BYTES = XY * XX * 8;
constexpr int R_OFF = 24192, X_OFF = 27648, SLOT = 32000;

__global__ void probe(const __grid_constant__ CUtensorMap mb, const __grid_constant__ CUtensorMap mr,
                      const __grid_constant__ CUtensorMap mx, double* out, int gx0, int gy0, int pl, int which) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 5 * SLOT + 20736);
  unsigned char* base = smem + 2 * SLOT;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t bytes = 0;
  if (which & 1) bytes += B_BYTES;
  if (which & 2) bytes += R_BYTES;
  if (which & 4) bytes += X_BYTES;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes) : "memory");
    if (which & 1)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   ::"r"(su(base)), "l"(reinterpret_cast<uint64_t>(&mb)), "r"(su(bar)), "r"(gx0), "r"(gy0), "r"(pl), "r"(0) : "memory");
    if (which & 2)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(base + R_OFF)), "l"(reinterpret_cast<uint64_t>(&mr)), "r"(su(bar)), "r"(gx0), "r"(gy0), "r"(pl) : "memory");
    if (which & 4)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(base + X_OFF)), "l"(reinterpret_cast<uint64_t>(&mx)), "r"(su(bar)), "r"(gx0 - 1), "r"(gy0 - 1), "r"(pl + 1) : "memory");
  }
  uint32_t ok = 0;
  for (int it = 0; it < (1 << 22) && !ok; ++it)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok) : "r"(su(bar)), "r"(0), "r"(1000000u) : "memory");
  if (threadIdx.x == 0) out[0] = ok;
  const double* b = reinterpret_cast<const double*>(base);
  if (threadIdx.x == 0) { out[1] = b[(3 * EY + 5) * EX + 7]; out[2] = reinterpret_cast<const double*>(base + R_OFF)[5 * EX + 7];
                          out[3] = reinterpret_cast<const double*>(base + X_OFF)[6 * XX + 8]; }
}

int main() {
  const int nx = 128, ny = 128, nz = 16; const size_t N = (size_t)nx * ny * nz, P = nx * ny;
  std::vector<double> hb(N * ST), hr(N), hx(N + 2 * P, 0.0);
  for (size_t i = 0; i < hb.size(); ++i) hb[i] = 1e6 + i;
  for (size_t i = 0; i < N; ++i) { hr[i] = 2e6 + i; hx[P + i] = 3e6 + i; }
  double *db, *dr, *dx, *o;
  cudaMalloc(&db, hb.size() * 8); cudaMalloc(&dr, N * 8); cudaMalloc(&dx, hx.size() * 8); cudaMalloc(&o, 64);
  cudaMemcpy(db, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dr, hr.data(), N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMap mb, mr, mx;
  { cuuint64_t d[4] = {nx, ny, nz, ST}, s[3] = {nx * 8, nx * ny * 8, N * 8}; cuuint32_t bx[4] = {EX, EY, 1, ST};
    printf("enc b %d\n", (int)enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, db, d, s, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  { cuuint64_t d[3] = {nx, ny, nz}, s[2] = {nx * 8, nx * ny * 8}; cuuint32_t bx[3] = {EX, EY, 1};
    printf("enc r %d\n", (int)enc(&mr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dr, d, s, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  { cuuint64_t d[3] = {nx, ny, nz + 2}, s[2] = {nx * 8, nx * ny * 8}; cuuint32_t bx[3] = {XX, XY, 1};
    printf("enc x %d\n", (int)enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dx, d, s, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  const int smem = 5 * SLOT + 20736 + 128;
  printf("setattr %s\n", cudaGetErrorString(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)));
  for (int which : {1, 2, 4, 7}) {
    probe<<<1, 432, smem>>>(mb, mr, mx, o, 30, 14, 5, which);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[4]; cudaMemcpy(ho, o, 32, cudaMemcpyDeviceToHost);
    int x = 30 + 7, y = 14 + 5;
    printf("which %d err=%s done=%g band=%g (exp %g) r=%g (exp %g) x=%g (exp %g)\n", which, cudaGetErrorString(e), ho[0],
           ho[1], 1e6 + 3 * N + 5 * P + y * nx + x, ho[2], 2e6 + 5 * P + y * nx + x, ho[3], 3e6 + 5 * P + (14 - 1 + 6) * nx + (30 - 1 + 8));
  }
  return 0;
}
