// Standalone timing of the fused chain (chain.cu) at a given grid size, without
// Python: links chain.cu and calls chain_launch() directly.  Not part of librk.
// nvcc ... -I include -I paper_1501_03358_b200/csrc chain_bench.cu ../../paper_1501_03358_b200/csrc/chain.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rk_internal.h"

__global__ void fillk(double* a, int64_t n, double base, double amp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = base + amp * (double)((i * 2654435761ull) % 1000) / 1000.0;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 128;
  const int reps = argc > 2 ? atoi(argv[2]) : 50;
  rk_ctx ctx;
  ctx.device = 0;
  cudaStreamCreate(&ctx.stream);
  cudaDeviceGetAttribute(&ctx.sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  ctx.l2_bytes = l2;
  rk_op op;
  op.ctx = &ctx;
  op.g.nx = n; op.g.ny = n; op.g.nz_global = n; op.g.z0 = 0; op.g.nz_local = n; op.g.periodic_mask = 0;
  op.S = 7; op.P = (int64_t)n * n; op.N = op.P * n;
  op.force_chain = true;
  cudaMalloc(&op.bands, sizeof(double) * 7 * op.N);
  fillk<<<1024, 256>>>(op.bands, op.N, 8.0, 1.0);
  fillk<<<1024, 256>>>(op.bands + op.N, 6 * op.N, -1.0, 0.5);
  double *xb, *r, *t, *mid, *out;
  cudaMalloc(&xb, sizeof(double) * (op.N + 2 * op.P));
  cudaMemset(xb, 0, sizeof(double) * (op.N + 2 * op.P));
  fillk<<<1024, 256>>>(xb + op.P, op.N, 0.0, 1.0);
  cudaMalloc(&r, sizeof(double) * op.N);
  fillk<<<1024, 256>>>(r, op.N, -0.5, 1.0);
  cudaMalloc(&t, sizeof(double) * op.N);
  cudaMalloc(&mid, sizeof(double) * op.N);
  cudaMalloc(&out, sizeof(double) * (op.N + 2 * op.P));
  printf("n=%d max_stages=%d sms=%d\n", n, rk::chain_max_stages(&op), ctx.sms);
  struct Cfg { const char* name; int k[3]; bool has_t, has_mid, rhs; double words; };
  Cfg cfgs[] = {{"SPMV1,SWEEP,SWEEP (+t)", {rk::CK_SPMV1, rk::CK_SWEEP, rk::CK_SWEEP}, true, false, false, 7 + 1 + 1 + 1},
                {"SWEEP,SWEEP,SWEEP", {rk::CK_SWEEP, rk::CK_SWEEP, rk::CK_SWEEP}, false, false, true, 7 + 1 + 1 + 1},
                {"SWEEP,SWEEP,SPMV (+mid)", {rk::CK_SWEEP, rk::CK_SWEEP, rk::CK_SPMV}, false, true, true, 7 + 1 + 1 + 2}};
  double om[3] = {0.8, 0.8, 1.0};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"32x16 pd2", "32x8 pd2", "16x8 pd2", "16x8 pd3", "16x16 pd2", "32x16 pd2 x-pairs"};
  for (int ci = 0; ci < 6; ++ci) {
  char buf[8];
  snprintf(buf, 8, "%d", ci);
  setenv("RK_CHAIN_CFG", buf, 1);
  printf("-- tile cfg %s (max stages %d)\n", names[ci], rk::chain_max_stages(&op));
  for (auto& c : cfgs) {
    auto run = [&] {
      rk::chain_launch(&op, 3, c.k, om, xb + op.P, c.rhs ? r : nullptr, c.has_t ? t : nullptr,
                       c.has_mid ? mid : nullptr, out + op.P);
    };
    for (int i = 0; i < 3; ++i) run();
    cudaEventRecord(a, ctx.stream);
    for (int i = 0; i < reps; ++i) run();
    cudaEventRecord(b, ctx.stream);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    const double us = 1e3 * ms / reps;
    printf("%-28s %8.1f us  %7.0f GB/s (alg %.0f W)  %s\n", c.name, us, c.words * 8.0 * op.N / (us * 1e-6) / 1e9,
           c.words, cudaGetErrorString(e));
  }
  }
  // two-stage launches (halo 1) for comparison, default tile config
  setenv("RK_CHAIN_CFG", "0", 1);
  {
    int k2[2] = {rk::CK_SWEEP, rk::CK_SWEEP};
    auto run = [&] { rk::chain_launch(&op, 2, k2, om, xb + op.P, r, nullptr, nullptr, out + op.P); };
    for (int i = 0; i < 3; ++i) run();
    cudaEventRecord(a, ctx.stream);
    for (int i = 0; i < reps; ++i) run();
    cudaEventRecord(b, ctx.stream);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1e3 * ms / reps;
    printf("NST=2 SWEEP,SWEEP %8.1f us (%.1f us/stage)  %s\n", us, us / 2, cudaGetErrorString(cudaGetLastError()));
    int k1[1] = {rk::CK_SWEEP};
    auto run1 = [&] { rk::chain_launch(&op, 1, k1, om, xb + op.P, r, nullptr, nullptr, out + op.P); };
    for (int i = 0; i < 3; ++i) run1();
    cudaEventRecord(a, ctx.stream);
    for (int i = 0; i < reps; ++i) run1();
    cudaEventRecord(b, ctx.stream);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("NST=1 SWEEP       %8.1f us  %s\n", 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
// chain_run's unfused fallback is not exercised here
namespace rk {
void stencil(rk_op*, int, const double*, const double*, double*, double*, double, double*, int) { abort(); }
}
