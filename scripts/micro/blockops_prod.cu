// Times librk's production block kernels (rk::bdot / rk::bupd, blockops.cu)
// through the built librk.so at c3/c4 sizes.  Not part of librk.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rk_internal.h"

__global__ void fillk(double* a, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v * (1 + (i % 7));
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : (1 << 21);
  const int ncol = argc > 2 ? atoi(argv[2]) : 20;
  rk_ctx* ctx = nullptr;
  if (rk_ctx_create(0, 0, 1, nullptr, nullptr, &ctx) != RK_OK) { printf("ctx: %s\n", rk_last_error()); return 1; }
  std::vector<const double*> cols;
  for (int c = 0; c < ncol; ++c) { double* p; cudaMalloc(&p, N * 8); fillk<<<1024, 256>>>(p, N, 1e-3); cols.push_back(p); }
  double *w, *d1, *out, *g;
  cudaMalloc(&w, N * 8); cudaMalloc(&d1, N * 8); cudaMalloc(&out, 4096); cudaMalloc(&g, 1024);
  fillk<<<1024, 256>>>(w, N, 1.0); fillk<<<1024, 256>>>(d1, N, 0.5); fillk<<<1, 128>>>(g, 128, 1e-9);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto f, int reps) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a, ctx->stream);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b, ctx->stream); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return 1e3 * ms / reps;
  };
  const double W = 8.0 * N;
  double us = timeit([&] { rk::bdot(ctx, cols, w, N, out); }, 20);
  printf("bdot  ncol=%d           %7.1f us %6.0f GB/s\n", ncol, us, (ncol + 1) * W / (us * 1e-6) / 1e9);
  us = timeit([&] { rk::bupd(ctx, cols, g, 1.0, w, N, {}, nullptr); }, 20);
  printf("bupd  ncol=%d nd=0      %7.1f us %6.0f GB/s\n", ncol, us, (ncol + 2) * W / (us * 1e-6) / 1e9);
  us = timeit([&] { rk::bupd(ctx, cols, g, 1.0, w, N, {d1}, out); }, 20);
  printf("bupd  ncol=%d nd=1(d)   %7.1f us %6.0f GB/s\n", ncol, us, (ncol + 3) * W / (us * 1e-6) / 1e9);
  us = timeit([&] { rk::bupd(ctx, cols, g, 1.0, w, N, {d1, nullptr}, out); }, 20);
  printf("bupd  ncol=%d nd=2(d,w) %7.1f us %6.0f GB/s\n", ncol, us, (ncol + 3) * W / (us * 1e-6) / 1e9);
  std::vector<const double*> cw(cols); cw.push_back(w);
  us = timeit([&] { rk::bdot(ctx, cw, w, N, out); }, 20);
  printf("bdot  ncol=%d (+w)      %7.1f us %6.0f GB/s\n", ncol + 1, us, (ncol + 1) * W / (us * 1e-6) / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
