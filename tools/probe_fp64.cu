// Microbenchmark probe (not part of the product path): measures the B200's
// FP64 FMA peak, FP64 exp() throughput and a streaming copy bandwidth with
// CUDA events, so DESIGN.md can state the ALU roofline of the ionic kernel.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void dexp_kernel(double* out, int iters) {
  double v = -80.0 + threadIdx.x * 1e-3, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
    acc0 += exp(v * 0.01 + i * 1e-6); acc1 += exp(v * 0.02 - i * 1e-6);
    acc2 += exp(v * 0.03 + i * 2e-6); acc3 += exp(v * 0.04 - i * 2e-6);
  }
  double s = acc0 + acc1 + acc2 + acc3;
  if (s == 12345.678) out[0] = s;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2\":%d,\"smem_optin\":%zu,\"clock_khz\":%d,\"coop\":%d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate, p.cooperativeLaunch);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma rep %d: %.3f ms  %.2f TFLOP/s fp64\n", rep, ms, fl / ms / 1e9);
  }
  for (int rep = 0; rep < 3; ++rep) {
    int it = 2048;
    cudaEventRecord(e0); dexp_kernel<<<blocks, threads>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ne = 4.0 * it * blocks * threads;
    printf("dexp rep %d: %.3f ms  %.2f Gexp/s\n", rep, ms, ne / ms / 1e6);
  }
  size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB per array
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<p.multiProcessorCount * 16, 256>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy rep %d: %.3f ms  %.1f GB/s\n", rep, ms, 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
