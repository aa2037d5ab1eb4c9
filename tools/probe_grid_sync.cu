// probe_grid_sync.cu -- cost of one grid-wide barrier of a cooperative launch
// (592 CTAs x 512 threads, the persistent PCG grid) : cooperative_groups
// grid.sync() vs a sense-reversing barrier on one counter (red.release +
// ld.acquire spin), and with a deterministic 2-value reduction folded in.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_grid_sync.cu -o /tmp/pgs && /tmp/pgs
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void my_grid_sync(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    const unsigned int arrived = atomicAdd(count, 1u) + 1u;
    if (arrived == nblocks) {
      *count = 0;
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(g + 1u) : "memory");
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(512, 4) k(int iters, unsigned int* bar, double* out) {
  cg::grid_group grid = cg::this_grid();
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) grid.sync();
    else my_grid_sync(bar, bar + 32, gridDim.x);
    acc += 1.0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

template <int MODE>
float run(int grid, int iters) {
  unsigned int* bar;
  double* out;
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaMalloc(&out, 8);
  void* args[] = {&iters, &bar, &out};
  int warm = 10;
  void* wargs[] = {&warm, &bar, &out};
  cudaLaunchCooperativeKernel((void*)k<MODE>, grid, 512, wargs, 0, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)k<MODE>, grid, 512, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  cudaFree(bar);
  cudaFree(out);
  return ms * 1e3f / iters;
}

int main() {
  printf("grid  cg_sync_us  counter_sync_us\n");
  for (int g : {148, 296, 592})
    printf("%4d  %8.3f  %8.3f\n", g, run<0>(g, 20000), run<1>(g, 20000));
  return 0;
}
