// probe_cluster_barrier.cu -- cost of one cluster-wide barrier on this GPU, by
// cluster size and flavour (DESIGN.md "Cluster engine" measurements).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_cluster_barrier.cu -o /tmp/pcb && /tmp/pcb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void bar_kernel(int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[16];
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      cl.sync();  // arrive (release) + wait (acquire)
    } else if (MODE == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    } else if (MODE == 2) {  // reduction pattern: DSMEM store + cluster barrier + read
      if (threadIdx.x < cl.num_blocks()) {
        double* d = cl.map_shared_rank(&slot[cl.block_rank()], threadIdx.x);
        *d = (double)i;
      }
      cl.sync();
      acc += slot[(i + threadIdx.x) & 15 % cl.num_blocks()];
    } else {  // CTA barrier only
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

template <int MODE>
float run(int C, int threads, int iters) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(bar_kernel<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, bar_kernel<MODE>, 10, out);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, bar_kernel<MODE>, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaFree(out);
  return ms * 1e3f / iters;  // us per barrier
}

int main() {
  const int iters = 20000;
  printf("C threads  cl.sync_us  relaxed_us  dsmem_reduce_us  syncthreads_us\n");
  for (int C : {1, 2, 4, 8, 16})
    for (int t : {256, 512})
      printf("%2d %4d  %8.3f  %8.3f  %8.3f  %8.3f\n", C, t, run<0>(C, t, iters), run<1>(C, t, iters),
             run<2>(C, t, iters), run<3>(C, t, iters));
  return 0;
}
