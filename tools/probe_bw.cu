// probe_bw.cu -- HBM ceilings for the PCG path's access mixes on one B200:
// pure streaming reads (8 B and 16 B per thread per load, evict-first), the
// copy the driver's MEASURED_PEAKS uses (read + write), and a read-mostly mix
// (12 B streamed + 16 B gathered from a resident window per 8 B written,
// like the S phase: values + column index, z/p gathers, q write).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_bw.cu -o /tmp/pbw && /tmp/pbw
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(512) rd8(const double* __restrict__ a, size_t n, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += __ldcs(a + i);
  if (s == 1.2345) out[0] = s;
}
__global__ void __launch_bounds__(512) rd16(const double2* __restrict__ a, size_t n2, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
// unrolled: 4 independent 16 B loads in flight per thread
__global__ void __launch_bounds__(512) rd16x4(const double2* __restrict__ a, size_t n2, double* out) {
  double s = 0.0;
  const size_t st = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * st < n2; i += 4 * st) {
    double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + st), v2 = __ldcs(a + i + 2 * st), v3 = __ldcs(a + i + 3 * st);
    s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n2; i += st) { double2 v = __ldcs(a + i); s += v.x + v.y; }
  if (s == 1.2345) out[0] = s;
}
__global__ void __launch_bounds__(512) cpy(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}
// S-phase-like: per row 15 slots of (8 B value, 4 B col) streamed in SELL-32
// order, gathers of two vectors at col (banded window), one 8 B write per row.
__global__ void __launch_bounds__(512) sell(const double* __restrict__ A, const int* __restrict__ col,
                                            const double* __restrict__ z, const double* __restrict__ p,
                                            double* __restrict__ q, int nslices, int w) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nslices; s += nw) {
    const size_t base = (size_t)s * w * 32;
    double sum = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) {
      const size_t t = base + (size_t)k * 32 + lane;
      const int c = __ldcs(col + t);
      sum += __ldcs(A + t) * (z[c] + 0.5 * p[c]);
    }
    q[(size_t)s * 32 + lane] = sum;
  }
}

// Slot pairs: lane holds slots (2j, 2j+1) of its row contiguously -> 16 B value
// loads and 8 B index loads; odd tail slot plain.  MINB: CTAs/SM bound.
template <int MINB, bool ZP>
__global__ void __launch_bounds__(512, MINB) sell2(const double* __restrict__ A, const int* __restrict__ col,
                                            const double* __restrict__ z, const double* __restrict__ p,
                                            const double2* __restrict__ zp,
                                            double* __restrict__ q, int nslices, int w) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int np = w >> 1;
  for (int s = gw; s < nslices; s += nw) {
    const size_t base = (size_t)s * w * 32;
    const double2* A2 = reinterpret_cast<const double2*>(A + base);
    const int2* C2 = reinterpret_cast<const int2*>(col + base);
    double sum = 0.0;
#pragma unroll 2
    for (int j = 0; j < np; ++j) {
      const double2 av = __ldcs(A2 + j * 32 + lane);
      const int2 c = __ldcs(C2 + j * 32 + lane);
      if (ZP) {
        const double2 g0 = zp[c.x], g1 = zp[c.y];
        sum += av.x * (g0.x + 0.5 * g0.y);
        sum += av.y * (g1.x + 0.5 * g1.y);
      } else {
        sum += av.x * (z[c.x] + 0.5 * p[c.x]);
        sum += av.y * (z[c.y] + 0.5 * p[c.y]);
      }
    }
    if (w & 1) {
      const size_t t = base + (size_t)np * 64 + lane;
      const int c = __ldcs(col + t);
      if (ZP) { const double2 g = zp[c]; sum += __ldcs(A + t) * (g.x + 0.5 * g.y); }
      else sum += __ldcs(A + t) * (z[c] + 0.5 * p[c]);
    }
    q[(size_t)s * 32 + lane] = sum;
  }
}
template <int MINB>
__global__ void __launch_bounds__(512, MINB) sell1(const double* __restrict__ A, const int* __restrict__ col,
                                            const double* __restrict__ z, const double* __restrict__ p,
                                            double* __restrict__ q, int nslices, int w) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nslices; s += nw) {
    const size_t base = (size_t)s * w * 32;
    double sum = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) {
      const size_t t = base + (size_t)k * 32 + lane;
      const int c = __ldcs(col + t);
      sum += __ldcs(A + t) * (z[c] + 0.5 * p[c]);
    }
    q[(size_t)s * 32 + lane] = sum;
  }
}

// Full S phase of Algorithm 1 as a standalone kernel: per row p = z + beta pold,
// deferred x += alpha pold, q = A p (gathers of z and pold), pnew / q / x
// writes and a per-CTA p.q partial.  PAIRS: slot-pair layout (16-byte values).
template <int MINB, bool PAIRS>
__global__ void __launch_bounds__(512, MINB) sfull(const double* __restrict__ A, const int* __restrict__ col,
    const double* __restrict__ z, const double* __restrict__ pold, double* __restrict__ pnew,
    double* __restrict__ x, double* __restrict__ q, double* __restrict__ part, int nslices, int w,
    double alpha, double beta) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int s = gw; s < nslices; s += nw) {
    const size_t base = (size_t)s * w * 32;
    const size_t i = (size_t)s * 32 + lane;
    const double po = pold[i];
    const double pi = z[i] + beta * po;
    x[i] = x[i] + alpha * po;
    double sum = 0.0;
    if (PAIRS) {
      const double2* A2 = reinterpret_cast<const double2*>(A + base) + lane;
      const int2* C2 = reinterpret_cast<const int2*>(col + base) + lane;
#pragma unroll 2
      for (int j = 0; j < (w >> 1); ++j) {
        const double2 av = __ldcs(A2 + 32 * j);
        const int2 c = __ldcs(C2 + 32 * j);
        sum += av.x * (z[c.x] + beta * pold[c.x]);
        sum += av.y * (z[c.y] + beta * pold[c.y]);
      }
      if (w & 1) {
        const size_t t = base + 32 * (size_t)(w - 1) + lane;
        const int c = __ldcs(col + t);
        sum += __ldcs(A + t) * (z[c] + beta * pold[c]);
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < w; ++k) {
        const size_t t = base + (size_t)k * 32 + lane;
        const int c = __ldcs(col + t);
        sum += __ldcs(A + t) * (z[c] + beta * pold[c]);
      }
    }
    pnew[i] = pi;
    q[i] = sum;
    acc += pi * sum;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double sh[16];
  if (lane == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}

__global__ void fill_col(int* col, int nslices, int w, int n, int band) {
  size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t tot = (size_t)nslices * w * 32;
  for (; t < tot; t += (size_t)gridDim.x * blockDim.x) {
    const size_t s = t / ((size_t)w * 32), k = (t / 32) % w, lane = t % 32;
    long row = (long)s * 32 + lane;
    const int offs[15] = {0, 1, -1, 200, -200, 201, -199, 50000, -50000, 50001, -49999, 50200, -50200, 50201, -50201};
    long c = row + offs[k % 15];
    if (c < 0) c = 0;
    if (c >= n) c = n - 1;
    col[t] = (int)c;
  }
}

template <class F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const size_t bytes = (size_t)4 << 30;  // 4 GiB >> L2
  double *a, *b, *out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  cudaMemset(b, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = bytes / 8;
  for (int per : {2, 4, 8}) {
    const int g = sms * per;
    float t1 = timeit([&] { rd8<<<g, 512>>>(a, n, out); }, 10);
    float t2 = timeit([&] { rd16<<<g, 512>>>((double2*)a, n / 2, out); }, 10);
    float t3 = timeit([&] { rd16x4<<<g, 512>>>((double2*)a, n / 2, out); }, 10);
    float t4 = timeit([&] { cpy<<<g, 512>>>((double2*)a, (double2*)b, n / 4); }, 10);  // 2 GiB each way
    printf("grid %d x 512: read8 %.0f GB/s  read16 %.0f GB/s  read16x4 %.0f GB/s  copy %.0f GB/s\n", g,
           bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6, bytes / t4 / 1e6);
  }
  // S-phase-like mix at 20 M rows, 15 slots
  const int nrows = 20000000, w = 15, nsl = nrows / 32;
  double *A, *z, *p, *q;
  int* col;
  cudaMalloc(&A, (size_t)nsl * w * 32 * 8);
  cudaMalloc(&col, (size_t)nsl * w * 32 * 4);
  cudaMalloc(&z, (size_t)nrows * 8);
  cudaMalloc(&p, (size_t)nrows * 8);
  cudaMalloc(&q, (size_t)nrows * 8);
  cudaMemset(A, 0, (size_t)nsl * w * 32 * 8);
  cudaMemset(z, 0, (size_t)nrows * 8);
  cudaMemset(p, 0, (size_t)nrows * 8);
  fill_col<<<sms * 8, 512>>>(col, nsl, w, nrows, 0);
  double2* zp;
  cudaMalloc(&zp, (size_t)nrows * 16);
  cudaMemset(zp, 0, (size_t)nrows * 16);
  const double alg = (double)nsl * 32 * (w * 12.0 + 8 + 16);  // matrix + q write + z,p once
  auto rep = [&](const char* name, float t) { printf("%-28s %.3f ms  %.0f GB/s algorithmic\n", name, t, alg / t / 1e6); };
  double *pold, *pnew, *x, *part;
  cudaMalloc(&pold, (size_t)nrows * 8); cudaMalloc(&pnew, (size_t)nrows * 8); cudaMalloc(&x, (size_t)nrows * 8);
  cudaMalloc(&part, 8192 * 8);
  cudaMemset(pold, 0, (size_t)nrows * 8); cudaMemset(x, 0, (size_t)nrows * 8);
  const double algS = (double)nsl * 32 * (w * 12.0 + 48);  // matrix + z, pold, x r/w, pnew, q (S phase bytes)
  auto repS = [&](const char* name, float t) { printf("%-28s %.3f ms  %.0f GB/s (S-phase bytes)\n", name, t, algS / t / 1e6); };
  repS("S full plain minb4", timeit([&] { sfull<4, false><<<sms * 4, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  repS("S full pairs minb4", timeit([&] { sfull<4, true><<<sms * 4, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  repS("S full plain minb3", timeit([&] { sfull<3, false><<<sms * 3, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  repS("S full pairs minb3", timeit([&] { sfull<3, true><<<sms * 3, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  repS("S full plain minb2", timeit([&] { sfull<2, false><<<sms * 2, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  repS("S full pairs minb2", timeit([&] { sfull<2, true><<<sms * 2, 512>>>(A, col, z, pold, pnew, x, q, part, nsl, w, 0.5, 0.25); }, 10));
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
