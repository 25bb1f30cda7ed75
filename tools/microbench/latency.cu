// Latency microbenchmarks on sm_100a: dependent DFMA / DP sqrt / DP div chains, warp shuffle
// reduction, __syncthreads (1024 threads), globaltimer resolution.  One CTA, clock64 cycles.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, double x0, int iters) {
  double x = x0 + threadIdx.x * 1e-12;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 1.0000001, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // div chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 0.5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // warp_sum (5 xor shuffles of doubles)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    x *= 1e-3;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    x += 1e-12;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // shared-memory round trip (store by thread 0, sync, load by all)
  __shared__ double sh;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) sh = x;
    __syncthreads();
    x = sh * 0.999 + 1e-9;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // globaltimer granularity
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); } while (g1 == g0);
  if (threadIdx.x == 0) cyc[6] = (long long)(g1 - g0);
  out[threadIdx.x] = x;
}

// L2 round trip: volatile load of a line written by this thread after a fence.
__global__ void l2lat(volatile unsigned long long *p, long long *cyc, int iters) {
  long long t0 = clock64();
  unsigned long long v = 0;
  for (int i = 0; i < iters; ++i) {
    v = p[v & 7];
  }
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / iters + (long long)(v & 1);
}

int main() {
  double *out; long long *cyc; unsigned long long *p;
  cudaMalloc(&out, 8192); cudaMalloc(&cyc, 64 * 8); cudaMalloc(&p, 4096);
  cudaMemset(p, 0, 4096);
  const char *names[] = {"DFMA dep", "DP sqrt dep", "DP div dep", "warp_sum(5 shfl f64)", "__syncthreads x1024thr",
                         "smem bcast + 2 syncs", "globaltimer step ns"};
  for (int threads : {32, 256, 1024}) {
    lat<<<1, threads>>>(out, cyc, 1.5, 2000);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost);
    printf("threads=%d:", threads);
    for (int i = 0; i < 7; ++i) printf("  %s=%lld", names[i], h[i]);
    printf("\n");
  }
  l2lat<<<1, 1>>>(p, cyc, 1000);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("volatile global load (L2) dep latency = %lld cycles\n", h);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
