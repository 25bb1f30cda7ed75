// Cross-SM exchange latency on sm_100a, the CPQR engine's pattern without its work:
//  (a) ping-pong: CTA 0 and CTA 1 alternately store a step tag and spin on the other's word
//      (gpu-scope relaxed 8-byte accesses, the engine's record format);
//  (b) all-to-all: G CTAs each store a tagged word per step and poll all G words (a lane polls
//      words lane, lane + 32, ..., all loads in flight, re-polling the stale ones) -- the engine's
//      record exchange, i.e. a grid barrier made of tagged words.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange exchange.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_rel(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void pingpong(unsigned long long *w, int iters, long long *cyc) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x, other = 1 - me;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (me == 0) {
      st_rel(&w[0 * 16], i);
      while (ld_rel(&w[1 * 16]) != (unsigned long long)i) {}
    } else {
      while (ld_rel(&w[0 * 16]) != (unsigned long long)i) {}
      st_rel(&w[1 * 16], i);
    }
  }
  if (me == 0) cyc[0] = (clock64() - t0) / iters;
  (void)other;
}

__global__ void alltoall(unsigned long long *w, int iters, long long *cyc) {
  const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x;
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    const unsigned long long tag = (unsigned long long)i;
    unsigned long long *slot = w + (size_t)(i & 1) * 256 * 4;
    if (lane == 0) st_rel(&slot[b * 4], tag);
    unsigned pending = 0;
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < G) pending |= 1u << t;
    unsigned long long v[8];
    while (pending) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (pending & (1u << t)) v[t] = ld_rel(&slot[(lane + 32 * t) * 4]);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if ((pending & (1u << t)) && v[t] == tag) pending &= ~(1u << t);
    }
    __syncwarp();
  }
  if (b == 0 && lane == 0) cyc[0] = (clock64() - t0) / iters;
}

int main() {
  unsigned long long *w;
  long long *cyc, h;
  cudaMalloc(&w, 1 << 20);
  cudaMalloc(&cyc, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(w, 0, 1 << 20);
    pingpong<<<2, 32>>>(w, 20000, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ping-pong (2 CTAs): %lld cycles per round trip (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
    for (int G : {2, 16, 74, 148}) {
      if (G > sms) continue;
      cudaMemset(w, 0, 1 << 20);
      alltoall<<<G, 32>>>(w, 5000, cyc);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("all-to-all tagged exchange, G = %3d CTAs: %lld cycles per step (%s)\n", G, h,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
