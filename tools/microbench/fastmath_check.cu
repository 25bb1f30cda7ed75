// Max ulp error of fast_rcp / fast_sqrt (internal.cuh) against the IEEE routines over random
// positive doubles spanning 2^-300 .. 2^300.   nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../../paper_1811_09334_b200/csrc/internal.cuh"

__global__ void check(uint64_t n, unsigned long long *worst) {
  unsigned long long wr = 0, ws = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const int ex = (int)(z % 600) - 300;
    const double m = 1.0 + (double)(z >> 12) * 0x1p-52;
    const double x = ldexp(m, ex);
    const double r0 = 1.0 / x, r1 = rqlpk::fast_rcp(x);
    const double s0 = sqrt(x), s1 = rqlpk::fast_sqrt(x);
    long long dr = (long long)__double_as_longlong(r0) - (long long)__double_as_longlong(r1);
    long long ds = (long long)__double_as_longlong(s0) - (long long)__double_as_longlong(s1);
    wr = max(wr, (unsigned long long)llabs(dr));
    ws = max(ws, (unsigned long long)llabs(ds));
  }
  atomicMax(&worst[0], wr);
  atomicMax(&worst[1], ws);
}

int main() {
  unsigned long long *w;
  cudaMallocManaged(&w, 16);
  w[0] = w[1] = 0;
  check<<<592, 256>>>(1ull << 28, w);
  cudaDeviceSynchronize();
  printf("fast_rcp max ulp %llu, fast_sqrt max ulp %llu over 2^28 samples\n", w[0], w[1]);
  return 0;
}
