// FP64 pipe microbenchmarks for sm_100a: SIMT DFMA vs DMMA (mma.sync m8n8k4 f64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double *out, int iters, double a0, double b0) {
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = threadIdx.x; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16_kernel(double *out, int iters, double a0, double b0) {
  // m16n8k16 f64: A 8 regs? (16x16 = 256 / 32 = 8), B 4 (16x8=128/32), C 4 (16x8=128/32)
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = threadIdx.x; c[i][2] = 0; c[i][3] = 1; }
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 - (threadIdx.x + i) * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz l2 %d MB smem/blk optin %zu\n", p.name, p.multiProcessorCount,
         p.clockRate, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  double *out; cudaMalloc(&out, 8);
  int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      if (threads * bps > 2048) continue;
      int iters = 20000;
      float ms = time_it([&] { dfma_kernel<8><<<sms * bps, threads>>>(out, iters, 1.0000001, 1e-7); });
      double flops = 2.0 * 8 * iters * (double)threads * sms * bps;
      printf("DFMA  chains=8 threads=%d blk/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 5000;
      float ms = time_it([&] { dmma_kernel<8><<<sms * bps, threads>>>(out, iters, 1.0000001, 1e-7); });
      double flops = 2.0 * 256 * 8 * iters * (double)(threads / 32) * sms * bps;
      printf("DMMA m8n8k4 chains=8 threads=%d blk/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  for (int threads : {128, 256}) {
    for (int bps : {1, 2, 4}) {
      int iters = 2000;
      float ms = time_it([&] { dmma16_kernel<4><<<sms * bps, threads>>>(out, iters, 1.0000001, 1e-7); });
      double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)(threads / 32) * sms * bps;
      printf("DMMA m16n8k16 chains=4 threads=%d blk/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
