// Launch gap of dependent tiny kernels in a CUDA graph, with and without programmatic
// dependent launch (PDL).   nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_gap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(double *x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0;
}

int main() {
  double *x;
  cudaMalloc(&x, 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int grid : {1, 148}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      const int N = 200;
      for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, tiny, x, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("pdl=%d grid=%3d: %.2f us per dependent kernel (%s)\n", pdl, grid, ms * 1e3 / (10 * N),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
