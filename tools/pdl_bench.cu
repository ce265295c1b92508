// Microbenchmark: per-kernel cost of a chain of small dependent kernels in a
// CUDA graph, with and without programmatic dependent launch (PDL).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/pdl_bench tools/pdl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(float* a, int n, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = a[i] * 1.0001f + 1.0f;
}

int main() {
  const int n = 1 << 20, chain = 30, reps = 200;
  float* a;
  cudaMalloc(&a, n * sizeof(float));
  cudaMemset(a, 0, n * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int blocks : {148, 1024, 4096}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < chain; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_small, a, blocks * 256 < n ? blocks * 256 : n, pdl);
      }
      cudaStreamEndCapture(s, &g);
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
      for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("pdl=%d blocks=%5d: %.2f us per kernel\n", pdl, blocks, 1e3f * ms / (reps * chain));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
