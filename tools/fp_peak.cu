// Non-tensor FP64 / FP32 FMA throughput of this B200 (the compute roof of the
// transfer kernels, which are float64 CUDA-core work, not tensor-core work).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/fp_peak tools/fp_peak.cu
//   tools/bin/fp_peak            -> one JSON line
//
// Each thread runs kChains independent FMA chains (enough ILP to hide the
// pipeline latency), the grid is a multiple of the SM count, and the result is
// stored so the compiler keeps the work.  2 flop per FMA.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <typename T>
__global__ void k_fma(T* out, T a, T b) {
  T acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = acc[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename T>
double run(int sms) {
  const int threads = 256, blocks = sms * 8;
  T* out;
  cudaMalloc(&out, sizeof(T) * threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fma<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_fma<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  const double flop = 2.0 * kChains * (double)kIters * threads * blocks;
  return flop / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const double f64 = run<double>(sms);
  const double f32 = run<float>(sms);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_fma_tflops\": %.3f, \"fp32_fma_tflops\": %.3f, "
         "\"max_sm_clock_mhz\": %.0f, \"how\": \"best of 10 launches, %d blocks x 256 threads, "
         "%d independent FMA chains x %d iterations per thread, 2 flop per FMA\"}\n",
         prop.name, sms, f64, f32, clk / 1e3, sms * 8, kChains, kIters);
  return 0;
}
