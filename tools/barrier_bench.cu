// Microbenchmark: latency of grid-wide reductions (sum of one double per CTA,
// result needed by every CTA) for several barrier designs on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0: counter + __threadfence (fence.sc)   mode 1: red.release + ld.acquire
// mode 2: per-CTA flags (all-to-all)            mode 3: cg grid.sync()
// mode 4: counter release/acquire, partials padded to 128 B lines
__global__ void k_bench(int mode, int iters, unsigned* bar, unsigned* flags, double* partials,
                        double* out) {
  __shared__ double s;
  double acc = 0.0;
  unsigned epoch = 0;
  const int n = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    double mine = 1.0 + blockIdx.x * 1e-3 + it;
    int par = it & 1;
    if (mode == 3) {
      if (threadIdx.x == 0) partials[par * 256 + blockIdx.x] = mine;
      cg::this_grid().sync();
      if (threadIdx.x < 32) {
        double x = 0;
        for (int c = threadIdx.x; c < n; c += 32) x += __ldcg(&partials[par * 256 + c]);
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
        if (threadIdx.x == 0) s = x;
      }
      __syncthreads();
      acc += s;
      continue;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int stride = (mode == 4) ? 16 : 1;
      double* part = partials + par * 256 * 16;
      if (lane == 0) part[blockIdx.x * stride] = mine;
      ++epoch;
      if (mode == 0) {
        if (lane == 0) {
          __threadfence();
          atomicAdd(bar, 1u);
          while (*(volatile unsigned*)bar < epoch * n) {
          }
          __threadfence();
        }
        __syncwarp();
      } else if (mode == 1 || mode == 4) {
        if (lane == 0) {
          red_release(bar, 1u);
          while (ld_acquire(bar) < epoch * n) {
          }
        }
        __syncwarp();
      } else if (mode == 2) {
        if (lane == 0) st_release(&flags[par * 256 + blockIdx.x], epoch);
        for (int c = lane; c < n; c += 32)
          while (ld_acquire(&flags[par * 256 + c]) < epoch) {
          }
        __syncwarp();
      }
      double x = 0;
      for (int c = lane; c < n; c += 32) x += __ldcg(&part[c * stride]);
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
      if (lane == 0) s = x;
    }
    __syncthreads();
    acc += s;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

int main() {
  unsigned *bar, *flags;
  double *partials, *out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&flags, 4 * 512);
  cudaMalloc(&partials, 8 * 256 * 16 * 2);
  cudaMalloc(&out, 8);
  const char* names[] = {"counter+fence", "counter rel/acq", "flags all-to-all", "cg grid.sync",
                         "counter rel/acq pad"};
  int ctas_list[] = {8, 16, 32, 64, 96, 148};
  for (int mode = 0; mode < 5; ++mode) {
    for (int ci = 0; ci < 6; ++ci) {
      int ctas = ctas_list[ci];
      int iters = 2000;
      cudaMemset(bar, 0, 4);
      cudaMemset(flags, 0, 4 * 512);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      void* args[] = {&mode, &iters, &bar, &flags, &partials, &out};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_bench, ctas, 512, args, 0, 0);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-22s ctas=%4d  %7.3f us/reduction %s\n", names[mode], ctas, 1e3 * ms / iters,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
