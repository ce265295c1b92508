// Probe: can a kernel be launched cooperatively AND with clusters, and what do
// cluster-level DSMEM reductions cost versus grid syncs?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_coop_probe tools/cluster_coop_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_probe(int iters, int mode, double* out) {
  __shared__ double slot[2][8];
  cg::cluster_group cl = cg::this_cluster();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    if (mode == 0) {  // cluster reduce through DSMEM
      if (cl.block_rank() < 8 && blockIdx.x < cl.num_blocks()) {
        if (threadIdx.x == 0) slot[par][0] = 1.0 + it + cl.block_rank();
        cl.sync();
        if (threadIdx.x < 32) {
          double x = 0.0;
          if (threadIdx.x < cl.num_blocks()) {
            double* remote = cl.map_shared_rank(&slot[par][0], threadIdx.x);
            x = *remote;
          }
          for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
          if (threadIdx.x == 0) acc += x;
        }
        __syncthreads();
      }
    } else {  // grid sync
      cg::this_grid().sync();
      acc += 1.0;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  for (int cs : {8, 16}) {
    if (cs == 16)
      cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cfg.gridDim = dim3(cs);
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_probe, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, nclusters, cudaGetErrorString(e));
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(cs * nclusters);
    for (int mode = 0; mode < 2; ++mode) {
      int iters = 4000;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      e = cudaLaunchKernelEx(&cfg, k_probe, iters, mode, out);
      cudaEventRecord(b);
      cudaError_t e2 = cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("  grid=%d mode=%s launch=%s sync=%s  %.3f us/op\n", cs * nclusters,
             mode == 0 ? "cluster-reduce" : "grid-sync", cudaGetErrorString(e),
             cudaGetErrorString(e2), 1e3 * ms / iters);
    }
  }
  return 0;
}
