// Microbenchmark: latency of a grid-wide all-reduce of K doubles (every CTA
// needs the sum, summed in a fixed CTA order) for fence-free designs that use
// self-validating 64-bit words: each double is split into two 32-bit halves,
// each stored as (epoch << 32 | half) so a reader can tell a complete, current
// value from a stale one without any fence or flag ordering.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o reduce_bench tools/reduce_bench.cu
//
// mode 0: cg::this_grid().sync() + partials (baseline)
// mode 1: all-to-all self-validating slots, every CTA polls every CTA's slot
// mode 2: clusters of C: DSMEM reduce to the cluster leader, leaders publish
//         self-validating slots, every CTA polls the leaders' slots
// mode 3: cluster-only reduce (C CTAs total)
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int K = 2;
constexpr int kMaxCtas = 160;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void publish(unsigned long long* slot, const double* v, unsigned ep) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v[k]);
    st_relaxed(slot + 2 * k, ((unsigned long long)ep << 32) | (b >> 32));
    st_relaxed(slot + 2 * k + 1, ((unsigned long long)ep << 32) | (b & 0xffffffffull));
  }
}

// lane-parallel poll of n slots (2K words each); returns the K sums in fixed
// slot order (lane-strided partial sums, then a butterfly)
__device__ __forceinline__ void poll_sum(const unsigned long long* slots, int n, unsigned ep,
                                         double* out) {
  const int lane = threadIdx.x & 31;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int s = lane; s < n; s += 32) {
    unsigned long long w[2 * K];
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) {
        w[j] = ld_relaxed(slots + (size_t)s * 2 * K + j);
        ok &= (unsigned)(w[j] >> 32) == ep;
      }
    } while (!ok);
#pragma unroll
    for (int k = 0; k < K; ++k)
      acc[k] += __longlong_as_double((long long)(((w[2 * k] & 0xffffffffull) << 32) |
                                                 (w[2 * k + 1] & 0xffffffffull)));
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[k] += __shfl_xor_sync(~0u, acc[k], o);
    out[k] = acc[k];
  }
}

// all slots' words loaded in one batch per lane (up to kMaxPer slots/lane),
// re-polled until every tag is current
template <int kMaxPer>
__device__ __forceinline__ void poll_sum_batched(const unsigned long long* slots, int n,
                                                 unsigned ep, double* out) {
  const int lane = threadIdx.x & 31;
  unsigned long long w[kMaxPer][2 * K];
  bool ok;
  do {
    ok = true;
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r) {
      const int s = lane + 32 * r;
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) {
        w[r][j] = (s < n) ? ld_relaxed(slots + (size_t)s * 2 * K + j) : ((unsigned long long)ep << 32);
        ok &= (unsigned)(w[r][j] >> 32) == ep;
      }
    }
  } while (!__all_sync(~0u, ok));
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r)
      acc += __longlong_as_double((long long)(((w[r][2 * k] & 0xffffffffull) << 32) |
                                              (w[r][2 * k + 1] & 0xffffffffull)));
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
    out[k] = acc;
  }
}

// two-level arrival counters + per-CTA release flags (monotonic epochs)
__device__ unsigned g_sub[16 * 32];   // one counter per group of 16 CTAs, 128 B apart
__device__ unsigned g_root[32];
__device__ unsigned g_flag[160 * 32]; // one release flag per CTA, 128 B apart

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void tree_barrier(unsigned epoch) {
  __syncthreads();
  const int n = gridDim.x, grp = blockIdx.x >> 4, ng = (n + 15) >> 4;
  const int gsize = min(16, n - grp * 16);
  if (threadIdx.x == 0) {
    const unsigned old = atom_add_acqrel(&g_sub[grp * 32], 1u);
    if (old == epoch * gsize - 1) {
      const unsigned o2 = atom_add_acqrel(&g_root[0], 1u);
      if (o2 == epoch * ng - 1) {
        // the acq_rel atomic above ordered every prior arrival; relaxed
        // stores suffice for the flags (readers acquire)
        for (int c = 0; c < n; ++c)
          asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&g_flag[c * 32]), "r"(epoch) : "memory");
      }
    }
    while (ld_acquire_u32(&g_flag[blockIdx.x * 32]) < epoch) {
    }
  }
  __syncthreads();
}

__global__ void k_bench(int mode, int iters, unsigned long long* slots, double* partials,
                        double* out) {
  __shared__ double s[K];
  __shared__ double cpart[K];
  double total = 0.0;
  const int n = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    const unsigned ep = (unsigned)it + 1u;
    double mine[K];
#pragma unroll
    for (int k = 0; k < K; ++k) mine[k] = 1.0 + blockIdx.x * 1e-3 + it + k;
    __syncthreads();
    if (mode == 6) {
      if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) partials[((it & 1) * K + k) * kMaxCtas + blockIdx.x] = mine[k];
      tree_barrier((unsigned)it + 1u);
      if (threadIdx.x < 32) {
        for (int k = 0; k < K; ++k) {
          double x = 0;
          for (int c = threadIdx.x; c < n; c += 32)
            x += __ldcg(&partials[((it & 1) * K + k) * kMaxCtas + c]);
          for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
          if (threadIdx.x == 0) s[k] = x;
        }
      }
    } else if (mode == 0) {
      if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) partials[((it & 1) * K + k) * kMaxCtas + blockIdx.x] = mine[k];
      cg::this_grid().sync();
      if (threadIdx.x < 32) {
        for (int k = 0; k < K; ++k) {
          double x = 0;
          for (int c = threadIdx.x; c < n; c += 32)
            x += __ldcg(&partials[((it & 1) * K + k) * kMaxCtas + c]);
          for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
          if (threadIdx.x == 0) s[k] = x;
        }
      }
    } else if (mode == 4) {
      // batched all-to-all
      unsigned long long* base = slots + (size_t)(it & 1) * kMaxCtas * 2 * K;
      if (threadIdx.x == 0) publish(base + (size_t)blockIdx.x * 2 * K, mine, ep);
      if (threadIdx.x < 32) {
        double r[K];
        poll_sum_batched<5>(base, n, ep, r);
        if (threadIdx.x == 0)
          for (int k = 0; k < K; ++k) s[k] = r[k];
      }
    } else if (mode == 5) {
      // two-level: groups of 16 publish to their leader's area; leaders sum
      // and publish to the top; everyone polls the top (<= 10 slots)
      unsigned long long* base = slots + (size_t)(it & 1) * kMaxCtas * 2 * K;
      unsigned long long* top = slots + (size_t)2 * kMaxCtas * 2 * K + (size_t)(it & 1) * 16 * 2 * K;
      const int grp = blockIdx.x / 16, ng = (n + 15) / 16;
      if (threadIdx.x == 0) publish(base + (size_t)blockIdx.x * 2 * K, mine, ep);
      if (threadIdx.x < 32) {
        double r[K];
        if ((blockIdx.x & 15) == 0) {
          const int cnt = min(16, n - grp * 16);
          poll_sum_batched<1>(base + (size_t)grp * 16 * 2 * K, cnt, ep, r);
          if (threadIdx.x == 0) publish(top + (size_t)grp * 2 * K, r, ep);
        }
        poll_sum_batched<1>(top, ng, ep, r);
        if (threadIdx.x == 0)
          for (int k = 0; k < K; ++k) s[k] = r[k];
      }
    } else if (mode == 1) {
      unsigned long long* base = slots + (size_t)(it & 1) * kMaxCtas * 2 * K;
      if (threadIdx.x == 0) publish(base + (size_t)blockIdx.x * 2 * K, mine, ep);
      if (threadIdx.x < 32) {
        double r[K];
        poll_sum(base, n, ep, r);
        if (threadIdx.x == 0)
          for (int k = 0; k < K; ++k) s[k] = r[k];
      }
    } else {
      cg::cluster_group cl = cg::this_cluster();
      const int crank = (int)cl.block_rank(), csz = (int)cl.num_blocks();
      if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) cpart[k] = mine[k];
      cl.sync();
      if (crank == 0 && threadIdx.x < 32) {
        double r[K];
        for (int k = 0; k < K; ++k) {
          double x = (threadIdx.x < csz) ? *cl.map_shared_rank(&cpart[k], threadIdx.x) : 0.0;
          for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
          r[k] = x;
        }
        if (mode == 3) {
          if (threadIdx.x == 0)
            for (int k = 0; k < K; ++k) s[k] = r[k];
        } else {
          const int cid = blockIdx.x / csz, ncl = n / csz;
          unsigned long long* base = slots + (size_t)(it & 1) * kMaxCtas * 2 * K;
          if (threadIdx.x == 0) publish(base + (size_t)cid * 2 * K, r, ep);
          poll_sum(base, ncl, ep, r);
          if (threadIdx.x == 0)
            for (int k = 0; k < K; ++k) s[k] = r[k];
        }
      }
      if (mode == 3 || crank != 0) {
        // followers: mode 2 polls leaders directly (no second cluster barrier)
        if (mode == 2 && threadIdx.x < 32) {
          const int ncl = n / csz;
          unsigned long long* base = slots + (size_t)(it & 1) * kMaxCtas * 2 * K;
          double r[K];
          poll_sum(base, ncl, ep, r);
          if (threadIdx.x == 0)
            for (int k = 0; k < K; ++k) s[k] = r[k];
        }
        if (mode == 3) {
          cl.sync();
          if (threadIdx.x < K) s[threadIdx.x] = *cl.map_shared_rank(&s[threadIdx.x], 0);
        }
      } else if (mode == 3) {
        cl.sync();
      }
    }
    __syncthreads();
    total += s[0] + s[K - 1];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = total;
}

int run(int mode, int ctas, int cluster, int threads, int iters, unsigned long long* slots,
        double* partials, double* out) {
  cudaMemset(slots, 0, sizeof(unsigned long long) * (2 * kMaxCtas + 32) * 2 * K);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_bench, mode, iters, slots, partials, out);
  cudaEventRecord(b);
  cudaError_t e2 = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  double h = 0;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("mode=%d ctas=%4d cluster=%2d threads=%4d  %7.3f us/reduction  %s %s\n", mode, ctas,
         cluster, threads, 1e3 * ms / iters, cudaGetErrorString(e), cudaGetErrorString(e2));
  cudaGetLastError();
  return 0;
}

int main() {
  unsigned long long* slots;
  double *partials, *out;
  cudaMalloc(&slots, sizeof(unsigned long long) * (2 * kMaxCtas + 32) * 2 * K);
  cudaMalloc(&partials, sizeof(double) * 2 * K * kMaxCtas);
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 4000;
  for (int threads : {256, 512}) {
    for (int ctas : {16, 64, 148}) run(0, ctas, 1, threads, iters, slots, partials, out);
    for (int ctas : {16, 64, 148}) {
      unsigned z[160 * 32] = {0};
      cudaMemcpyToSymbol(g_sub, z, sizeof(unsigned) * 16 * 32);
      cudaMemcpyToSymbol(g_root, z, sizeof(unsigned) * 32);
      cudaMemcpyToSymbol(g_flag, z, sizeof(unsigned) * 160 * 32);
      run(6, ctas, 1, threads, iters, slots, partials, out);
    }
    for (int ctas : {16, 64, 148}) run(1, ctas, 1, threads, iters, slots, partials, out);
    for (int ctas : {16, 32, 64, 148}) run(4, ctas, 1, threads, iters, slots, partials, out);
    for (int ctas : {32, 64, 148}) run(5, ctas, 1, threads, iters, slots, partials, out);
    for (int cl : {8, 16}) {
      int maxc = 0;
      cudaLaunchConfig_t q = {};
      q.blockDim = dim3(threads);
      q.gridDim = dim3(cl);
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = cl;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&maxc, (void*)k_bench, &q);
      printf("cluster %d threads %d: max active clusters %d (%s)\n", cl, threads, maxc,
             cudaGetErrorString(e));
      cudaGetLastError();
      if (maxc <= 0) continue;
      run(3, cl, cl, threads, iters, slots, partials, out);
      int one_per_sm = (148 / cl) * cl;
      if (maxc * cl < one_per_sm) one_per_sm = maxc * cl;
      run(2, one_per_sm, cl, threads, iters, slots, partials, out);
    }
  }
  return 0;
}
