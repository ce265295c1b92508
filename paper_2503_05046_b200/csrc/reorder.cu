// Once-per-step particle reordering by (sparse block, cell) on sm_100a.
//
// The reference keeps particles in input order and sorts a 10-bit truncated
// Morton key only as a reduction plan (transfer.py:85-102).  On the GPU the
// fused substep instead works on a sim-internal copy of the particle state
// sorted by the key  block_index * 64 + cell_in_block  (block_index = rank of
// the block key in the sorted sparse grid, grid.py:97), so that
//   * the particles of one grid cell are contiguous: their contacts form runs
//     with identical stencils (the solver's contact groups), and
//   * the particles of one 4^3 block are contiguous: P2G/G2P stencils of a
//     warp touch few blocks and the loads of particle state coalesce.
// Particles move by a small fraction of a cell per coupling step, so the
// order stays nearly sorted across the N substeps; it is rebuilt every step.
//
// Sort: stable LSD radix sort, 8-bit digits, as many passes as the key needs.
// Each pass: per-warp-tile digit histograms -> bucket-major exclusive scan ->
// stable scatter with __match_any_sync ranks (the same scheme as the
// bit-exact sort plan in binning.cu).  Stable + deterministic.
#include "common.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

constexpr int kRWarps = 8;
constexpr int kRTile = 1024;   // elements per warp tile
constexpr int kRBuckets = 256;

__global__ void k_sort_keys(const double* __restrict__ x, long long n, double h,
                            const unsigned long long* __restrict__ hkeys,
                            const int* __restrict__ hvals, unsigned mask,
                            unsigned* __restrict__ keys, int* __restrict__ vals, DevStatus* st) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int64_t b[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a] = base_cell(x[3 * i + a], h);
    int64_t key;
    int blk = -1;
    if (pack_block(b[0] >> 2, b[1] >> 2, b[2] >> 2, &key))
      blk = hash_find(hkeys, hvals, mask, (uint64_t)key);
    if (blk < 0) {
      raise_status(st, MPMRB_E_ALLOCATION, 70, i);
      blk = 0;
    }
    keys[i] = ((unsigned)blk << 6) | (unsigned)(((b[0] & 3) << 4) | ((b[1] & 3) << 2) | (b[2] & 3));
    vals[i] = (int)i;
  }
}

__global__ void __launch_bounds__(kRWarps * 32) k_radix_hist(const unsigned* __restrict__ keys,
                                                            long long n, int shift, int ntiles,
                                                            int* __restrict__ th) {
  __shared__ int hist[kRWarps][kRBuckets];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = lane; b < kRBuckets; b += 32) hist[wid][b] = 0;
  __syncwarp();
  const int tile = blockIdx.x * kRWarps + wid;
  if (tile >= ntiles) return;
  const long long base = (long long)tile * kRTile;
  for (int r = 0; r < kRTile; r += 32) {
    const long long i = base + r + lane;
    if (i < n) atomicAdd(&hist[wid][(keys[i] >> shift) & (kRBuckets - 1)], 1);
  }
  __syncwarp();
  for (int b = lane; b < kRBuckets; b += 32) th[(long long)b * ntiles + tile] = hist[wid][b];
}

__global__ void __launch_bounds__(kRWarps * 32) k_radix_scatter(
    const unsigned* __restrict__ kin, const int* __restrict__ vin, long long n, int shift,
    int ntiles, const int* __restrict__ scanned, unsigned* __restrict__ kout,
    int* __restrict__ vout) {
  __shared__ int run[kRWarps][kRBuckets];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tile = blockIdx.x * kRWarps + wid;
  if (tile >= ntiles) return;
  for (int b = lane; b < kRBuckets; b += 32) run[wid][b] = scanned[(long long)b * ntiles + tile];
  __syncwarp();
  const long long base = (long long)tile * kRTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRTile; r += 32) {
    const long long i = base + r + lane;
    const bool valid = i < n;
    const unsigned key = valid ? kin[i] : 0u;
    const unsigned d = valid ? ((key >> shift) & (kRBuckets - 1)) : (0x1000u + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & lt);
    int pos = 0;
    if (valid) pos = run[wid][d] + rank;
    __syncwarp();
    if (valid && rank == 0) run[wid][d] += __popc(peers);
    __syncwarp();
    if (valid) {
      kout[pos] = key;
      vout[pos] = vin[i];
    }
  }
}

// dst[i] = src[perm[i]] for W doubles per particle
template <int W>
__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ perm, long long n,
                         double* __restrict__ dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * W;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W, k = e - i * W;
    dst[e] = src[(long long)perm[i] * W + k];
  }
}
template <int W>
__global__ void k_scatter_back(const double* __restrict__ src, const int* __restrict__ perm,
                               long long n, double* __restrict__ dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * W;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W, k = e - i * W;
    dst[(long long)perm[i] * W + k] = src[e];
  }
}
// float64 user arrays <-> float32 sim-internal copy (fp32 performance mode)
template <int W>
__global__ void k_gather_f32(const double* __restrict__ src, const int* __restrict__ perm,
                             long long n, float* __restrict__ dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * W;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W, k = e - i * W;
    dst[e] = (float)src[(long long)perm[i] * W + k];
  }
}
template <int W>
__global__ void k_scatter_back_f32(const float* __restrict__ src, const int* __restrict__ perm,
                                   long long n, double* __restrict__ dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * W;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / W, k = e - i * W;
    dst[(long long)perm[i] * W + k] = (double)src[e];
  }
}
__global__ void k_gather_i64(const long long* __restrict__ src, const int* __restrict__ perm,
                             long long n, long long* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}
__global__ void k_map_ids(const int* __restrict__ ids, const int* __restrict__ perm,
                          const int* __restrict__ n_dev, long long cap, int* __restrict__ out) {
  const long long n = *n_dev < cap ? *n_dev : cap;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = perm[ids[i]];
}

unsigned gs_grid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

}  // namespace

// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of the
// keys.  Ping-pongs between (ka, va) and (kb, vb); the final values go to
// vals_out (which may alias neither input) and the final keys to *keys_out.
int sort_pairs_u32(Ctx& c, unsigned* ka, int* va, unsigned* kb, int* vb, long long n, int bits,
                   int* vals_out, unsigned** keys_out) {
  const int passes = bits <= 0 ? 1 : (bits + 7) / 8;
  const int ntiles = (int)((n + kRTile - 1) / kRTile);
  const long long hist_n = (long long)kRBuckets * ntiles;
  if (c.scratch[SS_HIST].grow(sizeof(int) * hist_n) || c.scratch[SS_TMP0].grow(sizeof(int) * hist_n))
    return MPMRB_E_CUDA;
  int* th = c.scratch[SS_HIST].as<int>();
  int* scanned = c.scratch[SS_TMP0].as<int>();
  const unsigned cta = (unsigned)((ntiles + kRWarps - 1) / kRWarps);
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_radix_hist<<<cta, kRWarps * 32, 0, c.stream>>>(ka, n, shift, ntiles, th);
    int rc = scan_exclusive_i32(c, th, scanned, hist_n, nullptr, nullptr, c.scratch[SS_TILE]);
    if (rc) return rc;
    const bool last = p == passes - 1;
    k_radix_scatter<<<cta, kRWarps * 32, 0, c.stream>>>(ka, va, n, shift, ntiles, scanned, kb,
                                                        last ? vals_out : vb);
    c.launches += 2;
    unsigned* tk = ka;
    ka = kb;
    kb = tk;
    int* tv = va;
    va = vb;
    vb = tv;
  }
  if (keys_out) *keys_out = ka;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_particle_sort(Ctx& c, const double* x, long long n, double h,
                         const unsigned long long* hkeys, const int* hvals, long long hash_cap,
                         long long n_blocks_cap, unsigned* keys2, int* vals2, int* perm_out) {
  if (n == 0) return MPMRB_OK;
  const unsigned mask = (unsigned)(hash_cap - 1);
  unsigned* ka = keys2;
  unsigned* kb = keys2 + n;
  int* va = vals2;
  int* vb = vals2 + n;
  k_sort_keys<<<gs_grid(n, 256), 256, 0, c.stream>>>(x, n, h, hkeys, hvals, mask, ka, va,
                                                     c.status);
  c.launches++;
  int bits = 6;
  while ((1LL << (bits - 6)) < n_blocks_cap) ++bits;
  return sort_pairs_u32(c, ka, va, kb, vb, n, bits, perm_out, nullptr);
}

int launch_particle_gather(Ctx& c, const int* perm, long long n, const double* src, int width,
                           double* dst) {
  if (n == 0) return MPMRB_OK;
  switch (width) {
    case 1: k_gather<1><<<gs_grid(n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 3: k_gather<3><<<gs_grid(3 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 9: k_gather<9><<<gs_grid(9 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    default: return set_error(MPMRB_E_INVALID, "gather width %d", width);
  }
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_particle_scatter(Ctx& c, const int* perm, long long n, const double* src, int width,
                            double* dst) {
  if (n == 0) return MPMRB_OK;
  switch (width) {
    case 1: k_scatter_back<1><<<gs_grid(n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 3: k_scatter_back<3><<<gs_grid(3 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 9: k_scatter_back<9><<<gs_grid(9 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    default: return set_error(MPMRB_E_INVALID, "scatter width %d", width);
  }
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_particle_gather_f32(Ctx& c, const int* perm, long long n, const double* src, int width,
                               float* dst) {
  if (n == 0) return MPMRB_OK;
  switch (width) {
    case 1: k_gather_f32<1><<<gs_grid(n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 3: k_gather_f32<3><<<gs_grid(3 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 9: k_gather_f32<9><<<gs_grid(9 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    default: return set_error(MPMRB_E_INVALID, "gather width %d", width);
  }
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_particle_scatter_f32(Ctx& c, const int* perm, long long n, const float* src, int width,
                                double* dst) {
  if (n == 0) return MPMRB_OK;
  switch (width) {
    case 1: k_scatter_back_f32<1><<<gs_grid(n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 3: k_scatter_back_f32<3><<<gs_grid(3 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    case 9: k_scatter_back_f32<9><<<gs_grid(9 * n, 256), 256, 0, c.stream>>>(src, perm, n, dst); break;
    default: return set_error(MPMRB_E_INVALID, "scatter width %d", width);
  }
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_gather_i64(Ctx& c, const int* perm, long long n, const long long* src, long long* dst) {
  if (n == 0) return MPMRB_OK;
  k_gather_i64<<<gs_grid(n, 256), 256, 0, c.stream>>>(src, perm, n, dst);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_map_ids(Ctx& c, const int* ids, const int* perm, const int* n_dev, long long cap,
                   int* out) {
  k_map_ids<<<gs_grid(cap, 256), 256, 0, c.stream>>>(ids, perm, n_dev, cap, out);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace mpmrb
