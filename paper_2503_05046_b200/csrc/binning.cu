// Particle binning and the block-sparse grid on sm_100a.
//
//  * 10-bit truncated Morton sort plan (transfer.py:44-102): one-pass stable
//    counting sort over 1024 buckets.  Each warp owns a 1024-element tile:
//    per-warp histograms -> device scan (bucket-major) -> stable scatter with
//    __match_any_sync ranks.  perm / inv_perm / bins are bit-exact.
//  * Sparse grid (grid.py:71-122): candidate blocks of every stencil are
//    inserted into an open-addressing GPU hash table (warp-deduplicated
//    atomicCAS); the unique keys are bitonic-sorted in shared memory so block
//    indices equal the reference's sorted np.unique order; the sorted index is
//    stored back into the hash slot, so node lookup is one probe sequence.
#include <climits>

#include "common.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

constexpr int kPlanWarpTile = 1024;   // elements per warp tile
constexpr int kPlanWarps = 8;         // warps per CTA
constexpr int kBuckets = 1024;        // 2^10 Morton buckets

// Morton key from the low bits of the biased cell (transfer.py:44-61).  Only
// the low 10 interleaved bits survive, i.e. bits 0..3 of x and 0..2 of y, z;
// the 2^20 bias does not touch them.  Range check as transfer.py:58-59.
__device__ __forceinline__ bool morton10(int64_t cx, int64_t cy, int64_t cz, uint16_t* key) {
  int64_t x = cx + kBias21, y = cy + kBias21, z = cz + kBias21;
  if (x < 0 || y < 0 || z < 0 || x > kMask21 || y > kMask21 || z > kMask21) return false;
  uint32_t k = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    k |= (uint32_t)((x >> i) & 1) << (3 * i);
    if (3 * i + 1 < 10) k |= (uint32_t)((y >> i) & 1) << (3 * i + 1);
    if (3 * i + 2 < 10) k |= (uint32_t)((z >> i) & 1) << (3 * i + 2);
  }
  *key = (uint16_t)(k & 1023u);
  return true;
}

__global__ void k_base_cells(const double* __restrict__ x, long long n, double h,
                             long long* __restrict__ cells) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  cells[i] = base_cell(x[i], h);
}

__global__ void k_morton(const double* __restrict__ x, long long n, double h,
                         uint16_t* __restrict__ keys, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint16_t k;
  if (!morton10(base_cell(x[3 * i], h), base_cell(x[3 * i + 1], h), base_cell(x[3 * i + 2], h),
                &k)) {
    raise_status(st, MPMRB_E_INVALID, 1, i);
    k = 0;
  }
  keys[i] = k;
}

__global__ void __launch_bounds__(kPlanWarps * 32) k_plan_hist(const uint16_t* __restrict__ keys,
                                                               long long n, int ntiles,
                                                               int* __restrict__ th) {
  __shared__ int hist[kPlanWarps][kBuckets];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = lane; b < kBuckets; b += 32) hist[wid][b] = 0;
  __syncwarp();
  int tile = blockIdx.x * kPlanWarps + wid;
  if (tile >= ntiles) return;
  long long base = (long long)tile * kPlanWarpTile;
  for (int r = 0; r < kPlanWarpTile; r += 32) {
    long long i = base + r + lane;
    if (i < n) atomicAdd(&hist[wid][keys[i]], 1);
  }
  __syncwarp();
  for (int b = lane; b < kBuckets; b += 32) th[(long long)b * ntiles + tile] = hist[wid][b];
}

// bins from the bucket-major exclusive scan (transfer.py:91-101)
__global__ void __launch_bounds__(kBuckets) k_plan_bins(const int* __restrict__ scanned,
                                                        int ntiles, long long n,
                                                        uint16_t* __restrict__ bin_keys,
                                                        long long* __restrict__ bin_starts,
                                                        int* __restrict__ bucket_rank,
                                                        int* n_bins) {
  __shared__ int sm[32];
  const int b = threadIdx.x;
  long long start = scanned[(long long)b * ntiles];
  long long next = (b + 1 < kBuckets) ? scanned[(long long)(b + 1) * ntiles] : n;
  int nonempty = next > start ? 1 : 0;
  // block exclusive scan of nonempty
  int lane = b & 31, wid = b >> 5;
  int inc = nonempty;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = sm[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    sm[lane] = s;
  }
  __syncthreads();
  int rank = (wid ? sm[wid - 1] : 0) + inc - nonempty;
  bucket_rank[b] = rank;
  if (nonempty) {
    bin_keys[rank] = (uint16_t)b;
    bin_starts[rank] = start;
  }
  int total = sm[31];
  if (b == 0) {
    bin_starts[total] = n;
    *n_bins = total;
  }
}

__global__ void __launch_bounds__(kPlanWarps * 32) k_plan_scatter(
    const uint16_t* __restrict__ keys, long long n, int ntiles, const int* __restrict__ scanned,
    const int* __restrict__ bucket_rank, long long* __restrict__ perm,
    long long* __restrict__ inv_perm, long long* __restrict__ bin_of) {
  __shared__ int run[kPlanWarps][kBuckets];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int tile = blockIdx.x * kPlanWarps + wid;
  if (tile >= ntiles) return;
  for (int b = lane; b < kBuckets; b += 32) run[wid][b] = scanned[(long long)b * ntiles + tile];
  __syncwarp();
  long long base = (long long)tile * kPlanWarpTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kPlanWarpTile; r += 32) {
    long long i = base + r + lane;
    bool valid = i < n;
    unsigned key = valid ? keys[i] : (0x10000u + lane);  // unique dummies
    unsigned peers = __match_any_sync(0xffffffffu, key);
    int rank = __popc(peers & lt);
    int pos = 0;
    if (valid) pos = run[wid][key] + rank;
    __syncwarp();
    if (valid && rank == 0) run[wid][key] += __popc(peers);
    __syncwarp();
    if (valid) {
      perm[pos] = i;
      inv_perm[i] = pos;
      bin_of[i] = bucket_rank[key];
    }
  }
}

__global__ void k_staleness(const uint16_t* __restrict__ plan_keys, const double* __restrict__ x,
                            long long n, double h, unsigned long long* changed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned c = 0;
  if (i < n) {
    uint16_t k = 0;
    morton10(base_cell(x[3 * i], h), base_cell(x[3 * i + 1], h), base_cell(x[3 * i + 2], h), &k);
    c = (k != plan_keys[i]) ? 1u : 0u;
  }
  unsigned b = __ballot_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(changed, (unsigned long long)__popc(b));
}

// ----------------------------------------------------------------- grid build

__global__ void k_hash_clear(unsigned long long* __restrict__ hkeys, long long cap,
                             int* __restrict__ nb) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < cap) hkeys[i] = kEmptyKey;
  if (i == 0) *nb = 0;
}

// Insert the <=8 candidate blocks of each particle's stencil (grid.py:82-96).
__global__ void k_block_insert(const double* __restrict__ x, long long n, double h,
                               unsigned long long* __restrict__ hkeys, unsigned mask,
                               long long* __restrict__ ukeys, long long block_cap,
                               int* __restrict__ nb, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool valid = i < n;
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (valid) {
    double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    if (!(isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]))) {
      raise_status(st, MPMRB_E_ALLOCATION, 1, i);  // grid.py:77-78
      valid = false;
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int64_t b = base_cell(p[a], h);
        lo[a] = b >> 2;
        hi[a] = (b + 2) >> 2;
      }
    }
  }
  // Fast path: the warp's candidate blocks fit a 2x2x2 box of blocks (the
  // common case for particles sorted by (block, cell)).  Each lane marks the
  // box blocks its stencil touches, the warp ORs the marks, and lanes 0-7
  // insert the marked blocks: one round of <= 8 inserts instead of eight
  // rounds of match + probe.
  {
    int wlo[3], whi[3];
    bool box = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      wlo[a] = __reduce_min_sync(0xffffffffu, valid ? (int)lo[a] : INT_MAX);
      whi[a] = __reduce_max_sync(0xffffffffu, valid ? (int)hi[a] : INT_MIN);
      box &= whi[a] - wlo[a] <= 1;
    }
    if (box) {  // warp-uniform (also true when no lane is valid: nothing to insert)
      unsigned marks = 0;
      if (valid) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int ix = (c >> 2) & 1, iy = (c >> 1) & 1, iz = c & 1;
          if ((ix && hi[0] == lo[0]) || (iy && hi[1] == lo[1]) || (iz && hi[2] == lo[2]))
            continue;
          const int dx = (int)(ix ? hi[0] : lo[0]) - wlo[0];
          const int dy = (int)(iy ? hi[1] : lo[1]) - wlo[1];
          const int dz = (int)(iz ? hi[2] : lo[2]) - wlo[2];
          marks |= 1u << ((dx << 2) | (dy << 1) | dz);
        }
      }
      marks = __reduce_or_sync(0xffffffffu, marks);
      if (lane < 8 && ((marks >> lane) & 1u)) {
        int64_t key;
        if (!pack_block(wlo[0] + ((lane >> 2) & 1), wlo[1] + ((lane >> 1) & 1),
                        wlo[2] + (lane & 1), &key)) {
          raise_status(st, MPMRB_E_ALLOCATION, 2, i - lane);  // grid.py:29-30
        } else {
          const unsigned long long k = (unsigned long long)key;
          unsigned s = hash64(k) & mask;
          for (unsigned probe = 0; probe <= mask; ++probe) {
            const unsigned long long cur = hkeys[s];
            if (cur == k) break;
            if (cur == kEmptyKey) {
              const unsigned long long old = atomicCAS(&hkeys[s], kEmptyKey, k);
              if (old == kEmptyKey) {
                const int idx = atomicAdd(nb, 1);
                if (idx < block_cap) ukeys[idx] = (long long)k;
                else raise_status(st, MPMRB_E_CAPACITY, 1, idx + 1);
                break;
              }
              if (old == k) break;
            }
            s = (s + 1) & mask;
          }
        }
      }
      return;
    }
  }
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    int ix = (c >> 2) & 1, iy = (c >> 1) & 1, iz = c & 1;
    bool want = valid && !((ix && hi[0] == lo[0]) || (iy && hi[1] == lo[1]) ||
                           (iz && hi[2] == lo[2]));
    int64_t key = -1;
    if (want && !pack_block(ix ? hi[0] : lo[0], iy ? hi[1] : lo[1], iz ? hi[2] : lo[2], &key)) {
      raise_status(st, MPMRB_E_ALLOCATION, 2, i);  // grid.py:29-30
      want = false;
    }
    // warp dedupe: only the lowest lane of each equal-key group inserts
    unsigned long long k = want ? (unsigned long long)key : (kEmptyKey - 1 - lane);
    unsigned peers = __match_any_sync(0xffffffffu, k);
    bool leader = want && (__ffs(peers) - 1 == lane);
    if (!leader) continue;
    unsigned s = hash64(k) & mask;
    for (unsigned probe = 0; probe <= mask; ++probe) {
      unsigned long long cur = hkeys[s];
      if (cur == k) break;
      if (cur == kEmptyKey) {
        unsigned long long old = atomicCAS(&hkeys[s], kEmptyKey, k);
        if (old == kEmptyKey) {
          int idx = atomicAdd(nb, 1);
          if (idx < block_cap) ukeys[idx] = (long long)k;
          else raise_status(st, MPMRB_E_CAPACITY, 1, idx + 1);
          break;
        }
        if (old == k) break;
      }
      s = (s + 1) & mask;
    }
  }
}

// The sorted block order (grid.py:97, np.unique) by ranking: a key's sorted
// index is the number of smaller keys (keys are unique).  kRankLanes lanes
// share a key, each counting over a strided slice of the keys staged in shared
// memory, so the O(nb^2) comparisons spread over nb * kRankLanes threads (a
// single-CTA bitonic sort of ~2.7k keys took 42 us, latency-bound on its
// 78 barrier stages).  Also writes each key's sorted index into its hash slot.
constexpr int kRankLanes = 8;
constexpr int kRankTile = 2048;
__global__ void __launch_bounds__(256) k_block_rank_par(
    const long long* __restrict__ ukeys, const int* __restrict__ nb_dev, long long block_cap,
    long long* __restrict__ block_keys, const unsigned long long* __restrict__ hkeys,
    int* __restrict__ hvals, unsigned mask) {
  __shared__ long long tile[kRankTile];
  const int nb = *nb_dev;
  if (nb > block_cap) return;  // capacity error already raised by k_block_insert
  if ((long long)blockIdx.x * (256 / kRankLanes) >= nb) return;  // CTA-uniform
  const int t = blockIdx.x * 256 + threadIdx.x;
  const int i = t / kRankLanes, sub = t % kRankLanes;
  const long long key = i < nb ? ukeys[i] : LLONG_MAX;
  int rank = 0;
  for (int base = 0; base < nb; base += kRankTile) {
    __syncthreads();
    const int lim = min(kRankTile, nb - base);
    for (int q = threadIdx.x; q < lim; q += 256) tile[q] = ukeys[base + q];
    __syncthreads();
    for (int j = sub; j < lim; j += kRankLanes) rank += tile[j] < key ? 1 : 0;
  }
#pragma unroll
  for (int o = 1; o < kRankLanes; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (sub == 0 && i < nb) {
    block_keys[rank] = key;
    unsigned s = hash64((unsigned long long)key) & mask;
    while (hkeys[s] != (unsigned long long)key) s = (s + 1) & mask;
    hvals[s] = rank;
  }
}

__global__ void k_node_ids(const unsigned long long* __restrict__ hkeys,
                           const int* __restrict__ hvals, unsigned mask,
                           const long long* __restrict__ coords, long long m,
                           long long* __restrict__ ids, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int64_t c[3] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
  int64_t key;
  int b = -1;
  if (pack_block(c[0] >> 2, c[1] >> 2, c[2] >> 2, &key))
    b = hash_find(hkeys, hvals, mask, (uint64_t)key);
  if (b < 0) {
    raise_status(st, MPMRB_E_ALLOCATION, 3, i);
    ids[i] = 0;
    return;
  }
  ids[i] = (long long)b * kNodesPerBlock + (((c[0] & 3) << 4) | ((c[1] & 3) << 2) | (c[2] & 3));
}

__global__ void k_build_stencil(const unsigned long long* __restrict__ hkeys,
                                const int* __restrict__ hvals, unsigned mask, double h,
                                const double* __restrict__ x, long long n,
                                double* __restrict__ weights, long long* __restrict__ nodes,
                                double* __restrict__ dpos, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  Stencil1 s;
  make_stencil1(p, h, s);
  StencilBlocks sb;
  if (!resolve_blocks(s, hkeys, hvals, mask, sb)) {
    raise_status(st, MPMRB_E_ALLOCATION, 4, i);
    return;
  }
  int k = 0;
  for (int ox = 0; ox < 3; ++ox)
    for (int oy = 0; oy < 3; ++oy)
      for (int oz = 0; oz < 3; ++oz, ++k) {
        weights[27 * i + k] = __dmul_rn(__dmul_rn(s.w[0][ox], s.w[1][oy]), s.w[2][oz]);
        nodes[27 * i + k] = stencil_node(s, sb, ox, oy, oz);
        dpos[81 * i + 3 * k + 0] = __dmul_rn(__dsub_rn((double)ox, s.fx[0]), h);
        dpos[81 * i + 3 * k + 1] = __dmul_rn(__dsub_rn((double)oy, s.fx[1]), h);
        dpos[81 * i + 3 * k + 2] = __dmul_rn(__dsub_rn((double)oz, s.fx[2]), h);
      }
}

}  // namespace

// ---------------------------------------------------------------- launchers

int launch_base_cells(Ctx& c, const double* x, long long n, double h, long long* cells) {
  if (n == 0) return MPMRB_OK;
  k_base_cells<<<grid_for(3 * n, 256), 256, 0, c.stream>>>(x, n, h, cells);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_sort_plan(Ctx& c, const double* x, long long n, double h, uint16_t* keys,
                     long long* perm, long long* inv_perm, uint16_t* bin_keys,
                     long long* bin_starts, long long* bin_of, int* n_bins_dev) {
  int ntiles = (int)((n + kPlanWarpTile - 1) / kPlanWarpTile);
  if (ntiles < 1) ntiles = 1;
  long long hist_n = (long long)kBuckets * ntiles;
  if (c.scratch[SS_HIST].grow(sizeof(int) * hist_n) ||
      c.scratch[SS_TMP0].grow(sizeof(int) * hist_n) ||
      c.scratch[SS_TMP1].grow(sizeof(int) * kBuckets))
    return MPMRB_E_CUDA;
  int* th = c.scratch[SS_HIST].as<int>();
  int* scanned = c.scratch[SS_TMP0].as<int>();
  int* brank = c.scratch[SS_TMP1].as<int>();
  if (n > 0) {
    k_morton<<<grid_for(n, 256), 256, 0, c.stream>>>(x, n, h, keys, c.status);
    c.launches++;
  }
  unsigned cta = (unsigned)((ntiles + kPlanWarps - 1) / kPlanWarps);
  k_plan_hist<<<cta, kPlanWarps * 32, 0, c.stream>>>(keys, n, ntiles, th);
  c.launches++;
  int rc = scan_exclusive_i32(c, th, scanned, hist_n, nullptr, nullptr, c.scratch[SS_TILE]);
  if (rc) return rc;
  k_plan_bins<<<1, kBuckets, 0, c.stream>>>(scanned, ntiles, n, bin_keys, bin_starts, brank,
                                           n_bins_dev);
  k_plan_scatter<<<cta, kPlanWarps * 32, 0, c.stream>>>(keys, n, ntiles, scanned, brank, perm,
                                                       inv_perm, bin_of);
  c.launches += 2;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_morton_only(Ctx& c, const double* x, long long n, double h, uint16_t* keys) {
  if (n == 0) return MPMRB_OK;
  k_morton<<<grid_for(n, 256), 256, 0, c.stream>>>(x, n, h, keys, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_staleness(Ctx& c, const uint16_t* plan_keys, const double* x, long long n, double h,
                     unsigned long long* changed_dev) {
  MPMRB_CUDA_OK(cudaMemsetAsync(changed_dev, 0, sizeof(unsigned long long), c.stream));
  if (n == 0) return MPMRB_OK;
  k_staleness<<<grid_for(n, 256), 256, 0, c.stream>>>(plan_keys, x, n, h, changed_dev);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_grid_build(Ctx& c, const double* x, long long n, double h, long long* block_keys,
                      long long block_cap, unsigned long long* hkeys, int* hvals,
                      long long hash_cap, long long* ukeys, int* nb_dev) {
  unsigned mask = (unsigned)(hash_cap - 1);
  k_hash_clear<<<grid_for(hash_cap, 256), 256, 0, c.stream>>>(hkeys, hash_cap, nb_dev);
  c.launches++;
  if (n > 0) {
    k_block_insert<<<grid_for(n, 256), 256, 0, c.stream>>>(x, n, h, hkeys, mask, ukeys,
                                                          block_cap, nb_dev, c.status);
    c.launches++;
  }
  k_block_rank_par<<<grid_for(block_cap * kRankLanes, 256), 256, 0, c.stream>>>(
      ukeys, nb_dev, block_cap, block_keys, hkeys, hvals, mask);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_node_ids(Ctx& c, const mpmrb_grid_view& g, const long long* coords, long long m,
                    long long* ids) {
  if (m == 0) return MPMRB_OK;
  k_node_ids<<<grid_for(m, 256), 256, 0, c.stream>>>(
      (const unsigned long long*)g.hash_keys, (const int*)g.hash_vals, (unsigned)(g.hash_cap - 1),
      coords, m, ids, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_build_stencil(Ctx& c, const mpmrb_grid_view& g, const double* x, long long n,
                         double* weights, long long* nodes, double* dpos) {
  if (n == 0) return MPMRB_OK;
  k_build_stencil<<<grid_for(n, 128), 128, 0, c.stream>>>(
      (const unsigned long long*)g.hash_keys, (const int*)g.hash_vals, (unsigned)(g.hash_cap - 1),
      g.h, x, n, weights, nodes, dpos, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace mpmrb
