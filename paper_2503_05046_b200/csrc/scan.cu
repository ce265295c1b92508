// Device-wide exclusive prefix sums, hand-written: int32 scans run single-pass
// (decoupled look-back, k_scan_onepass); int64 scans and contexts without the
// scan state run three-phase (tile reduce, single-CTA scan of tile sums, tile
// down-sweep).  Used for contact
// compaction (collision.py:88-132 ordering), active-node compaction
// (solver.py:203-205) and the Morton counting sort (transfer.py:89).
//
// Counts may live on the device (n_dev) so the launches can sit inside a CUDA
// graph whose sizes are only known on the GPU.
#include "common.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;  // 2048
constexpr int kTopThreads = 1024;

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// exclusive block scan of one value per thread; returns block total via *tot
template <class T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* sm /*NT/32*/, T* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = (lane < NT / 32) ? sm[lane] : T(0);
    s = warp_incl_scan(s);
    if (lane < NT / 32) sm[lane] = s;
  }
  __syncthreads();
  T warp_off = wid ? sm[wid - 1] : T(0);
  *tot = sm[NT / 32 - 1];
  __syncthreads();
  return warp_off + inc - v;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_reduce(const T* __restrict__ in,
                                                              long long n_cap, const int* n_dev,
                                                              T* __restrict__ tiles) {
  __shared__ T sm[kScanThreads / 32];
  long long n = n_dev ? (long long)*n_dev : n_cap;
  long long base = (long long)blockIdx.x * kTile;
  if (base >= n) {
    if (threadIdx.x == 0) tiles[blockIdx.x] = T(0);
    return;
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    long long idx = base + (long long)i * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  T tot;
  block_excl_scan<T, kScanThreads>(s, sm, &tot);
  if (threadIdx.x == 0) tiles[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(kTopThreads) k_tile_scan(T* __restrict__ tiles, int ntiles,
                                                           T* total) {
  __shared__ T sm[kTopThreads / 32];
  __shared__ T carry;
  if (threadIdx.x == 0) carry = T(0);
  __syncthreads();
  for (int base = 0; base < ntiles; base += kTopThreads) {
    int i = base + threadIdx.x;
    T v = (i < ntiles) ? tiles[i] : T(0);
    T tot;
    T ex = block_excl_scan<T, kTopThreads>(v, sm, &tot);
    if (i < ntiles) tiles[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_down(const T* __restrict__ in,
                                                            T* __restrict__ out, long long n_cap,
                                                            const int* n_dev,
                                                            const T* __restrict__ tiles) {
  __shared__ T sm[kScanThreads / 32];
  long long n = n_dev ? (long long)*n_dev : n_cap;
  long long base = (long long)blockIdx.x * kTile;
  if (base >= n) return;
  // each thread owns kScanItems consecutive elements
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    long long idx = base + (long long)threadIdx.x * kScanItems + i;
    v[i] = (idx < n) ? in[idx] : T(0);
    s += v[i];
  }
  T tot;
  T ex = block_excl_scan<T, kScanThreads>(s, sm, &tot);
  T run = tiles[blockIdx.x] + ex;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    long long idx = base + (long long)threadIdx.x * kScanItems + i;
    if (idx < n) out[idx] = run;
    run += v[i];
  }
}

// Single-pass scan with decoupled look-back (int32): each CTA takes a tile by
// ticket, publishes its aggregate, and warp 0 walks back over the preceding
// tiles' status words until it meets an inclusive prefix.  A status word is
// [epoch:30 | flag:2 | value:32]; the epoch is read before the ticket and
// advanced by the CTA that takes the last ticket, so stale words of earlier
// launches never match and nothing is reset between launches or graph replays.
// (The epoch wraps after 2^30 launches on one context; a stale word could then
// match only if no launch in between covered its tile.)
constexpr unsigned kStAgg = 1u, kStInc = 2u;
__device__ __forceinline__ unsigned long long st_word(unsigned ep, unsigned flag, int v) {
  return ((unsigned long long)(ep & 0x3fffffffu) << 34) | ((unsigned long long)flag << 32) |
         (unsigned long long)(unsigned)v;
}
constexpr int kOpThreads = 256, kOpItems = 16;
constexpr int kOpTile = kOpThreads * kOpItems;  // 4096
__global__ void __launch_bounds__(kOpThreads) k_scan_onepass(const int* __restrict__ in,
                                                             int* __restrict__ out,
                                                             long long n_cap, const int* n_dev,
                                                             int* total,
                                                             unsigned long long* state) {
  __shared__ int sm[kOpThreads / 32];
  __shared__ int s_tile, s_prefix;
  __shared__ unsigned s_epoch;
  unsigned* ctrl = reinterpret_cast<unsigned*>(state);  // [0] ticket, [1] epoch
  volatile unsigned long long* st = state + 1;
  if (threadIdx.x == 0) {
    const unsigned ep = *reinterpret_cast<volatile unsigned*>(ctrl + 1);
    __threadfence();
    const int t = (int)atomicAdd(ctrl, 1u);
    if (t == (int)gridDim.x - 1) {  // every CTA holds its ticket and has read the epoch
      __threadfence();
      atomicExch(ctrl, 0u);
      atomicAdd(ctrl + 1, 1u);
    }
    s_tile = t;
    s_epoch = ep;
  }
  __syncthreads();
  const int t = s_tile;
  const unsigned ep = s_epoch & 0x3fffffffu;
  const long long n = n_dev ? (long long)*n_dev : n_cap;
  const long long base = (long long)t * kOpTile;
  if (base >= n) {
    if (t == 0 && threadIdx.x == 0 && total) *total = 0;
    return;  // tiles are taken in order: no live tile waits on a dead one
  }
  // each warp owns a contiguous chunk of 32 x kOpItems elements, read and
  // written in coalesced rounds of 32; round r's inclusive warp scan carries
  // the running total of rounds < r
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long chunk = base + (long long)wid * (32 * kOpItems);
  int v[kOpItems];
#pragma unroll
  for (int r = 0; r < kOpItems; ++r) {
    const long long idx = chunk + r * 32 + lane;
    v[r] = idx < n ? in[idx] : 0;
  }
  int run = 0;
#pragma unroll
  for (int r = 0; r < kOpItems; ++r) {
    const int inc = warp_incl_scan(v[r]);
    v[r] = run + inc - v[r];  // exclusive within the warp's chunk
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 31) sm[wid] = run;
  __syncthreads();
  int tot = 0, woff = 0;
#pragma unroll
  for (int k = 0; k < kOpThreads / 32; ++k) {
    const int x = sm[k];
    woff += k < wid ? x : 0;
    tot += x;
  }
  if (threadIdx.x == 0) st[t] = st_word(ep, t == 0 ? kStInc : kStAgg, tot);
  if (t > 0 && wid == 0) {
    int excl = 0;
    for (int j = t - 1;; j -= 32) {
      const int idx = j - lane;
      unsigned long long w;
      bool ready;
      do {
        w = idx >= 0 ? st[idx] : st_word(ep, kStInc, 0);
        ready = (unsigned)(w >> 34) == ep && ((w >> 32) & 3u) != 0u;
      } while (!__all_sync(0xffffffffu, ready));
      const unsigned inc = __ballot_sync(0xffffffffu, ((w >> 32) & 3u) == kStInc);
      const int first = inc ? __ffs(inc) - 1 : 32;  // nearest tile holding an inclusive prefix
      int val = lane <= first ? (int)(unsigned)w : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
      excl += val;
      if (inc) break;
    }
    if (lane == 0) {
      st[t] = st_word(ep, kStInc, excl + tot);
      s_prefix = excl;
    }
  }
  __syncthreads();
  const int off = (t > 0 ? s_prefix : 0) + woff;
#pragma unroll
  for (int r = 0; r < kOpItems; ++r) {
    const long long idx = chunk + r * 32 + lane;
    if (idx < n) out[idx] = off + v[r];
  }
  if (total && threadIdx.x == 0 && n - base <= kOpTile)  // the last live tile
    *total = (t > 0 ? s_prefix : 0) + tot;
}

template <class T>
int scan_impl(Ctx& c, const T* in, T* out, long long n_cap, const int* n_dev, T* total_dev,
              DevBuf& tiles) {
  long long ntiles = (n_cap + kTile - 1) / kTile;
  if (ntiles < 1) ntiles = 1;
  if (tiles.grow(sizeof(T) * ntiles) != MPMRB_OK) return MPMRB_E_CUDA;
  T* t = tiles.as<T>();
  k_tile_reduce<T><<<(unsigned)ntiles, kScanThreads, 0, c.stream>>>(in, n_cap, n_dev, t);
  k_tile_scan<T><<<1, kTopThreads, 0, c.stream>>>(t, (int)ntiles, total_dev);
  k_tile_down<T><<<(unsigned)ntiles, kScanThreads, 0, c.stream>>>(in, out, n_cap, n_dev, t);
  c.launches += 3;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace

int scan_exclusive_i32(Ctx& c, const int* in, int* out, long long n_cap, const int* n_dev,
                       int* total_dev, DevBuf& tiles) {
  const long long ntiles = n_cap > 0 ? (n_cap + kOpTile - 1) / kOpTile : 1;
  if (c.scan_state && ntiles <= kOnePassMaxTiles) {
    k_scan_onepass<<<(unsigned)ntiles, kOpThreads, 0, c.stream>>>(in, out, n_cap, n_dev,
                                                                    total_dev, c.scan_state);
    c.launches++;
    MPMRB_CUDA_OK(cudaGetLastError());
    return MPMRB_OK;
  }
  return scan_impl<int>(c, in, out, n_cap, n_dev, total_dev, tiles);
}

int scan_exclusive_i64(Ctx& c, const long long* in, long long* out, long long n,
                       long long* total_dev, DevBuf& tiles) {
  return scan_impl<long long>(c, in, out, n, nullptr, total_dev, tiles);
}

}  // namespace mpmrb
