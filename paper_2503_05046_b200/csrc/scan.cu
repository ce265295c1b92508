// Device-wide exclusive prefix sums (hand-written, three-phase: tile reduce,
// single-CTA scan of tile sums, tile down-sweep).  Used for contact
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
  return scan_impl<int>(c, in, out, n_cap, n_dev, total_dev, tiles);
}

int scan_exclusive_i64(Ctx& c, const long long* in, long long* out, long long n,
                       long long* total_dev, DevBuf& tiles) {
  return scan_impl<long long>(c, in, out, n, nullptr, total_dev, tiles);
}

}  // namespace mpmrb
