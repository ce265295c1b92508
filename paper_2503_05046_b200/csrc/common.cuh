// Shared device helpers for the sm_100a MPM–rigid coupling kernels.
//
// Hot-path arithmetic is float64, matching the reference (every
// reference array is float64, e.g. grid.py:55-61).  The fused substep also has
// an fp32 performance mode for the per-particle state and arithmetic (M3T,
// Stencil1T with T = float; grid, contacts and the solve stay float64).  B200 has full-rate
// FP64 CUDA cores (no tensor cores are used: the path is gather/scatter and
// per-particle 3x3 algebra, not a dense contraction).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mpmrb_b200.h"

namespace mpmrb {

constexpr int kBlockEdge = 4;      // grid.py:16
constexpr int kNodesPerBlock = 64;  // grid.py:17
constexpr int64_t kBias21 = int64_t(1) << 20;  // grid.py:18, transfer.py:35
constexpr int64_t kMask21 = (int64_t(1) << 21) - 1;
constexpr double kMassEps = 1e-12;  // grid.py:19
constexpr double kSigmaFloor = 0.05;  // materials.py:21
constexpr uint64_t kEmptyKey = ~uint64_t(0);

// ----------------------------------------------------------------- status
// First error wins; the host reads it back once per step / API call.
struct DevStatus {
  int code;
  int detail;
  long long aux;
};

__device__ __forceinline__ void raise_status(DevStatus* st, int code, int detail = 0,
                                             long long aux = 0) {
  if (atomicCAS(&st->code, 0, code) == 0) {
    st->detail = detail;
    st->aux = aux;
  }
}

// ----------------------------------------------------------------- small linear algebra
// 3x3 row-major matrices in the particle arithmetic type T: double (the
// reference's float64) or float (the fp32 performance mode, sim.cu).
template <class T>
struct M3T {
  T a[9];  // row-major
  __device__ __forceinline__ T& operator()(int i, int j) { return a[3 * i + j]; }
  __device__ __forceinline__ T operator()(int i, int j) const { return a[3 * i + j]; }
};
using M3 = M3T<double>;

template <class T>
__device__ __forceinline__ M3T<T> m3_load(const T* p) {
  M3T<T> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.a[i] = p[i];
  return m;
}
template <class T>
__device__ __forceinline__ void m3_store(T* p, const M3T<T>& m) {
#pragma unroll
  for (int i = 0; i < 9; ++i) p[i] = m.a[i];
}
template <class T = double>
__device__ __forceinline__ M3T<T> m3_identity() {
  M3T<T> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.a[i] = (i % 4 == 0) ? T(1) : T(0);
  return m;
}
template <class T>
__device__ __forceinline__ M3T<T> m3_mul(const M3T<T>& x, const M3T<T>& y) {
  M3T<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r(i, j) = x(i, 0) * y(0, j) + x(i, 1) * y(1, j) + x(i, 2) * y(2, j);
  return r;
}
template <class T>
__device__ __forceinline__ M3T<T> m3_mul_bt(const M3T<T>& x, const M3T<T>& y) {  // x @ y^T
  M3T<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r(i, j) = x(i, 0) * y(j, 0) + x(i, 1) * y(j, 1) + x(i, 2) * y(j, 2);
  return r;
}
// determinant as column triple product c0 . (c1 x c2) (materials.py:49-54)
template <class T>
__device__ __forceinline__ T m3_det(const M3T<T>& m) {
  T k0 = m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2);
  T k1 = m(2, 1) * m(0, 2) - m(0, 1) * m(2, 2);
  T k2 = m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2);
  return m(0, 0) * k0 + m(1, 0) * k1 + m(2, 0) * k2;
}
// inverse-transpose via the adjugate (materials.py:57-67)
template <class T>
__device__ __forceinline__ M3T<T> m3_inv_transpose(const M3T<T>& m) {
  // columns a0,a1,a2 of m; result columns are a1xa2, a2xa0, a0xa1 over det
  T c0[3] = {m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2), m(2, 1) * m(0, 2) - m(0, 1) * m(2, 2),
             m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2)};
  T c1[3] = {m(1, 2) * m(2, 0) - m(2, 2) * m(1, 0), m(2, 2) * m(0, 0) - m(0, 2) * m(2, 0),
             m(0, 2) * m(1, 0) - m(1, 2) * m(0, 0)};
  T c2[3] = {m(1, 0) * m(2, 1) - m(2, 0) * m(1, 1), m(2, 0) * m(0, 1) - m(0, 0) * m(2, 1),
             m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1)};
  T det = m(0, 0) * c0[0] + m(1, 0) * c0[1] + m(2, 0) * c0[2];
  M3T<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    r(i, 0) = c0[i] / det;
    r(i, 1) = c1[i] / det;
    r(i, 2) = c2[i] / det;
  }
  return r;
}

template <class T>
__device__ __forceinline__ bool m3_finite(const M3T<T>& m) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) ok &= isfinite(m.a[i]);
  return ok;
}

// ----------------------------------------------------------------- keys
// (b + 2^20) per axis, packed x<<42 | y<<21 | z (grid.py:26-31)
__device__ __forceinline__ bool pack_block(int64_t bx, int64_t by, int64_t bz, int64_t* key) {
  int64_t x = bx + kBias21, y = by + kBias21, z = bz + kBias21;
  if (x < 0 || y < 0 || z < 0 || x > kMask21 || y > kMask21 || z > kMask21) return false;
  *key = (x << 42) | (y << 21) | z;
  return true;
}

// floor(x/h - 0.5): IEEE division then subtraction, never a reciprocal
// multiply (grid.py:34-36)
__device__ __forceinline__ int64_t base_cell(double x, double h) {
  return (int64_t)floor(__dsub_rn(__ddiv_rn(x, h), 0.5));
}

__device__ __forceinline__ uint32_t hash64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return (uint32_t)k;
}

// Open-addressing lookup of a block key; returns block index or -1.
__device__ __forceinline__ int hash_find(const unsigned long long* __restrict__ hkeys,
                                         const int* __restrict__ hvals, uint32_t mask,
                                         uint64_t key) {
  uint32_t s = hash64(key) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    unsigned long long k = hkeys[s];
    if (k == key) return hvals[s];
    if (k == kEmptyKey) return -1;
    s = (s + 1) & mask;
  }
  return -1;
}

// ----------------------------------------------------------------- B-spline stencil
// Per-particle quadratic B-spline data (mpm.py:39-53), kept in registers.
struct Stencil1 {
  int64_t base[3];
  double fx[3];
  double w[3][3];  // w[axis][offset]
};

__device__ __forceinline__ void make_stencil1(const double* x, double h, Stencil1& s) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double q = __ddiv_rn(x[a], h);
    int64_t b = (int64_t)floor(__dsub_rn(q, 0.5));
    double f = __dsub_rn(q, (double)b);
    s.base[a] = b;
    s.fx[a] = f;
    // explicit _rn ops: no FMA contraction, so weights match NumPy bitwise
    double t0 = __dsub_rn(1.5, f), t1 = __dsub_rn(f, 1.0), t2 = __dsub_rn(f, 0.5);
    s.w[a][0] = __dmul_rn(0.5, __dmul_rn(t0, t0));
    s.w[a][1] = __dsub_rn(0.75, __dmul_rn(t1, t1));
    s.w[a][2] = __dmul_rn(0.5, __dmul_rn(t2, t2));
  }
}

// The same stencil with fractions and weights in the particle arithmetic
// type T (fp32 performance mode): the base cell is still the IEEE float64
// floor(x/h - 0.5) of the float64 position, so nodes and blocks are the
// float64 path's.
template <class T>
struct Stencil1T {
  int64_t base[3];
  T fx[3];
  T w[3][3];
};
template <class T>
__device__ __forceinline__ void make_stencil1_t(const double* x, double h, Stencil1T<T>& s) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double q = __ddiv_rn(x[a], h);
    const int64_t b = (int64_t)floor(__dsub_rn(q, 0.5));
    const T f = (T)__dsub_rn(q, (double)b);
    s.base[a] = b;
    s.fx[a] = f;
    const T t0 = T(1.5) - f, t1 = f - T(1), t2 = f - T(0.5);
    s.w[a][0] = T(0.5) * (t0 * t0);
    s.w[a][1] = T(0.75) - t1 * t1;
    s.w[a][2] = T(0.5) * (t2 * t2);
  }
}
template <>
__device__ __forceinline__ void make_stencil1_t<double>(const double* x, double h,
                                                       Stencil1T<double>& s) {
  Stencil1 d;
  make_stencil1(x, h, d);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    s.base[a] = d.base[a];
    s.fx[a] = d.fx[a];
#pragma unroll
    for (int o = 0; o < 3; ++o) s.w[a][o] = d.w[a][o];
  }
}

// Resolve the <=8 blocks a stencil touches; blk[ix][iy][iz] indexed by
// whether axis offset lands in the low (0) or high (1) block.
struct StencilBlocks {
  int idx[8];
  int64_t lo[3];
};

template <class S>
__device__ __forceinline__ bool resolve_blocks(const S& s,
                                               const unsigned long long* __restrict__ hkeys,
                                               const int* __restrict__ hvals, uint32_t mask,
                                               StencilBlocks& sb) {
  int64_t lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = s.base[a] >> 2;
    hi[a] = (s.base[a] + 2) >> 2;
    sb.lo[a] = lo[a];
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int ix = (i >> 2) & 1, iy = (i >> 1) & 1, iz = i & 1;
    // skip duplicate combos (high == low on an axis)
    if ((ix && hi[0] == lo[0]) || (iy && hi[1] == lo[1]) || (iz && hi[2] == lo[2])) {
      sb.idx[i] = -1;
      continue;
    }
    int64_t key;
    if (!pack_block(ix ? hi[0] : lo[0], iy ? hi[1] : lo[1], iz ? hi[2] : lo[2], &key)) {
      ok = false;
      sb.idx[i] = -1;
      continue;
    }
    int b = hash_find(hkeys, hvals, mask, (uint64_t)key);
    if (b < 0) ok = false;
    sb.idx[i] = b;
  }
  return ok;
}

// Linear node id of stencil slot (ox,oy,oz) (grid.py:121: block*64 + (lx*4+ly)*4+lz)
template <class S>
__device__ __forceinline__ int stencil_node(const S& s, const StencilBlocks& sb, int ox,
                                            int oy, int oz) {
  int64_t cx = s.base[0] + ox, cy = s.base[1] + oy, cz = s.base[2] + oz;
  int ix = (int)((cx >> 2) != sb.lo[0]);
  int iy = (int)((cy >> 2) != sb.lo[1]);
  int iz = (int)((cz >> 2) != sb.lo[2]);
  int b = sb.idx[(ix << 2) | (iy << 1) | iz];
  return b * kNodesPerBlock + (int)(((cx & 3) << 4) | ((cy & 3) << 2) | (cz & 3));
}

// ----------------------------------------------------------------- reductions
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem /*>= NT/32*/) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < NT / 32) ? smem[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

}  // namespace mpmrb

#define MPMRB_CUDA_OK(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) return ::mpmrb::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
  } while (0)
