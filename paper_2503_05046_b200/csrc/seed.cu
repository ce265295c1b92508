// GPU state construction: the jittered-lattice box
// seeding of the reference (particles.py:81-136), bit-identical to NumPy.
//
// The reference draws the jitter with numpy.random.default_rng(seed).uniform
// over the (points, 3) array in row-major order.  That generator is PCG64
// (128-bit LCG, XSL-RR output) and Generator.uniform returns
//   low + (high - low) * ((next64 >> 11) * 2^-53).
// Element e of the stream is the output after e + 1 LCG steps from the seeded
// state, so every thread jumps ahead independently (O(log e) 128-bit
// multiply-adds, the standard LCG advance) and reproduces NumPy's values
// bit for bit.  The host passes the seeded state (NumPy's SeedSequence
// hashing stays on the host: bit_generator.state).  The in-box filter keeps
// NumPy's order through a stable compaction.
#include "common.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;
}

__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_output(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  const unsigned long long x = hi ^ lo;
  const unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

struct BoxSeed {
  long long lo[3], ext[3];  // cell range [lo, lo + ext)
  int per_axis;
  double step, jlow, jrange, h;
  double center[3], half[3];
  unsigned long long s_hi, s_lo, i_hi, i_lo;
  bool jitter;
};

__device__ __forceinline__ bool seed_point(const BoxSeed& b, long long p, double* out) {
  const int ppc = b.per_axis * b.per_axis * b.per_axis;
  const long long cell = p / ppc;
  const int o = (int)(p - cell * ppc);
  const long long cz = cell % b.ext[2], cy = (cell / b.ext[2]) % b.ext[1],
                  cx = cell / (b.ext[2] * b.ext[1]);
  const int oz = o % b.per_axis, oy = (o / b.per_axis) % b.per_axis,
            ox = o / (b.per_axis * b.per_axis);
  const long long c[3] = {b.lo[0] + cx, b.lo[1] + cy, b.lo[2] + cz};
  const int oo[3] = {ox, oy, oz};
  double j[3] = {0.0, 0.0, 0.0};
  if (b.jitter) {
    const u128 s0 = ((u128)b.s_hi << 64) | b.s_lo, inc = ((u128)b.i_hi << 64) | b.i_lo;
    u128 s = pcg_advance(s0, inc, 3ull * (unsigned long long)p + 1ull);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (d) s = s * pcg_mult() + inc;
      const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
      j[d] = __dadd_rn(b.jlow, __dmul_rn(b.jrange, u));  // no FMA: NumPy rounds twice
    }
  }
  bool inside = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    // ((cell + (o + 0.5) step) + jitter) * h, the NumPy operation order
    const double off = __dmul_rn(__dadd_rn((double)oo[d], 0.5), b.step);
    const double v = __dmul_rn(__dadd_rn(__dadd_rn((double)c[d], off), j[d]), b.h);
    out[d] = v;
    inside &= fabs(v - b.center[d]) <= b.half[d];
  }
  return inside;
}

__global__ void k_seed_count(BoxSeed b, long long m, int* __restrict__ flag) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m;
       p += (long long)gridDim.x * blockDim.x) {
    double x[3];
    flag[p] = seed_point(b, p, x) ? 1 : 0;
  }
}

__global__ void k_seed_emit(BoxSeed b, long long m, const int* __restrict__ flag,
                            const int* __restrict__ off, long long cap, double* __restrict__ xout) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m;
       p += (long long)gridDim.x * blockDim.x) {
    if (!flag[p]) continue;
    const long long k = off[p];
    if (k >= cap) continue;
    double x[3];
    seed_point(b, p, x);
#pragma unroll
    for (int d = 0; d < 3; ++d) xout[3 * k + d] = x[d];
  }
}

unsigned sd_grid(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

}  // namespace

int launch_seed_box(Ctx& c, const long long* lo, const long long* hi, int per_axis,
                    double jitter, double h, const double* center, const double* half,
                    const unsigned long long* state4, double* x_out, long long cap,
                    long long* n_host) {
  BoxSeed b{};
  long long ncell = 1;
  for (int d = 0; d < 3; ++d) {
    b.lo[d] = lo[d];
    b.ext[d] = hi[d] - lo[d];
    if (b.ext[d] <= 0) {
      *n_host = 0;
      return MPMRB_OK;
    }
    ncell *= b.ext[d];
    b.center[d] = center[d];
    b.half[d] = half[d];
  }
  b.per_axis = per_axis;
  b.step = 1.0 / per_axis;
  b.jitter = jitter > 0.0;
  const double low = -0.5 * b.step * jitter, high = 0.5 * b.step * jitter;
  b.jlow = low;
  b.jrange = high - low;  // Generator.uniform: low + (high - low) * u
  b.h = h;
  b.s_hi = state4[0];
  b.s_lo = state4[1];
  b.i_hi = state4[2];
  b.i_lo = state4[3];
  const long long m = ncell * per_axis * per_axis * per_axis;
  if (c.scratch[SS_TMP2].grow(sizeof(int) * (m + 1)) || c.scratch[SS_TMP3].grow(sizeof(int) * (m + 1)) ||
      c.scratch[SS_COUNT].grow(64))
    return MPMRB_E_CUDA;
  int* flag = c.scratch[SS_TMP2].as<int>();
  int* off = c.scratch[SS_TMP3].as<int>();
  int* total = c.scratch[SS_COUNT].as<int>();
  k_seed_count<<<sd_grid(m), 256, 0, c.stream>>>(b, m, flag);
  c.launches++;
  int rc = scan_exclusive_i32(c, flag, off, m, nullptr, total, c.scratch[SS_TILE]);
  if (rc) return rc;
  int nh = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&nh, total, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
  *n_host = nh;
  if (!x_out) return MPMRB_OK;  // count only
  if (nh > cap) return MPMRB_E_CAPACITY;
  k_seed_emit<<<sd_grid(m), 256, 0, c.stream>>>(b, m, flag, off, cap, x_out);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace mpmrb
