// Particle <-> grid transfers on sm_100a: float64, or float32 particle state
// and arithmetic in the fp32 performance mode (the grid stays float64).
//
//  * k_p2g   : stress (polar / Hencky) + 27-node x 7-channel APIC/MLS scatter
//              (mpm.py:66-99, materials.py:113-122).  One thread per particle,
//              stencil kept in registers (never materialised, unlike the
//              reference's (n,27,3) arrays), float64 REDG atomics into the
//              node channels.
//  * k_grid_update : v_k, v*, active mask (mpm.py:102-115) + per-warp active
//              counts for the ordered active-node compaction (solver.py:203).
//  * k_g2p   : gather, APIC C, advection, F update, singular-value clamp
//              (mpm.py:118-138, materials.py:86-110), Drucker-Prager return map
//              for sand, divergence check (coupling.py:153-165).
#include <climits>

#include "common.cuh"
#include "internal.h"
#include "svd3.cuh"

namespace mpmrb {

namespace {

template <class T>
__device__ __forceinline__ M3T<T> particle_stress(const M3T<T>& f, const mpmrb_material& m) {
  return (m.kind == MPMRB_MAT_SAND) ? kirchhoff_hencky<T>(f, (T)m.mu, (T)m.lam)
                                    : kirchhoff_fixed_corotated<T>(f, (T)m.mu, (T)m.lam);
}

__global__ void k_scatter_reduce(const long long* __restrict__ ids, const double* __restrict__ vals,
                                 long long rows, long long k, long long nch, long long n_out,
                                 double* __restrict__ out, DevStatus* st) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= rows * k) return;
  long long node = ids[e];
  if (node < 0 || node >= n_out) {
    raise_status(st, MPMRB_E_INVALID, 10, e);
    return;
  }
  for (long long ch = 0; ch < nch; ++ch) atomicAdd(&out[node * nch + ch], vals[e * nch + ch]);
}

// Deterministic scatter (transfer.py:135-145, 178-187): the reference sums
// each (node, channel) with np.bincount, i.e. sequentially in flattened
// (row, slot) order starting from 0.0.  The entries are stably sorted by node
// id (their entry index rides along as the value), so each node's entries sit
// contiguously in that same order; one thread per node then folds them left
// to right -- the same float operations in the same order as the reference,
// hence bitwise-identical sums, independent of any sort plan.
__global__ void k_ordered_keys(const long long* __restrict__ ids, long long e_n, long long n_out,
                               unsigned* __restrict__ keys, int* __restrict__ vals,
                               DevStatus* st) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e_n;
       e += (long long)gridDim.x * blockDim.x) {
    long long node = ids[e];
    if (node < 0 || node >= n_out) {
      raise_status(st, MPMRB_E_INVALID, 12, e);
      node = 0;
    }
    keys[e] = (unsigned)node;
    vals[e] = (int)e;
  }
}

// seg_start[node] = first sorted position with key >= node (n_out + 1 entries)
__global__ void k_ordered_bounds(const unsigned* __restrict__ skeys, long long e_n, long long n_out,
                                 long long* __restrict__ seg_start) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= e_n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long prev = i == 0 ? -1 : (long long)skeys[i - 1];
    const long long cur = i == e_n ? n_out : (long long)skeys[i];
    for (long long q = prev + 1; q <= cur; ++q) seg_start[q] = i;
  }
}

template <int NCH>
__global__ void k_ordered_sum(const int* __restrict__ sidx, const long long* __restrict__ seg_start,
                              const double* __restrict__ vals, long long n_out, long long nch,
                              double* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n_out;
       q += (long long)gridDim.x * blockDim.x) {
    const long long a = seg_start[q], b = seg_start[q + 1];
    if (NCH > 0) {
      double acc[NCH > 0 ? NCH : 1];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.0;
      for (long long j = a; j < b; ++j) {
        const long long e = sidx[j];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[ch] += vals[e * NCH + ch];
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) out[q * NCH + ch] = acc[ch];
    } else {
      for (long long ch = 0; ch < nch; ++ch) {
        double acc = 0.0;
        for (long long j = a; j < b; ++j) acc += vals[(long long)sidx[j] * nch + ch];
        out[q * nch + ch] = acc;
      }
    }
  }
}

__global__ void k_stresses(const double* __restrict__ f, const long long* __restrict__ mid,
                           long long n, const mpmrb_material* __restrict__ mats, int nmat,
                           double* __restrict__ tau, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long m = mid[i];
  if (m < 0 || m >= nmat) {
    raise_status(st, MPMRB_E_INVALID, 11, i);
    return;
  }
  M3 t = particle_stress(m3_load(f + 9 * i), mats[m]);
  m3_store(tau + 9 * i, t);
}

constexpr int kWarpTile = 128;  // nodes per warp tile (e.g. 4 x 4 x 8)

// A warp's particles, in lane order, are cut into segments of consecutive
// lanes [s0, s1) whose stencils fit one node tile: <= kWarpTile nodes and <= 2
// blocks per axis (so the tile's blocks resolve with <= 8 hash lookups).  A
// warp inside one block is one segment; a warp straddling two blocks
// (consecutive in key order, not necessarily adjacent in space) is two.  s1 is
// the first lane whose prefix bounding box no longer fits: prefix boxes only
// grow, and one stencil always fits, so s1 > s0.
struct WarpSeg {
  int s1, lo[3], nx, ny, nz;
};
__device__ __forceinline__ WarpSeg warp_segment(const int (&b)[3], bool live, int lane, int s0,
                                                int n_live) {
  const bool act = live && lane >= s0;
  int mn[3], mx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    mn[a] = act ? b[a] : INT_MAX;
    mx[a] = act ? b[a] : INT_MIN;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int tn = __shfl_up_sync(0xffffffffu, mn[a], o);
      const int tx = __shfl_up_sync(0xffffffffu, mx[a], o);
      if (lane >= o) {
        mn[a] = min(mn[a], tn);
        mx[a] = max(mx[a], tx);
      }
    }
  }
  bool fits = true;
  if (act) {
    const int px = mx[0] - mn[0] + 3, py = mx[1] - mn[1] + 3, pz = mx[2] - mn[2] + 3;
    fits = px * py * pz <= kWarpTile && (((mn[0] + px - 1) >> 2) - (mn[0] >> 2) <= 1) &&
           (((mn[1] + py - 1) >> 2) - (mn[1] >> 2) <= 1) &&
           (((mn[2] + pz - 1) >> 2) - (mn[2] >> 2) <= 1);
  }
  const unsigned bad = __ballot_sync(0xffffffffu, act && !fits);
  WarpSeg sg;
  sg.s1 = bad ? __ffs(bad) - 1 : n_live;
#pragma unroll
  for (int a = 0; a < 3; ++a) sg.lo[a] = __shfl_sync(0xffffffffu, mn[a], sg.s1 - 1);
  sg.nx = __shfl_sync(0xffffffffu, mx[0], sg.s1 - 1) - sg.lo[0] + 3;
  sg.ny = __shfl_sync(0xffffffffu, mx[1], sg.s1 - 1) - sg.lo[1] + 3;
  sg.nz = __shfl_sync(0xffffffffu, mx[2], sg.s1 - 1) - sg.lo[2] + 3;
  return sg;
}

// The <= 8 blocks a tile with lower corner lo spans: lane l < 8 resolves block
// lo/4 + (l>>2 & 1, l>>1 & 1, l & 1) through the hash table (-1 if absent);
// the other lanes read them by shuffle (tile_block).
__device__ __forceinline__ int tile_blocks(const GridDev& g, const int (&lo)[3], int lane) {
  int myblk = -1;
  if (lane < 8) {
    int64_t bkey;
    if (pack_block((lo[0] >> 2) + ((lane >> 2) & 1), (lo[1] >> 2) + ((lane >> 1) & 1),
                   (lo[2] >> 2) + (lane & 1), &bkey))
      myblk = hash_find(g.hkeys, g.hvals, g.mask, (uint64_t)bkey);
  }
  return myblk;
}
// tile node q -> (qx, qy, qz) for a tile of nx x ny x nz nodes (z fastest),
// dividing by multiply-shift: exact for q < 4096 and ny, nz <= 15 (a tile
// spans at most 2 blocks, 10 nodes, per axis)
struct TileDiv {
  int ny, nz, my, mz;
};
__device__ __forceinline__ TileDiv tile_div(int ny, int nz) {
  return TileDiv{ny, nz, (65536 + ny - 1) / ny, (65536 + nz - 1) / nz};
}
__device__ __forceinline__ void tile_coords(const TileDiv& d, int q, int& qx, int& qy, int& qz) {
  const int a = (q * d.mz) >> 16;  // q / nz
  qz = q - a * d.nz;
  qx = (a * d.my) >> 16;  // a / ny
  qy = a - qx * d.ny;
}

// block of grid cell (gx, gy, gz) in the tile (all lanes must call)
__device__ __forceinline__ int tile_block(int myblk, const int (&lo)[3], int gx, int gy, int gz) {
  const int bsel = (((gx >> 2) - (lo[0] >> 2)) << 2) | (((gy >> 2) - (lo[1] >> 2)) << 1) |
                   ((gz >> 2) - (lo[2] >> 2));
  return __shfl_sync(0xffffffffu, myblk, bsel & 7);
}

// P2G (mpm.py:66-99 with the stress of materials.py:113-122), warp-level.
// Each warp takes 32 consecutive particles (the fused path sorts particles by
// (block, cell) once per step, so a warp covers a few neighbouring cells):
//   1. the warp's lanes are cut into segments of consecutive particles whose
//      stencils fit a private shared-memory node tile of <= kWarpTile nodes
//      (one segment inside a block, two across a block boundary);
//   2. slot-parallel accumulation (step 4 below): lane k < 27 owns stencil
//      slot k and walks the segment's particles in order, summing runs of
//      same-cell particles in registers and adding them to the tile (one
//      particle's 27 slots are 27 distinct nodes: no atomics, no reduction);
//   3. the tile is flushed with one float64 atomic per node and channel,
//      ~18x fewer global atomics than a per-particle scatter (27 x 7).
constexpr int kP2GThreads = 128;
// per-particle P2G record in shared memory (affine form, see k_p2g step 4):
// m, pad | A (3), Bf (3) | G (9) | K (9) | 1-D weights wx, wy, wz (9) | pad
constexpr int kPayM = 0, kPayA = 2, kPayB = 5, kPayG = 8, kPayK = 17, kPayW = 26;
constexpr int kPayStride = 36;

// the record's first kPayW entries (everything but the weights) with 16 B
// shared-memory loads
template <class T>
__device__ __forceinline__ void load_payload(const T* rec, T (&q)[kPayW]) {
  if constexpr (sizeof(T) == 8) {
#pragma unroll
    for (int k = 0; k < kPayW / 2; ++k) {
      const double2 d2 = reinterpret_cast<const double2*>(rec)[k];
      q[2 * k] = d2.x;
      q[2 * k + 1] = d2.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kPayW / 4; ++k) {
      const float4 f4 = reinterpret_cast<const float4*>(rec)[k];
      q[4 * k] = f4.x;
      q[4 * k + 1] = f4.y;
      q[4 * k + 2] = f4.z;
      q[4 * k + 3] = f4.w;
    }
#pragma unroll
    for (int k = (kPayW / 4) * 4; k < kPayW; ++k) q[k] = rec[k];
  }
}
// Per-particle P2G payload: m, m v, m C, S = -dt D^-1 V0 tau and the external
// impulse dt f of cloth vertex forces.  Cloth roles (cloth.cu): vertex
// particles carry no stress (their in-plane forces arrive in fext), element
// particles carry the transverse stress written by k_cloth_forces.
template <class T>
__device__ __forceinline__ void particle_payload(const ParticlesT<T>& p, long long i, double h,
                                                 double dt, const mpmrb_material* mats, int nmat,
                                                 Stencil1T<T>& s, T& m, T* mv, M3T<T>& mC,
                                                 M3T<T>& S, T* fi, DevStatus* st) {
  double xp[3] = {p.x[3 * i], p.x[3 * i + 1], p.x[3 * i + 2]};
  make_stencil1_t<T>(xp, h, s);
  long long mid = p.mid[i];
  if (mid < 0 || mid >= nmat) {
    raise_status(st, MPMRB_E_INVALID, 21, i);
    mid = 0;
  }
  m = p.mass[i];
  const int role = p.role ? p.role[i] : MPMRB_CLOTH_NONE;
  M3T<T> tau;
  if (role == MPMRB_CLOTH_ELEMENT && p.tau) {
#pragma unroll
    for (int k = 0; k < 9; ++k) tau.a[k] = (T)p.tau[9 * i + k];
  } else if (role != MPMRB_CLOTH_NONE || mats[mid].kind == MPMRB_MAT_CLOTH) {
#pragma unroll
    for (int k = 0; k < 9; ++k) tau.a[k] = T(0);
  } else if (p.tau_cache && mats[mid].kind == MPMRB_MAT_SAND && *p.tau_valid) {
    const T* t6 = p.tau_cache + 6 * i;  // xx yy zz xy xz yz
    tau.a[0] = t6[0];
    tau.a[4] = t6[1];
    tau.a[8] = t6[2];
    tau.a[1] = tau.a[3] = t6[3];
    tau.a[2] = tau.a[6] = t6[4];
    tau.a[5] = tau.a[7] = t6[5];
  } else {
    tau = particle_stress<T>(m3_load(p.f + 9 * i), mats[mid]);
  }
  const double dinv = 4.0 / (h * h);
  const T coef = (T)((-dt * dinv) * (double)p.vol0[i]);
  const M3T<T> C = m3_load(p.c + 9 * i);
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    S.a[k] = coef * tau.a[k];
    mC.a[k] = m * C.a[k];
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    mv[d] = m * p.v[3 * i + d];
    fi[d] = (role == MPMRB_CLOTH_VERTEX && p.fext) ? (T)(dt * p.fext[3 * i + d]) : T(0);
  }
}

// Deterministic P2G (mpm.py:66-99 with mode="deterministic"): the (n, 27, 7)
// per-entry contributions of the reference, materialised in its slot order
// (x-major OFFSETS, mpm.py:25) and channel layout [w m, w (m v + m C dpos),
// w (S dpos)], for the ordered scatter (launch_scatter_reduce_ordered).
__global__ void k_p2g_entries(GridDev g, ParticlesDev p, const mpmrb_material* __restrict__ mats,
                              int nmat, double dt, long long* __restrict__ nodes,
                              double* __restrict__ vals, DevStatus* st) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  Stencil1T<double> s;
  double m, mv[3], fi[3];
  M3 mC, S;
  particle_payload<double>(p, i, g.h, dt, mats, nmat, s, m, mv, mC, S, fi, st);
  StencilBlocks sb;
  if (!resolve_blocks(s, g.hkeys, g.hvals, g.mask, sb)) {
    raise_status(st, MPMRB_E_ALLOCATION, 23, i);
    return;
  }
  const double h = g.h;
  for (int k = 0; k < 27; ++k) {
    const int ox = k / 9, oy = (k / 3) % 3, oz = k % 3;
    const double dp[3] = {(ox - s.fx[0]) * h, (oy - s.fx[1]) * h, (oz - s.fx[2]) * h};
    const double w = (s.w[0][ox] * s.w[1][oy]) * s.w[2][oz];
    nodes[i * 27 + k] = stencil_node(s, sb, ox, oy, oz);
    double* o = vals + (i * 27 + k) * 7;
    o[0] = w * m;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double a = (dp[0] * mC(d, 0) + dp[1] * mC(d, 1)) + dp[2] * mC(d, 2);
      const double b = (dp[0] * S(d, 0) + dp[1] * S(d, 1)) + dp[2] * S(d, 2);
      o[1 + d] = w * (mv[d] + a);
      o[4 + d] = w * (b + fi[d]);
    }
  }
}

__global__ void k_split7(const double* __restrict__ in, long long n, double* __restrict__ mass,
                         double* __restrict__ mom_apic, double* __restrict__ mom_force) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const double* r = in + 7 * q;
    mass[q] = r[0];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      mom_apic[3 * q + d] = r[1 + d];
      mom_force[3 * q + d] = r[4 + d];
    }
  }
}

#ifndef MPMRB_P2G_MINB
// resident CTAs per SM the register budget is sized for: with lane segments
// P2G is faster at 3 (up to 168 registers, no spills; 0.355 -> 0.338 ms at
// 1M), G2P at 4 (0.242 vs 0.268 ms at 3)
#define MPMRB_P2G_MINB 3
#endif
#ifndef MPMRB_G2P_MINB
#define MPMRB_G2P_MINB 4
#endif
// the float32 G2P fits 8 CTAs per SM in 64 registers (a 128 B stack): 0.129
// -> 0.118 ms at 1M against its default 79 registers at 6 CTAs
#ifndef MPMRB_G2P_MINB_F32
#define MPMRB_G2P_MINB_F32 8
#endif
// the float32 P2G fits 5 CTAs per SM (96 registers, 39 KB of tiles each):
// 0.214 -> 0.202 ms at 1M against 121 registers at 4
#ifndef MPMRB_P2G_MINB_F32
#define MPMRB_P2G_MINB_F32 5
#endif
template <class T>
struct P2GMinBlocks {
  static constexpr int value = MPMRB_P2G_MINB;
};
template <>
struct P2GMinBlocks<float> {
  static constexpr int value = MPMRB_P2G_MINB_F32;
};
template <class T>
struct G2PMinBlocks {
  static constexpr int value = MPMRB_G2P_MINB;
};
template <>
struct G2PMinBlocks<float> {
  static constexpr int value = MPMRB_G2P_MINB_F32;
};
template <class T>
__global__ void __launch_bounds__(kP2GThreads, P2GMinBlocks<T>::value) k_p2g(GridDev g, ParticlesT<T> p,
                                                     const mpmrb_material* __restrict__ mats,
                                                     int nmat, double dt,
                                                     double* __restrict__ gmass,
                                                     double* __restrict__ mom_apic,
                                                     double* __restrict__ mom_force,
                                                     DevStatus* st) {
  __shared__ double s_tile[kP2GThreads / 32][7][kWarpTile];
  __shared__ __align__(16) T s_pay[kP2GThreads / 32][16][kPayStride];  // 16 particles' payloads
  __shared__ int s_cell[kP2GThreads / 32][16];  // their base cells' tile node index
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long w0 = ((long long)blockIdx.x * kP2GThreads) + wid * 32;
  if (w0 >= p.n) return;
  const double h = g.h;
  long long i = w0 + lane;
  const bool live = i < p.n;
  const int n_live = (int)min((long long)32, p.n - w0);
  // 1. base cells and this lane's payload (registers)
  int b[3] = {0, 0, 0};
  Stencil1T<T> s;
  T m = T(0), mv[3] = {T(0), T(0), T(0)}, fi[3] = {T(0), T(0), T(0)};
  M3T<T> mC, S;
  if (live) {
    particle_payload<T>(p, i, h, dt, mats, nmat, s, m, mv, mC, S, fi, st);
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a] = (int)s.base[a];
  }
  double (*tile)[kWarpTile] = s_tile[wid];
  const int ox = lane / 9, oy = (lane / 3) % 3, oz = lane % 3;
  const T oxT = T(ox), oyT = T(oy), ozT = T(oz);
  const bool slot_lane = lane < 27;
  // 2. segments of lanes whose stencils fit one node tile (warp_segment)
#pragma unroll 1
  for (int s0 = 0; s0 < n_live;) {
    const bool act = live && lane >= s0;
    const WarpSeg sg = warp_segment(b, live, lane, s0, n_live);
    const int s1 = sg.s1, nx = sg.nx, ny = sg.ny, nz = sg.nz;
    const int lo[3] = {sg.lo[0], sg.lo[1], sg.lo[2]};
    const int nnode = nx * ny * nz;
    const int slot_off = (ox * ny + oy) * nz + oz;  // this slot lane's node from the base cell's
    const TileDiv td = tile_div(ny, nz);
    // 3. zero the segment's node tile
    __syncwarp();
    for (int q = lane; q < nnode; q += 32)
#pragma unroll
      for (int ch = 0; ch < 7; ++ch) tile[ch][q] = 0.0;
    // 4. slot-parallel accumulation: lane k < 27 owns stencil slot k and walks
    // the segment's particles in lane order, adding particle p's 7
    // contributions to node (cell_p + offset_k).  One particle's 27 slots are
    // 27 distinct nodes, so the tile updates need neither atomics nor a
    // reduction, and each node's sum runs in particle order (deterministic).
    // The payloads travel through shared memory in halves of 16 particles, one
    // contiguous record per particle (vector loads), in affine form: with the
    // slot offset o and dpos = (o - fx) h,
    //   m v + mC dpos = A + G o,   S dpos + dt f = Bf + K o,
    // G = h mC, K = h S, A = m v - G fx, Bf = dt f - K fx  (mpm.py:89-93).
    T acc[7];
    int q_run = -1;  // node of the particle run being summed in acc
#pragma unroll 1
    for (int half = s0 >> 4; half <= (s1 - 1) >> 4; ++half) {
      __syncwarp();
      if ((lane >> 4) == half && act) {
        T* rec = s_pay[wid][lane & 15];
        const T hT = (T)h;
        T G[9], K[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          G[k] = hT * mC.a[k];
          K[k] = hT * S.a[k];
        }
        rec[kPayM] = m;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          rec[kPayA + d] = mv[d] - (G[3 * d] * s.fx[0] + G[3 * d + 1] * s.fx[1] + G[3 * d + 2] * s.fx[2]);
          rec[kPayB + d] = fi[d] - (K[3 * d] * s.fx[0] + K[3 * d + 1] * s.fx[1] + K[3 * d + 2] * s.fx[2]);
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          rec[kPayG + k] = G[k];
          rec[kPayK + k] = K[k];
          rec[kPayW + k] = s.w[k / 3][k % 3];
        }
        s_cell[wid][lane & 15] = ((b[0] - lo[0]) * ny + (b[1] - lo[1])) * nz + (b[2] - lo[2]);
      }
      __syncwarp();
      if (slot_lane) {
        // consecutive particles of one cell (sorted order) hit the same node:
        // their contributions are summed in registers and added to the tile
        // when the cell changes (warp-uniform, so one flush writes 27 distinct
        // nodes), which also keeps the tile's read-modify-write chains short
        const int r1 = min(16, s1 - 16 * half);
#pragma unroll 1
        for (int r = max(0, s0 - 16 * half); r < r1; ++r) {
          const T* rec = s_pay[wid][r];
          T q[kPayW];
          load_payload<T>(rec, q);
          const T w = (rec[kPayW + ox] * rec[kPayW + 3 + oy]) * rec[kPayW + 6 + oz];
          T v[7];
          v[0] = w * q[kPayM];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const T* g = q + kPayG + 3 * d;
            const T* k = q + kPayK + 3 * d;
            v[1 + d] = w * (q[kPayA + d] + (g[0] * oxT + g[1] * oyT + g[2] * ozT));
            v[4 + d] = w * (q[kPayB + d] + (k[0] * oxT + k[1] * oyT + k[2] * ozT));
          }
          const int qn = s_cell[wid][r] + slot_off;
          if (qn != q_run) {
            // the run changes on every slot lane at once (the cell changed)
            __syncwarp(0x07ffffffu);
            if (q_run >= 0)
#pragma unroll
              for (int ch = 0; ch < 7; ++ch) tile[ch][q_run] += (double)acc[ch];
#pragma unroll
            for (int ch = 0; ch < 7; ++ch) acc[ch] = v[ch];
            q_run = qn;
          } else {
#pragma unroll
            for (int ch = 0; ch < 7; ++ch) acc[ch] += v[ch];
          }
        }
      }
    }
    if (slot_lane && q_run >= 0)
#pragma unroll
      for (int ch = 0; ch < 7; ++ch) tile[ch][q_run] += (double)acc[ch];
    __syncwarp();
    // 5. flush: one atomic per (node, channel).  The tile spans at most 2
    // blocks per axis (<= 8 blocks, nodes <= 10 per axis): lanes 0-7 resolve
    // one block each through the hash table, the others read them by shuffle.
    const int myblk = tile_blocks(g, lo, lane);
    for (int q0 = 0; q0 < nnode; q0 += 32) {
      const int q = q0 + lane;
      const bool inb = q < nnode;
      int qx = 0, qy = 0, qz = 0;
      if (inb) tile_coords(td, q, qx, qy, qz);
      const int gx = lo[0] + qx, gy = lo[1] + qy, gz = lo[2] + qz;
      const int blk = tile_block(myblk, lo, gx, gy, gz);
      if (!inb) continue;
      double v[7];
      bool any = false;
#pragma unroll
      for (int ch = 0; ch < 7; ++ch) {
        v[ch] = tile[ch][q];
        any |= v[ch] != 0.0;
      }
      if (!any) continue;
      if (blk < 0) {
        raise_status(st, MPMRB_E_ALLOCATION, 22, w0);
        continue;
      }
      const long long node =
          (long long)blk * kNodesPerBlock + (((gx & 3) << 4) | ((gy & 3) << 2) | (gz & 3));
      atomicAdd(&gmass[node], v[0]);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        atomicAdd(&mom_apic[3 * node + d], v[1 + d]);
        atomicAdd(&mom_force[3 * node + d], v[4 + d]);
      }
    }
    s0 = s1;
  }
}

// One thread per allocated node (mpm.py:102-115).  n_nodes = 64*nb from the
// device (nb_dev) when given.
__global__ void k_grid_update(long long n_cap, const int* __restrict__ nb_dev,
                              const double* __restrict__ mass, const double* __restrict__ mom_apic,
                              const double* __restrict__ mom_force, double gx, double gy,
                              double gz, double dt, unsigned char* __restrict__ active,
                              double* __restrict__ v_k, double* __restrict__ v_star,
                              double* __restrict__ v_next, int* __restrict__ warp_count) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long n = nb_dev ? (long long)(*nb_dev) * kNodesPerBlock : n_cap;
  if (n > n_cap) n = n_cap;
  bool act = false;
  if (i < n) {
    double m = mass[i];
    act = m > kMassEps;
    double vk[3] = {0.0, 0.0, 0.0}, vs[3] = {0.0, 0.0, 0.0};
    if (act) {
      double inv_m = 1.0 / m;
      double g[3] = {gx, gy, gz};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        vk[d] = mom_apic[3 * i + d] * inv_m;
        vs[d] = (mom_apic[3 * i + d] + mom_force[3 * i + d]) * inv_m + dt * g[d];
      }
    }
    active[i] = act ? 1 : 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      v_k[3 * i + d] = vk[d];
      v_star[3 * i + d] = vs[d];
      if (v_next) v_next[3 * i + d] = vs[d];  // zero-contact passthrough (coupling.py:125-129)
    }
  }
  if (warp_count) {
    unsigned b = __ballot_sync(0xffffffffu, act);
    if ((threadIdx.x & 31) == 0 && (i - (threadIdx.x & 31)) < n_cap)
      warp_count[i >> 5] = __popc(b);
  }
}

template <class T>
__global__ void __launch_bounds__(128, G2PMinBlocks<T>::value) k_g2p(GridDev g, ParticlesT<T> p,
                                             const mpmrb_material* __restrict__ mats, int nmat,
                                             const double* __restrict__ v_next, double dt,
                                             unsigned long long* __restrict__ clamped,
                                             int* __restrict__ health, DevStatus* st) {
  __shared__ T s_v[128 / 32][3][kWarpTile];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool live = i < p.n;
  bool was_clamped = false;
  const double h = g.h;
  // Warp tile (as in k_p2g): each segment of the warp's sorted particles
  // (warp_segment) gathers from a shared-memory copy of the <= kWarpTile grid
  // velocities its stencils cover, staged with one hash lookup per block.
  const int n_live = (int)max(0LL, min(32LL, p.n - (i - lane)));
  int b[3] = {0, 0, 0};
  double xp[3] = {0.0, 0.0, 0.0};
  Stencil1T<T> s;
  if (live) {
#pragma unroll
    for (int a = 0; a < 3; ++a) xp[a] = p.x[3 * i + a];
    make_stencil1_t<T>(xp, h, s);
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a] = (int)s.base[a];
  }
  T (*tv)[kWarpTile] = s_v[wid];
  const T hT = (T)h;
  T vn[3] = {T(0), T(0), T(0)};
  M3T<T> B;
#pragma unroll
  for (int k = 0; k < 9; ++k) B.a[k] = T(0);
#pragma unroll 1
  for (int s0 = 0; s0 < n_live;) {
    const WarpSeg sg = warp_segment(b, live, lane, s0, n_live);
    const int nx = sg.nx, ny = sg.ny, nz = sg.nz;
    const int lo[3] = {sg.lo[0], sg.lo[1], sg.lo[2]};
    const int myblk = tile_blocks(g, lo, lane);
    const int nnode = nx * ny * nz;
    const TileDiv td = tile_div(ny, nz);
    __syncwarp();  // the previous segment's gathers are done
    for (int q0 = 0; q0 < nnode; q0 += 32) {
      const int q = q0 + lane;
      const bool inb = q < nnode;
      int qx = 0, qy = 0, qz = 0;
      if (inb) tile_coords(td, q, qx, qy, qz);
      const int gx = lo[0] + qx, gy = lo[1] + qy, gz = lo[2] + qz;
      const int blk = tile_block(myblk, lo, gx, gy, gz);
      if (!inb) continue;
      // nodes outside the allocated blocks are never in a live stencil
      const long long node =
          (long long)(blk < 0 ? 0 : blk) * kNodesPerBlock + (((gx & 3) << 4) | ((gy & 3) << 2) | (gz & 3));
#pragma unroll
      for (int d = 0; d < 3; ++d) tv[d][q] = blk < 0 ? T(0) : (T)v_next[3 * node + d];
    }
    __syncwarp();
    if (live && lane >= s0 && lane < sg.s1) {
      const int cbq = ((b[0] - lo[0]) * ny + (b[1] - lo[1])) * nz + (b[2] - lo[2]);
#pragma unroll 1
      for (int ox = 0; ox < 3; ++ox) {
        const T dx = (T(ox) - s.fx[0]) * hT;
#pragma unroll 1
        for (int oy = 0; oy < 3; ++oy) {
          const T dy = (T(oy) - s.fx[1]) * hT;
          const T wxy = s.w[0][ox] * s.w[1][oy];
          const int qxy = cbq + (ox * ny + oy) * nz;
#pragma unroll
          for (int oz = 0; oz < 3; ++oz) {
            const T dz = (T(oz) - s.fx[2]) * hT;
            const T w = wxy * s.w[2][oz];
            const int q = qxy + oz;
            T wv[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              wv[d] = w * tv[d][q];
              vn[d] += wv[d];
              B(d, 0) += wv[d] * dx;
              B(d, 1) += wv[d] * dy;
              B(d, 2) += wv[d] * dz;
            }
          }
        }
      }
    }
    s0 = sg.s1;
  }
  if (live) {
    {
      const T dinv = (T)(4.0 / (h * h));
      M3T<T> C;
#pragma unroll
      for (int k = 0; k < 9; ++k) C.a[k] = dinv * B.a[k];
      M3T<T> A = m3_identity<T>();
      const T dtT = (T)dt;
#pragma unroll
      for (int k = 0; k < 9; ++k) A.a[k] += dtT * C.a[k];
      const bool cloth = p.role && p.role[i] != MPMRB_CLOTH_NONE;
      M3T<T> F = m3_load(p.f + 9 * i);
      if (!cloth) {  // cloth particles carry no F (cloth.cu: d3 per element)
        F = m3_mul(A, F);
        if (!(m3_det(F) > T(0)) || !m3_finite(F)) {
          F = clamp_singular_values(F);
          was_clamped = true;
        }
      }
      long long mid = p.mid[i];
      if (!cloth && mid >= 0 && mid < nmat && mats[mid].kind == MPMRB_MAT_SAND) {
        T dq = T(0);
        const T mu = (T)mats[mid].mu, lam = (T)mats[mid].lam, al = (T)mats[mid].dp_alpha;
        if (p.tau_cache) {
          M3T<T> t;
          F = dp_return_map_tau<T>(F, mu, lam, al, &dq, &t);
          T* t6 = p.tau_cache + 6 * i;
          t6[0] = t.a[0];
          t6[1] = t.a[4];
          t6[2] = t.a[8];
          t6[3] = t.a[1];
          t6[4] = t.a[2];
          t6[5] = t.a[5];
        } else {
          F = dp_return_map<T>(F, mu, lam, al, &dq);
        }
        if (p.plastic) p.plastic[i] += dq;
      }
      double xn[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        xn[d] = xp[d] + dt * (double)vn[d];
        p.x[3 * i + d] = xn[d];
        p.v[3 * i + d] = vn[d];
      }
      m3_store(p.c + 9 * i, C);
      m3_store(p.f + 9 * i, F);
      if (health) {
        const double lim = h * (double)((1 << 20) - 2);
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d)
          ok &= isfinite(xn[d]) && isfinite(vn[d]) && fabs(xn[d]) < lim;
        if (!ok) atomicOr(health, 1);
      }
    }
  }
  if (p.tau_valid && blockIdx.x == 0 && threadIdx.x == 0) *p.tau_valid = 1;  // read by the next P2G
  if (clamped) {
    unsigned b = __ballot_sync(0xffffffffu, was_clamped);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(clamped, (unsigned long long)__popc(b));
  }
}

__global__ void k_clamp(const double* __restrict__ f, long long n, double* __restrict__ out,
                        unsigned long long* __restrict__ nbad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < n) {
    M3 F = m3_load(f + 9 * i);
    bad = !(m3_det(F) > 0.0) || !m3_finite(F);
    if (bad) F = clamp_singular_values(F);
    m3_store(out + 9 * i, F);
  }
  unsigned b = __ballot_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(nbad, (unsigned long long)__popc(b));
}

// materials.py:57-83 on a stack of 3x3 matrices: the Higham polar rotation
// (per-matrix stop, see svd3.cuh) or the adjugate inverse-transpose.
__global__ void k_polar(const double* __restrict__ f, long long n, int inv_t_only,
                        double* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const M3 F = m3_load(f + 9 * i);
  m3_store(out + 9 * i, inv_t_only ? m3_inv_transpose(F) : polar_rotation(F));
}

// coupling.py:153-165: finite x, v and |x| < h (2^20 - 2)
__global__ void k_health(const double* __restrict__ x, const double* __restrict__ v, long long n,
                         double lim, int* __restrict__ bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  double xi = x[i], vi = v[i];
  if (!(isfinite(xi) && isfinite(vi) && fabs(xi) < lim)) atomicOr(bad, 1);
}

}  // namespace

int launch_health(Ctx& c, const double* x, const double* v, long long n, double h, int* bad) {
  if (n == 0) return MPMRB_OK;
  k_health<<<grid_for(3 * n, 256), 256, 0, c.stream>>>(x, v, n, h * (double)((1 << 20) - 2), bad);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_polar(Ctx& c, const double* f, long long n, int inv_t_only, double* out) {
  if (n == 0) return MPMRB_OK;
  k_polar<<<grid_for(n, 128), 128, 0, c.stream>>>(f, n, inv_t_only, out);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_clamp(Ctx& c, const double* f, long long n, double* out, unsigned long long* nbad) {
  MPMRB_CUDA_OK(cudaMemsetAsync(nbad, 0, 8, c.stream));
  if (n == 0) return MPMRB_OK;
  k_clamp<<<grid_for(n, 128), 128, 0, c.stream>>>(f, n, out, nbad);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_scatter_reduce(Ctx& c, const long long* ids, const double* vals, long long rows,
                          long long k, long long nch, long long n_out, double* out) {
  MPMRB_CUDA_OK(cudaMemsetAsync(out, 0, sizeof(double) * n_out * nch, c.stream));
  if (rows * k == 0) return MPMRB_OK;
  k_scatter_reduce<<<grid_for(rows * k, 256), 256, 0, c.stream>>>(ids, vals, rows, k, nch, n_out,
                                                                  out, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_scatter_reduce_ordered(Ctx& c, const long long* ids, const double* vals,
                                  long long rows, long long k, long long nch, long long n_out,
                                  double* out) {
  const long long e_n = rows * k;
  if (n_out == 0) return MPMRB_OK;
  if (e_n == 0) {
    MPMRB_CUDA_OK(cudaMemsetAsync(out, 0, sizeof(double) * n_out * nch, c.stream));
    return MPMRB_OK;
  }
  if (e_n >= (1LL << 31) || n_out >= (1LL << 31))
    return set_error(MPMRB_E_INVALID, "ordered scatter: %lld entries / %lld nodes exceed int32",
                     e_n, n_out);
  // scratch: keys 2 e_n (u32), idx 3 e_n (i32), seg_start n_out + 1 (i64)
  if (c.scratch[SS_ORD_K].grow(sizeof(unsigned) * 2 * e_n) ||
      c.scratch[SS_ORD_I].grow(sizeof(int) * 3 * e_n) ||
      c.scratch[SS_ORD_S].grow(sizeof(long long) * (n_out + 1)))
    return MPMRB_E_CUDA;
  unsigned* keys = c.scratch[SS_ORD_K].as<unsigned>();
  int* idx = c.scratch[SS_ORD_I].as<int>();
  long long* seg = c.scratch[SS_ORD_S].as<long long>();
  k_ordered_keys<<<grid_for(e_n, 256), 256, 0, c.stream>>>(ids, e_n, n_out, keys, idx, c.status);
  c.launches++;
  int bits = 1;
  while ((1LL << bits) < n_out) ++bits;
  unsigned* skeys = nullptr;
  int rc = sort_pairs_u32(c, keys, idx, keys + e_n, idx + e_n, e_n, bits, idx + 2 * e_n, &skeys);
  if (rc) return rc;
  k_ordered_bounds<<<grid_for(e_n + 1, 256), 256, 0, c.stream>>>(skeys, e_n, n_out, seg);
  c.launches++;
  const int* sidx = idx + 2 * e_n;
  const unsigned g = grid_for(n_out, 128);
  switch (nch) {
    case 1: k_ordered_sum<1><<<g, 128, 0, c.stream>>>(sidx, seg, vals, n_out, nch, out); break;
    case 3: k_ordered_sum<3><<<g, 128, 0, c.stream>>>(sidx, seg, vals, n_out, nch, out); break;
    case 7: k_ordered_sum<7><<<g, 128, 0, c.stream>>>(sidx, seg, vals, n_out, nch, out); break;
    case 9: k_ordered_sum<9><<<g, 128, 0, c.stream>>>(sidx, seg, vals, n_out, nch, out); break;
    default: k_ordered_sum<0><<<g, 128, 0, c.stream>>>(sidx, seg, vals, n_out, nch, out); break;
  }
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_stresses(Ctx& c, const double* f, const long long* mid, long long n,
                    const mpmrb_material* mats_dev, int nmat, double* tau) {
  if (n == 0) return MPMRB_OK;
  k_stresses<<<grid_for(n, 128), 128, 0, c.stream>>>(f, mid, n, mats_dev, nmat, tau, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

template <class T>
int launch_p2g_t(Ctx& c, const GridDev& g, const ParticlesT<T>& p, const mpmrb_material* mats_dev,
                 int nmat, double dt, double* mass, double* mom_apic, double* mom_force) {
  if (p.n == 0) return MPMRB_OK;
  k_p2g<T><<<grid_for(p.n, kP2GThreads), kP2GThreads, 0, c.stream>>>(
      g, p, mats_dev, nmat, dt, mass, mom_apic, mom_force, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}
int launch_p2g(Ctx& c, const GridDev& g, const ParticlesDev& p, const mpmrb_material* mats_dev,
               int nmat, double dt, double* mass, double* mom_apic, double* mom_force) {
  return launch_p2g_t<double>(c, g, p, mats_dev, nmat, dt, mass, mom_apic, mom_force);
}
int launch_p2g(Ctx& c, const GridDev& g, const ParticlesF32& p, const mpmrb_material* mats_dev,
               int nmat, double dt, double* mass, double* mom_apic, double* mom_force) {
  return launch_p2g_t<float>(c, g, p, mats_dev, nmat, dt, mass, mom_apic, mom_force);
}

int launch_p2g_ordered(Ctx& c, const GridDev& g, const ParticlesDev& p,
                       const mpmrb_material* mats_dev, int nmat, double dt, long long n_nodes,
                       double* mass, double* mom_apic, double* mom_force) {
  if (p.n == 0 || n_nodes == 0) {
    if (n_nodes) {
      MPMRB_CUDA_OK(cudaMemsetAsync(mass, 0, 8 * n_nodes, c.stream));
      MPMRB_CUDA_OK(cudaMemsetAsync(mom_apic, 0, 24 * n_nodes, c.stream));
      MPMRB_CUDA_OK(cudaMemsetAsync(mom_force, 0, 24 * n_nodes, c.stream));
    }
    return MPMRB_OK;
  }
  const long long e_n = p.n * 27;
  if (c.scratch[SS_ORD_N].grow(sizeof(long long) * e_n) ||
      c.scratch[SS_ORD_V].grow(sizeof(double) * 7 * e_n) ||
      c.scratch[SS_ORD_O].grow(sizeof(double) * 7 * n_nodes))
    return MPMRB_E_CUDA;
  long long* nodes = c.scratch[SS_ORD_N].as<long long>();
  double* vals = c.scratch[SS_ORD_V].as<double>();
  double* out7 = c.scratch[SS_ORD_O].as<double>();
  k_p2g_entries<<<grid_for(p.n, 128), 128, 0, c.stream>>>(g, p, mats_dev, nmat, dt, nodes, vals,
                                                         c.status);
  c.launches++;
  int rc = launch_scatter_reduce_ordered(c, nodes, vals, p.n, 27, 7, n_nodes, out7);
  if (rc) return rc;
  k_split7<<<grid_for(n_nodes, 256), 256, 0, c.stream>>>(out7, n_nodes, mass, mom_apic, mom_force);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_grid_update(Ctx& c, long long n_cap, const int* nb_dev, const double* mass,
                       const double* mom_apic, const double* mom_force, double gx, double gy,
                       double gz, double dt, unsigned char* active, double* v_k, double* v_star,
                       double* v_next, int* warp_count) {
  if (n_cap == 0) return MPMRB_OK;
  k_grid_update<<<grid_for(n_cap, 256), 256, 0, c.stream>>>(n_cap, nb_dev, mass, mom_apic,
                                                            mom_force, gx, gy, gz, dt, active,
                                                            v_k, v_star, v_next, warp_count);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

template <class T>
int launch_g2p_t(Ctx& c, const GridDev& g, const ParticlesT<T>& p, const mpmrb_material* mats_dev,
                 int nmat, const double* v_next, double dt, unsigned long long* clamped_dev,
                 int* health_dev) {
  if (p.n == 0) return MPMRB_OK;
  k_g2p<T><<<grid_for(p.n, 128), 128, 0, c.stream>>>(g, p, mats_dev, nmat, v_next, dt,
                                                     clamped_dev, health_dev, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}
int launch_g2p(Ctx& c, const GridDev& g, const ParticlesDev& p, const mpmrb_material* mats_dev,
               int nmat, const double* v_next, double dt, unsigned long long* clamped_dev,
               int* health_dev) {
  return launch_g2p_t<double>(c, g, p, mats_dev, nmat, v_next, dt, clamped_dev, health_dev);
}
int launch_g2p(Ctx& c, const GridDev& g, const ParticlesF32& p, const mpmrb_material* mats_dev,
               int nmat, const double* v_next, double dt, unsigned long long* clamped_dev,
               int* health_dev) {
  return launch_g2p_t<float>(c, g, p, mats_dev, nmat, v_next, dt, clamped_dev, health_dev);
}

}  // namespace mpmrb
