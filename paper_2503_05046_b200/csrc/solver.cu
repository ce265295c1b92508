// Globally convergent quasi-Newton convex contact solve on sm_100a
// (solver.py:197-382), run entirely on the device as ONE persistent
// cooperative kernel: no host round trip per iteration or per line-search
// evaluation.
//
// Structure (v5).
//  * Free nodes (active nodes no contact stencil touches) have g = m(v - v*),
//    H = m I, so dv = -(v - v*) and v - v* shrinks by (1 - alpha) per step.
//    Their whole contribution to every reduction is a closed form in
//    P = prod(1 - alpha) and three sums taken once (S0, Q0, Q1 below); they
//    are written once, in the epilogue, as v = v* + P (v0 - v*).  The
//    iteration only touches contact nodes and contacts.
//  * Each contact owner writes one 80 B record per iteration: R^T g_c and
//    R^T G_c R.  Each contact node gathers the records of the contacts whose
//    stencil holds it, weighted by w and w^2 of its slot, through a sorted CSR
//    of (contact run, slot) entries (the contacts of one grid cell share all
//    27 nodes and form one run).  Fixed summation order (ascending contact id
//    per node), no atomics: a solve is bitwise reproducible run to run.  (v4
//    summed w R^T g per (run, slot) in the contact phase instead: 27 records
//    per run, ~100 MB written and read per iteration at 1M particles.)
//  * The exact line search (solver.py:266-298) runs on a small group of CTAs
//    (sized to the contact count) whose all-reduces use fence-free
//    self-validating slots (~1 us for 16 CTAs vs ~3 us for a 148-CTA grid
//    sync, tools/reduce_bench.cu).  Each evaluation is closed form per contact:
//    one rsqrt, no division.
//
// Phases per iteration (solver.py:338-357):
//   N  contact nodes: pending v += alpha dv, gather records -> J^T g and the
//      Hessian block, gradient, residual/norms, 3x3 Cholesky -> dv, a1, a2;
//      free-node terms in closed form                         [grid reduce]
//   D  contacts: dvc = R J dv and phi'(0)            [gather to the LS group]
//   LS group: <= ls_max evaluations                [group reduce each]
//      -> alpha broadcast to every CTA
//   U  contacts: vc += alpha dvc, contact gradient/Hessian -> records
//                                                             [grid sync]
//
// vc is advanced as vc + alpha dvc (= R J (v + alpha dv) + b exactly in real
// arithmetic) instead of being re-gathered from v; the difference is roundoff.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "contact.cuh"
#include "internal.h"
#include "solver.cuh"

namespace mpmrb {

namespace {

constexpr int kThreads = kSolverThreads;
constexpr int kChunk = 32;        // contacts per ownership chunk: one warp, one contact per lane
constexpr int kWarps = kThreads / 32;
constexpr int kSwStride = 33;  // staged weights sw[k * 33 + lane]: rows padded (bank conflicts)
constexpr int kMaxRed = 8;        // reduction lanes per grid reduce
// contacts per line-search thread held in registers (= the contacts per thread
// the group is sized for, so no dead slots; 3 and 5 measured slower at 2M)
constexpr int kLS = 4;
constexpr int kEPL = 4;  // phase N: adjacency entries per lane in flight (no spills at 4)

// slot areas (64-bit words), see kSolverSlotWords
constexpr long long kSlotA = 0;                                  // [2][ctas][6]  gather (3 values)
constexpr long long kSlotB = kSlotA + 2LL * kMaxSolverCtas * 6;  // [2][ctas][4]  group (2 values)
constexpr long long kSlotC = kSlotB + 2LL * kMaxSolverCtas * 4;  // [2][4]        broadcast (2)

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------ self-validating slots
// A double is published as two 64-bit words (tag << 32 | half).  64-bit
// aligned stores are single-copy atomic, so a reader that sees the current
// tag in both words has the complete, current value: no fence or flag
// ordering is needed for the scalars themselves.  Tags advance by one per use
// of a channel and persist across solves (SolverArgs::chan).
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// release / acquire fences at GPU scope (lighter than __threadfence's fence.sc)
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int K>
__device__ __forceinline__ void slot_publish(unsigned long long* slot, const double* v,
                                             unsigned tag) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[k]);
    const unsigned long long t = (unsigned long long)tag << 32;
    st_relaxed(slot + 2 * k, t | (b >> 32));
    st_relaxed(slot + 2 * k + 1, t | (b & 0xffffffffull));
  }
}

// Warp-wide: wait for n slots (<= 32*PER) of K doubles carrying `tag`, and
// sum them in slot order (lane-strided partials then a butterfly: the same
// order in every CTA, so all CTAs get bitwise-identical sums).
template <int K, int PER, int SLEEP_NS = 0>
__device__ __forceinline__ void slot_poll_sum(const unsigned long long* slots, int n,
                                              unsigned tag, double* out) {
  const int lane = threadIdx.x & 31;
  unsigned long long w[PER][2 * K];
  bool ok;
  do {
    ok = true;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int s = lane + 32 * r;
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) {
        w[r][j] = (s < n) ? ld_relaxed(slots + (long long)s * 2 * K + j)
                          : ((unsigned long long)tag << 32);
        ok &= (unsigned)(w[r][j] >> 32) == tag;
      }
    }
    if (SLEEP_NS > 0 && !__all_sync(0xffffffffu, ok)) __nanosleep(SLEEP_NS);
  } while (!__all_sync(0xffffffffu, ok));
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < PER; ++r)
      acc += __longlong_as_double((long long)(((w[r][2 * k] & 0xffffffffull) << 32) |
                                              (w[r][2 * k + 1] & 0xffffffffull)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    out[k] = acc;
  }
}

// ------------------------------------------------------------ grid reductions
// Grid barrier on a monotonic arrival counter: every CTA adds 1 (release)
// and polls, with a short sleep, until all arrivals of this barrier have
// landed (acquire).  No reset and no release hop by a last arriver; the
// counter's value at the barrier's start persists across solves (chan[3]).
// cg::this_grid().sync() spins every CTA on the arrival word itself, which
// under load delayed the release by ~10 us (tools/solver_scaling.py).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Sync {
  double* partials;  // [2][kMaxRed][kMaxSolverCtas]
  int nctas;
  unsigned long long* prof;  // CTA 0 / thread 0 only: [10] time inside grid syncs
  unsigned long long* cta_in_sync;  // thread 0 of each CTA (profiling only)
  unsigned* bar;     // [0] monotonic arrival count
  unsigned* gen;     // the count at this barrier's start (thread 0)
  __device__ __forceinline__ void operator()() const {
    if (nctas == 1) {
      __syncthreads();
      return;
    }
    unsigned long long t0 = (prof || cta_in_sync) ? gtime() : 0ull;
    __syncthreads();
    if (threadIdx.x == 0) {
const unsigned target = *gen + (unsigned)nctas;
      red_release_add_u32(bar, 1u);
      while ((int)(ld_acquire_u32(bar) - target) < 0) __nanosleep(32);
      *gen = target;
    }
    __syncthreads();
    if (prof) atomicAdd(prof + 10, gtime() - t0);
    if (cta_in_sync) *cta_in_sync += gtime() - t0;
  }
};

// Block sum of K values into sm[32*kMaxRed + k] (valid after the call's
// trailing barrier in every thread of the CTA).
template <int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], double* sm, double* res) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sm[k * 32 + wid] = x;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = (lane < kThreads / 32) ? sm[k * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      res[k] = x;  // every lane of warp 0 holds the block sum
    }
  }
}

// Sum K values over all threads of all participating CTAs through a grid
// sync; every thread receives the totals.  Partials are double-buffered: a
// CTA racing into the next reduction writes the other half while slower CTAs
// still read this one, and the grid sync inside the next reduction closes the
// window.  The sync also orders all prior global writes (data barrier).
template <int K>
__device__ void reduce_all(const Sync& sync, int& parity, double (&v)[K], double (&out)[K],
                           double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* part = sync.partials + parity * (kMaxRed * kMaxSolverCtas);
  parity ^= 1;
  double bs[K];
  block_reduce<K>(v, sm, bs);
  if (wid == 0 && lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (sync.nctas == 1) sm[32 * kMaxRed + k] = bs[k];
      else part[k * kMaxSolverCtas + blockIdx.x] = bs[k];
    }
  }
  if (sync.nctas > 1) {
    sync();
    if (wid == 0) {
      constexpr int kR = (kMaxSolverCtas + 31) / 32;
      double x[K][kR];
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int c = lane + 32 * r;
          x[k][r] = (c < sync.nctas) ? __ldcg(&part[k * kMaxSolverCtas + c]) : 0.0;
        }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double s = x[k][0];
#pragma unroll
        for (int r = 1; r < kR; ++r) s += x[k][r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sm[32 * kMaxRed + k] = s;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = sm[32 * kMaxRed + k];
  __syncthreads();
}

// All-reduce of K values over the line-search group (CTAs 0..G-1) through
// channel B slots; G == 1 is a plain block reduction.
// The result goes through one of two shared-memory buffers (alternating per
// call, `rpar`), so no trailing barrier is needed before the next call.
template <int K>
__device__ void group_reduce(int G, unsigned long long* slots, unsigned& tag, double (&v)[K],
                             double (&out)[K], double* sm, unsigned& rpar) {
  double* res = sm + 32 * kMaxRed + 4 * (rpar & 1u);
  ++rpar;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double bs[K];
  block_reduce<K>(v, sm, bs);
  if (wid == 0) {
    if (G == 1) {
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = bs[k];
    } else {
      unsigned long long* base = slots + kSlotB + (long long)(tag & 1u) * kMaxSolverCtas * 4;
      if (lane == 0) slot_publish<K>(base + (long long)blockIdx.x * 2 * K, bs, tag);
      double r[K];
      slot_poll_sum<K, 2>(base, G, tag, r);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = r[k];
    }
  }
  if (G > 1) ++tag;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = res[k];
}

__device__ __forceinline__ void load_frame(const double* fr, long long c, double* R) {
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(fr + 9 * c + k);
}

// R (sum_k w_k u[node_k]); dead slots (node < 0) carry w = 0 and add nothing.
// All 27 node indices are loaded first and the value loads carry no branch,
// so the whole gather costs two dependent memory round trips (a branch on each
// loaded index serialised 27 of them).  Weights come from global memory
// (slot-major) or, when staged, from shared memory sw[k * kSwStride + lane].
// u is written by other CTAs earlier in this kernel (ordered by a grid sync,
// which also invalidates L1): plain coherent loads, no __restrict__ (that would
// allow the non-coherent path) and no volatile asm (__ldcg would pin the loads
// in program order behind the FMAs that consume them).
template <bool kStaged>
__device__ __forceinline__ void gather_contact_t(const SolverArgs& a, long long c,
                                                 const double* u, const double* R,
                                                 const double* sw, int lane, double* out) {
  int nd[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) nd[k] = __ldg(&a.cnodes[(long long)k * a.nc_cap + c]);
  double up[3] = {0.0, 0.0, 0.0};
  // three batches of nine slots: 27 value loads in flight per batch (register
  // budget), i.e. one index round trip + three value round trips in total
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    double x[9], y[9], z[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int k = 9 * b + q;
      const long long j = 3LL * (nd[k] >= 0 ? nd[k] : 0);
      x[q] = u[j];
      y[q] = u[j + 1];
      z[q] = u[j + 2];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int k = 9 * b + q;
      const double w = kStaged ? sw[k * kSwStride + lane] : __ldg(&a.cw[(long long)k * a.nc_cap + c]);
      if (nd[k] >= 0) {
        up[0] += w * x[q];
        up[1] += w * y[q];
        up[2] += w * z[q];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) out[r] = R[3 * r] * up[0] + R[3 * r + 1] * up[1] + R[3 * r + 2] * up[2];
}

__device__ __forceinline__ void gather_contact(const SolverArgs& a, long long c, const double* u,
                                               const double* R, double* out) {
  gather_contact_t<false>(a, c, u, R, nullptr, 0, out);
}
__device__ __forceinline__ void gather_contact_sw(const SolverArgs& a, long long c,
                                                  const double* u, const double* R,
                                                  const double* sw, int lane, double* out) {
  gather_contact_t<true>(a, c, u, R, sw, lane, out);
}

// Stage the 27 stencil weights of the warp's chunk [c0, c0 + 32) into
// sw[k * kSwStride + lane] (slot-major loads, coalesced, all in flight at once).
__device__ __forceinline__ void stage_weights(const SolverArgs& a, long long c0, int nc,
                                              double* sw) {
  const int lane = threadIdx.x & 31;
  const long long c = c0 + lane;
  double w[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) w[k] = (c < nc) ? __ldg(&a.cw[(long long)k * a.nc_cap + c]) : 0.0;
#pragma unroll
  for (int k = 0; k < 27; ++k) sw[k * kSwStride + lane] = w[k];
  __syncwarp();
}

// From vc: world gradient gw = R^T g_c, Hessian block R^T G R (6 entries used
// by the Cholesky) and the contact energy (solver.py:111-167).
__device__ __forceinline__ double contact_terms(const ContactModel& cm, const double* vc,
                                                double vhat, double mug, const double* R,
                                                double* gw, double* rgr) {
  double g[3], G[4];
  const double energy = cm_eval(cm, vc, vhat, mug, g, G);
#pragma unroll
  for (int j = 0; j < 3; ++j) gw[j] = g[0] * R[j] + g[1] * R[3 + j] + g[2] * R[6 + j];
  double GR[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    GR[j] = G[0] * R[j] + G[3] * R[3 + j];
    GR[3 + j] = G[3] * R[j] + G[1] * R[3 + j];
    GR[6 + j] = G[2] * R[6 + j];
  }
  const int ri[6] = {0, 1, 2, 1, 2, 2}, rj[6] = {0, 1, 2, 0, 0, 1};
#pragma unroll
  for (int e = 0; e < 6; ++e)
    rgr[e] = R[ri[e]] * GR[rj[e]] + R[3 + ri[e]] * GR[3 + rj[e]] + R[6 + ri[e]] * GR[6 + rj[e]];
  return energy;
}

// Line-search derivative terms of one contact at step alpha (solver.py:
// 266-325 with contact_model.py:75-111 along the line): adds g_c.dvc to d1 and
// dvc^T G_c dvc to d2.  Closed form: one rsqrt, no division.
__device__ __forceinline__ void ls_terms(const ContactModel& cm, double inv_eps, const double* vc,
                                         const double* dvc, double vhat, double mug,
                                         double alpha, double& d1, double& d2) {
  const double gap = vhat - (vc[2] + alpha * dvc[2]);
  d1 -= (cm.K * fmax(0.0, gap)) * dvc[2];
  if (gap >= 0.0) d2 += cm.K * (dvc[2] * dvc[2]);
  const double t0 = vc[0] + alpha * dvc[0], t1 = vc[1] + alpha * dvc[1];
  const double s2 = t0 * t0 + t1 * t1;
  const double td = t0 * dvc[0] + t1 * dvc[1];
  const double dd = dvc[0] * dvc[0] + dvc[1] * dvc[1];
  if (s2 > cm.eps_v * cm.eps_v) {
    const double r = rsqrt(s2);
    const double av = mug * r;
    d1 += av * td;
    d2 += av * (dd - (r * r) * (td * td));
  } else {
    const double av = mug * inv_eps;
    d1 += av * td;
    d2 += av * dd;
  }
}

// The same with the per-line-search constants of a contact precomputed
// (LsRec): gap0 = vhat - vc_n, dvn, K dvn^2, |dvt|^2, mu gamma_lag.
struct LsRec {
  double t0, t1, d0, d1, gap0, dvn, kdvn2, dd, mug;
};
__device__ __forceinline__ LsRec ls_rec(const ContactModel& cm, const double* vc,
                                        const double* dvc, double vhat, double mug) {
  LsRec r;
  r.t0 = vc[0];
  r.t1 = vc[1];
  r.d0 = dvc[0];
  r.d1 = dvc[1];
  r.gap0 = vhat - vc[2];
  r.dvn = dvc[2];
  r.kdvn2 = cm.K * (dvc[2] * dvc[2]);
  r.dd = dvc[0] * dvc[0] + dvc[1] * dvc[1];
  r.mug = mug;
  return r;
}
__device__ __forceinline__ void ls_terms_rec(const ContactModel& cm, double eps2, double inv_eps,
                                             const LsRec& c, double alpha, double& d1,
                                             double& d2) {
  const double kdvn2 = c.kdvn2, cdd = c.dd;
  const double gap = c.gap0 - alpha * c.dvn;
  if (gap > 0.0) d1 -= (cm.K * gap) * c.dvn;
  if (gap >= 0.0) d2 += kdvn2;
  const double t0 = c.t0 + alpha * c.d0, t1 = c.t1 + alpha * c.d1;
  const double s2 = t0 * t0 + t1 * t1;
  const double td = t0 * c.d0 + t1 * c.d1;
  if (s2 > eps2) {
    const double r = rsqrt(s2);
    const double av = c.mug * r;
    d1 += av * td;
    d2 += av * (cdd - (r * r) * (td * td));
  } else {
    const double av = c.mug * inv_eps;
    d1 += av * td;
    d2 += av * cdd;
  }
}

// Per-node part of phase N given the gathered jt (3) and Hessian sums hs (6):
// gradient, residual/norm/energy partials, regularised 3x3 Cholesky
// (solver.py:224-256), direction dv and the line-search coefficients.
struct NodeIn {
  double m, v[3], vs[3];
};

__device__ __forceinline__ void node_finish(const SolverArgs& a, long long i, const NodeIn& nin,
                                            const double* jt, const double* hs, double* red,
                                            int& reg_count) {
  const double m = nin.m;
  const double inv_m = 1.0 / m;
  double dvs[3], g[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double vi = nin.v[d];
    dvs[d] = vi - nin.vs[d];
    g[d] = m * dvs[d] + jt[d];
    red[0] += g[d] * g[d] * inv_m;
    red[1] += m * vi * vi;
    red[2] += jt[d] * jt[d] * inv_m;
    red[3] += m * dvs[d] * dvs[d];
  }
  double h[6] = {m + hs[0], m + hs[1], m + hs[2], hs[3], hs[4], hs[5]};
  double l11 = 0, l21 = 0, l31 = 0, l22 = 0, l32 = 0, l33 = 0;
  bool good = false;
  for (int attempt = 0; attempt < 4; ++attempt) {
    l11 = sqrt(h[0]);
    l21 = h[3] / l11;
    l31 = h[4] / l11;
    l22 = sqrt(h[1] - l21 * l21);
    l32 = (h[5] - l31 * l21) / l22;
    l33 = sqrt(h[2] - l31 * l31 - l32 * l32);
    good = isfinite(l11) && isfinite(l22) && isfinite(l33) && l11 > 0.0 && l22 > 0.0 &&
           l33 > 0.0;
    if (good || attempt == 3) break;
    ++reg_count;
    const double tr = h[0] + h[1] + h[2];
    const double bump = 1e-12 * fmax(tr, 1.0) * (attempt == 0 ? 1.0 : (attempt == 1 ? 10.0 : 100.0));
    h[0] += bump;
    h[1] += bump;
    h[2] += bump;
  }
  if (!good) red[7] = 1.0;
  const double y1 = -g[0] / l11;
  const double y2 = (-g[1] - l21 * y1) / l22;
  const double y3 = (-g[2] - l31 * y1 - l32 * y2) / l33;
  const double x3 = y3 / l33;
  const double x2 = (y2 - l32 * x3) / l22;
  const double x1 = (y1 - l21 * x2 - l31 * x3) / l11;
  const double dvv[3] = {x1, x2, x3};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    a.dv[3 * i + d] = dvv[d];
    const double mdv = m * dvv[d];
    red[5] += dvs[d] * mdv;
    red[6] += dvv[d] * mdv;
  }
}

// Phase U (and the init) on one warp chunk of contacts [c0, c0 + 32), one
// contact per lane: new contact velocity, then the contact's record for the
// node gathers of the next N phase -- world gradient R^T g_c (3) and Hessian
// block R^T G_c R (6) -- and its energy.  The stencil weight is applied by the
// gathering node (w and w^2 per (contact, slot)), so a contact's record is
// written once instead of once per stencil slot.
__device__ __forceinline__ void contact_update_chunk(const SolverArgs& a, const ContactModel& cm,
                                                     long long c0, int nc, bool init,
                                                     double alpha, const double* s_w,
                                                     double& e_acc) {
  const int lane = threadIdx.x & 31;
  const long long c = c0 + lane;
  if (c >= nc) return;
  double R[9], vc[3], gw[3], rgr[6], vhat, mug;
  load_frame(a.frames, c, R);
  if (init) {
    gather_contact_sw(a, c, a.v0, R, s_w, lane, vc);
#pragma unroll
    for (int d = 0; d < 3; ++d) vc[d] += a.bias[3 * c + d];
    vhat = -a.phi[c] / cm.den;
    mug = a.mu[c] * a.gamma_lag[c];
    a.cvhat[c] = vhat;
    a.cmug[c] = mug;
  } else {
#pragma unroll
    for (int d = 0; d < 3; ++d) vc[d] = a.vc[3 * c + d] + alpha * a.dvc[3 * c + d];
    vhat = a.cvhat[c];
    mug = a.cmug[c];
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) a.vc[3 * c + d] = vc[d];
  e_acc += contact_terms(cm, vc, vhat, mug, R, gw, rgr);
  double2* out = reinterpret_cast<double2*>(a.cellsum + c * kCellSumStride);
  out[0] = make_double2(gw[0], gw[1]);
  out[1] = make_double2(gw[2], rgr[0]);
  out[2] = make_double2(rgr[1], rgr[2]);
  out[3] = make_double2(rgr[3], rgr[4]);
  out[4] = make_double2(rgr[5], 0.0);
}

// Adds one contact's record, weighted by its stencil weight w for this node,
// to a node's sums: J^T g (w R^T g) and the Hessian block (w^2 R^T G R).
__device__ __forceinline__ void add_contact_record(double w, const double2 (&q)[5], double* acc) {
  const double w2 = w * w;
  acc[0] += w * q[0].x;
  acc[1] += w * q[0].y;
  acc[2] += w * q[1].x;
  acc[3] += w2 * q[1].y;
  acc[4] += w2 * q[2].x;
  acc[5] += w2 * q[2].y;
  acc[6] += w2 * q[3].x;
  acc[7] += w2 * q[3].y;
  acc[8] += w2 * q[4].x;
}

__global__ void __launch_bounds__(kThreads, 1) k_qn_solve(SolverArgs a) {
  __shared__ double sm[32 * kMaxRed + kMaxRed];
  extern __shared__ double s_dyn[];  // [kWarps][27][32] staged stencil weights
  __shared__ double s_bc[4];
  __shared__ int s_flag;
  const int nd = *a.nd_dev;
  const int nc = *a.nc_dev;
  if (a.skip_if_no_contacts && nc == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.out->converged = 1;
      a.out->iterations = 0;
      a.out->ls_evals = 0;
      a.out->status = 0;
      a.out->n_contacts = 0;
      a.out->n_dofs = 3 * nd;
      if (a.p_out) *a.p_out = 1.0;
    }
    return;
  }
  // The whole cooperative grid participates (cg grid sync spans every CTA);
  // a problem small enough for one CTA runs on CTA 0 with __syncthreads only.
  int nctas = (int)gridDim.x;
  if (a.force_ctas == 0 && nc <= 1024 && nd <= 8192) nctas = 1;
  if (a.force_ctas == 1) nctas = 1;
  if (nctas == 1 && blockIdx.x != 0) return;
  // line-search group: ~3 contacts per thread, at least one CTA
  int G = 1;
  if (nctas > 1) {
    // kLS contacts per thread, all in registers (4: measured optimum between
    // per-evaluation compute
    // and the all-to-all reduction latency, which grows with the group)
    G = (a.force_ls_ctas > 0) ? a.force_ls_ctas : (nc + kThreads * kLS - 1) / (kThreads * kLS);
    if (G < 1) G = 1;
    if (G > nctas) G = nctas;
    if (G > 64) G = 64;  // slot_poll_sum<.., 2> polls at most 64 slots
  }
  const bool in_group = (int)blockIdx.x < G;
  const int ng = a.su.counts[0];
  const int n_cn = a.su.counts[1];
  const int n_fn = nd - n_cn;
  (void)ng;
  unsigned tagA = a.chan[0], tagB = a.chan[1], tagC = a.chan[2];
  unsigned long long in_sync_acc = 0;
  unsigned bar_gen = a.chan[3];  // generation word persists across solves
  Sync sync{a.partials, nctas,
            (a.prof && blockIdx.x == 0 && threadIdx.x == 0) ? a.prof : nullptr,
            (a.prof && threadIdx.x == 0) ? &in_sync_acc : nullptr, a.bar, &bar_gen};
  int parity = 0;
  unsigned grp_par = 0;  // group_reduce result buffer parity
  const long long nthr = (long long)nctas * kThreads;
  const ContactModel cm{a.K, a.den, a.eps_v};
  const double inv_eps = 1.0 / a.eps_v;
  const bool prof = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
  const bool cprof = a.prof && threadIdx.x == 0;  // per-CTA phase work times
  unsigned long long cta_t0 = 0, cta_acc[5] = {0, 0, 0, 0, 0};
  auto cta_start = [&]() {
    if (cprof) cta_t0 = gtime();
  };
  auto cta_stop = [&](int ph) {
    __syncthreads();
    if (cprof) cta_acc[ph] += gtime() - cta_t0;
  };
  unsigned long long pt[kSolverProf] = {0};
  unsigned long long tmark = prof ? gtime() : 0ull;
  auto lap = [&](int slot) {
    if (prof) {
      unsigned long long t = gtime();
      pt[slot] += t - tmark;
      tmark = t;
    }
  };
  double* v = a.v;
  // Work is interleaved across CTAs at warp granularity so that small node /
  // contact counts still spread over every SM: virtual thread id vt puts 32
  // consecutive items on one warp and consecutive warps on consecutive CTAs.
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long vt = ((long long)wid * nctas + blockIdx.x) * 32 + lane;
  const long long chunk0 = ((long long)wid * nctas + blockIdx.x) * kChunk;
  const long long chunk_step = (long long)nctas * kThreads;
  double* s_w_w = s_dyn + wid * (27 * kSwStride);
  // every warp owns at most one chunk: its weights stay staged for the solve
  const bool resident = (long long)nc <= (long long)nctas * kThreads;

  // ---- init: contact nodes v = v0; free-node sums; contacts
  for (long long t = vt; t < n_cn; t += nthr) {
    const long long i = a.su.cn[t];
#pragma unroll
    for (int d = 0; d < 3; ++d) v[3 * i + d] = a.v0[3 * i + d];
  }
  double S0 = 0.0, Q0 = 0.0, Q1 = 0.0;
  double e_acc = 0.0;  // this thread's contact energy at the current vc
  {
    double r3[3] = {0.0, 0.0, 0.0};
    for (long long t = vt; t < n_fn; t += nthr) {
      const long long i = a.su.fn[t];
      const double m = a.m[i];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double vs = a.v_star[3 * i + d];
        const double e0 = a.v0[3 * i + d] - vs;
        r3[0] += m * e0 * e0;
        r3[1] += m * vs * vs;
        r3[2] += m * vs * e0;
      }
    }
    for (long long c0 = chunk0; c0 < nc; c0 += chunk_step) {
      stage_weights(a, c0, nc, s_w_w);
      contact_update_chunk(a, cm, c0, nc, true, 0.0, s_w_w, e_acc);
    }
    double s3[3];
    reduce_all<3>(sync, parity, r3, s3, sm);  // also publishes vc / cellsum grid-wide
    S0 = s3[0] + a.ext_free[0];
    Q0 = s3[1] + a.ext_free[1];
    Q1 = s3[2] + a.ext_free[2];
  }
  lap(0);

  // lanes per contact node in phase N: 4 (more entries in flight per node)
  // while the contact nodes fit in one pass of the grid, else 2 (twice the
  // nodes in flight per warp; measured in round 1: 16.4 -> 10.7 us of N work per
  // iteration with 31k contact nodes, no change with 9k)
  const int NL = 4LL * n_cn > (long long)nctas * kThreads ? 2 : 4;
  int iterations = 0, ls_evals_total = 0, status = 0;
  bool converged = false;
  double alpha_prev = 0.0;  // pending v += alpha dv, applied by each node's owner in N
  double P = 1.0;           // free nodes: v - v* = P (v0 - v*)
  for (int it = 0;; ++it) {
    // ---- N: pending update, gathers, gradient, residual, Hessian, direction
    double red[8] = {0, 0, 0, 0, e_acc, 0, 0, 0};
    int reg_count = 0;
    cta_start();
    if (it > 0) P *= (1.0 - alpha_prev);
    {
      // NL lanes per contact node (32 / NL nodes per warp), warp-interleaved
      // over CTAs
      const int kNPW = 32 / NL;
      const int grp = lane / NL, gl = lane & (NL - 1);
      const long long vw = (long long)wid * nctas + blockIdx.x, nw = (long long)nctas * kWarps;
      for (long long t0 = vw * kNPW; t0 < n_cn; t0 += nw * kNPW) {
        const long long t = t0 + grp;
        const bool live = t < n_cn;
        const int4 rec = live ? a.su.cn_rec[t] : make_int4(0, 0, 0, 0);
        const long long i = rec.x;
        NodeIn nin;
        if (live && gl == 0) {
          nin.m = a.m[i];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            nin.v[d] = v[3 * i + d];
            nin.vs[d] = a.v_star[3 * i + d];
          }
          if (it > 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              nin.v[d] = nin.v[d] + alpha_prev * a.dv[3 * i + d];
              v[3 * i + d] = nin.v[d];
            }
          }
        }
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        // up to kEPL (contact, slot) entries per lane per pass: all entries,
        // then all records and weights, in flight
        for (int eb = rec.y + gl; eb < rec.z; eb += kEPL * NL) {
          int key[kEPL];
#pragma unroll
          for (int j = 0; j < kEPL; ++j)
            key[j] = (eb + NL * j < rec.z) ? __ldg(&a.su.ent[eb + NL * j]) : -1;
          double2 q[kEPL][5];
          double w[kEPL];
#pragma unroll
          for (int j = 0; j < kEPL; ++j) {
            const int kk = key[j] < 0 ? 0 : key[j];
            const long long c = kk >> 5;
            w[j] = __ldg(&a.cw[(long long)(kk & 31) * a.nc_cap + c]);
            const double2* src = reinterpret_cast<const double2*>(a.cellsum + c * kCellSumStride);
#pragma unroll
            for (int r = 0; r < 5; ++r) q[j][r] = src[r];
          }
#pragma unroll
          for (int j = 0; j < kEPL; ++j)
            if (key[j] >= 0) add_contact_record(w[j], q[j], acc);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
          for (int o = NL / 2; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (live && gl == 0) node_finish(a, i, nin, acc, acc + 3, red, reg_count);
      }
    }
    lap(6);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      // free nodes in closed form: g = m P e0, dv = -P e0
      const double p2s = P * P * S0;
      red[0] += p2s;
      red[1] += Q0 + 2.0 * P * Q1 + p2s;
      red[3] += p2s;
      red[5] -= p2s;
      red[6] += p2s;
    }
    if (reg_count) atomicAdd(&a.out->regularized, reg_count);
    cta_stop(0);
    cta_start();
    double s[8];
    reduce_all<8>(sync, parity, red, s, sm);
    cta_stop(3);
    lap(1);
    const double residual = sqrt(s[0]);
    const double threshold = a.eps_a + a.eps_r * fmax(sqrt(s[1]), sqrt(s[2]));
    if (blockIdx.x == 0 && threadIdx.x == 0 && it <= a.max_iters) {
      if (a.tr_obj) a.tr_obj[it] = 0.5 * s[3] + s[4];
      if (a.tr_res) a.tr_res[it] = residual;
      if (a.tr_thr) a.tr_thr[it] = threshold;
    }
    // test-last loop; iteration 0 tests eps_a only (solver.py:339-345)
    if (it >= a.max_iters) {
      converged = residual < threshold;
      break;
    }
    if (residual < (it > 0 ? threshold : a.eps_a)) {
      converged = true;
      break;
    }
    if (s[7] > 0.0) {
      status = MPMRB_E_NONFINITE;  // Hessian block not SPD after regularization
      break;
    }
    const double a1 = s[5], a2 = s[6];

    // ---- D: dvc = R J dv, the phi'(0) contact term (solver.py:305-310, 269)
    // and the first line-search evaluation, which is always at alpha = 1
    // (solver.py:276): its contact sums travel with phi'(0) to the group
    double r0 = 0.0, r1 = 0.0, r1dd = 0.0;
    cta_start();
    for (long long c0 = chunk0; c0 < nc; c0 += chunk_step) {
      const long long c = c0 + lane;
      if (c < nc) {
        double R[9], dvc[3], vc[3];
        load_frame(a.frames, c, R);
        if (resident) gather_contact_sw(a, c, a.dv, R, s_w_w, lane, dvc);
        else gather_contact(a, c, a.dv, R, dvc);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          a.dvc[3 * c + d] = dvc[d];
          vc[d] = a.vc[3 * c + d];
        }
        double dd2 = 0.0;
        const double vh = a.cvhat[c], mg = a.cmug[c];
        ls_terms(cm, inv_eps, vc, dvc, vh, mg, 0.0, r0, dd2);
        ls_terms(cm, inv_eps, vc, dvc, vh, mg, 1.0, r1, r1dd);
      }
    }
    __syncwarp();
    lap(7);
    cta_stop(1);
    // hand the contact data and the phi'(0) / alpha = 1 partials to the group
    double d0s = 0.0, e1s = 0.0, e1dd = 0.0;
    if (nctas == 1) {
      double rr[3] = {r0, r1, r1dd}, ss[3];
      group_reduce<3>(1, a.slots, tagB, rr, ss, sm, grp_par);
      d0s = ss[0];
      e1s = ss[1];
      e1dd = ss[2];
    } else {
      double rr[3] = {r0, r1, r1dd}, bs[3];
      block_reduce<3>(rr, sm, bs);
      unsigned long long* base = a.slots + kSlotA + (long long)(tagA & 1u) * kMaxSolverCtas * 6;
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();  // release this CTA's dvc writes (bar.sync made them CTA-visible)
        slot_publish<3>(base + 6LL * blockIdx.x, bs, tagA);
      }
      if (in_group && threadIdx.x < 32) {
        double r[3];
        slot_poll_sum<3, (kMaxSolverCtas + 31) / 32>(base, nctas, tagA, r);
        fence_acq_rel_gpu();  // acquire: the producers' dvc writes are visible below
        if (threadIdx.x == 0) {
          s_bc[0] = r[0];
          s_bc[1] = r[1];
          s_bc[2] = r[2];
        }
      }
      ++tagA;
      __syncthreads();
      d0s = s_bc[0];
      e1s = s_bc[1];
      e1dd = s_bc[2];
      __syncthreads();
    }
    lap(2);
    double alpha_final = 0.0;
    if (in_group) {
      const double d0 = a1 + d0s;
      if (!isfinite(d0) || d0 >= 0.0) {
        status = MPMRB_E_NOT_DESCENT;
      } else {
        // ---- LS: exact line search (solver.py:266-298) over the group
        const long long gtid = (long long)blockIdx.x * kThreads + threadIdx.x;
        const long long gthr = (long long)G * kThreads;
        const double eps2 = cm.eps_v * cm.eps_v;
        LsRec lv[kLS];
#pragma unroll
        for (int j = 0; j < kLS; ++j) {
          const long long c = gtid + j * gthr;
          double vc[3] = {0.0, 0.0, 0.0}, dvc[3] = {0.0, 0.0, 0.0}, vh = 0.0, mg = 0.0;
          if (c < nc) {  // absent contacts keep dvc = 0, mug = 0 and add exactly 0
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              vc[d] = __ldcg(&a.vc[3 * c + d]);
              dvc[d] = __ldcg(&a.dvc[3 * c + d]);
            }
            vh = __ldcg(&a.cvhat[c]);
            mg = __ldcg(&a.cmug[c]);
          }
          lv[j] = ls_rec(cm, vc, dvc, vh, mg);
        }
        double lo = 0.0, hi = INFINITY, alpha = 1.0;
        alpha_final = -1.0;
        int evals = 0;
        for (int ev = 1; ev <= a.ls_max; ++ev) {
          unsigned long long tls0 = prof ? gtime() : 0ull;
          double ss[2];
          if (ev == 1) {  // alpha = 1: summed in phase D
            ss[0] = e1s;
            ss[1] = e1dd;
          } else {
            double rr[2] = {0.0, 0.0};
#pragma unroll
            for (int j = 0; j < kLS; ++j) ls_terms_rec(cm, eps2, inv_eps, lv[j], alpha, rr[0], rr[1]);
            for (long long c = gtid + kLS * gthr; c < nc; c += gthr) {
              double vc[3], dvc[3];
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                vc[d] = __ldcg(&a.vc[3 * c + d]);
                dvc[d] = __ldcg(&a.dvc[3 * c + d]);
              }
              ls_terms(cm, inv_eps, vc, dvc, __ldcg(&a.cvhat[c]), __ldcg(&a.cmug[c]), alpha, rr[0],
                       rr[1]);
            }
            unsigned long long tls1 = prof ? gtime() : 0ull;
            group_reduce<2>(G, a.slots, tagB, rr, ss, sm, grp_par);
            if (prof) {
              unsigned long long tls2 = gtime();
              pt[12] += tls1 - tls0;
              pt[13] += tls2 - tls1;
            }
          }
          evals = ev;
          const double d = a1 + a2 * alpha + ss[0];
          const double dd = a2 + ss[1];
          if (fabs(d) <= a.ls_tol * fabs(d0)) {
            alpha_final = alpha;
            break;
          }
          if (d > 0.0) hi = alpha;
          else lo = alpha;
          double cand = (isfinite(dd) && dd > 0.0) ? alpha - d / dd : NAN;
          if (isfinite(hi)) {
            if (!(lo < cand && cand < hi) || !isfinite(cand)) cand = 0.5 * (lo + hi);
          } else {
            if (!isfinite(cand) || cand <= lo) cand = 2.0 * fmax(alpha, 1e-8);
          }
          alpha = cand;
        }
        if (alpha_final < 0.0) alpha_final = (lo > 0.0) ? lo : alpha;  // solver.py:296-298
        ls_evals_total += evals;
      }
      if (nctas > 1 && blockIdx.x == 0 && threadIdx.x == 0) {
        const double pub[2] = {alpha_final, (double)status};
        slot_publish<2>(a.slots + kSlotC + (long long)(tagC & 1u) * 4, pub, tagC);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0 && a.tr_alpha && status == 0)
        a.tr_alpha[it] = alpha_final;
    } else if (threadIdx.x < 32) {
      double r[2];
      slot_poll_sum<2, 1, 128>(a.slots + kSlotC + (long long)(tagC & 1u) * 4, 1, tagC, r);
      if (threadIdx.x == 0) {
        s_bc[0] = r[0];
        s_bc[1] = r[1];
      }
    }
    if (nctas > 1) {
      ++tagC;
      __syncthreads();
      if (!in_group) {
        alpha_final = s_bc[0];
        status = (int)s_bc[1];
      }
      __syncthreads();
    }
    lap(3);
    if (status) break;
    // ---- U: vc += alpha dvc, contact terms -> cellsum for the next N
    e_acc = 0.0;
    cta_start();
    for (long long c0 = chunk0; c0 < nc; c0 += chunk_step)
      contact_update_chunk(a, cm, c0, nc, false, alpha_final, s_w_w, e_acc);
    lap(8);
    cta_stop(2);
    sync();  // cellsum and vc visible grid-wide
    lap(4);
    alpha_prev = alpha_final;
    ++iterations;
  }
  // The last N applied every pending update, so contact-node v is final here.
  // ---- epilogue: free nodes in closed form, scatter, impulses (solver.py:363-365)
  bool finite_v = true;
  for (long long t = vt; t < n_cn; t += nthr) {
    const long long i = a.su.cn[t];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double vi = v[3 * i + d];
      finite_v &= isfinite(vi);
      if (a.v_next_full) a.v_next_full[3 * (long long)a.act[i] + d] = vi;
    }
  }
  for (long long t = vt; t < n_fn; t += nthr) {
    const long long i = a.su.fn[t];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double vs = a.v_star[3 * i + d];
      const double vi = vs + P * (a.v0[3 * i + d] - vs);
      v[3 * i + d] = vi;
      finite_v &= isfinite(vi);
      if (a.v_next_full) a.v_next_full[3 * (long long)a.act[i] + d] = vi;
    }
  }
  for (long long c0 = chunk0; c0 < nc; c0 += chunk_step) {
    const long long c = c0 + lane;
    if (c < nc) {
      double vc[3], g[3], Gd[4];
#pragma unroll
      for (int d = 0; d < 3; ++d) vc[d] = a.vc[3 * c + d];
      cm_eval(cm, vc, a.cvhat[c], a.cmug[c], g, Gd);
#pragma unroll
      for (int d = 0; d < 3; ++d) a.gamma[3 * c + d] = -g[d];
    }
  }
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  if (!finite_v) s_flag = 1;
  __syncthreads();
  if (s_flag && threadIdx.x == 0) atomicOr(&a.out->status_flags, 1);
  if (cprof)
    for (int ph = 0; ph < 4; ++ph) a.prof[kSolverProf + ph * 160 + blockIdx.x] += cta_acc[ph];
  if (cprof) a.prof[kSolverProf + 4 * 160 + blockIdx.x] += in_sync_acc;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out->converged = converged ? 1 : 0;
    a.out->iterations = iterations;
    a.out->ls_evals = ls_evals_total;
    a.out->status = status;
    a.out->n_contacts = nc;
    a.out->n_dofs = 3 * nd;
    if (a.p_out) *a.p_out = P;
    a.chan[0] = tagA;
    a.chan[1] = tagB;
    a.chan[2] = tagC;
    if (nctas > 1) a.chan[3] = bar_gen;
    if (prof) {
      lap(5);
      for (int k = 0; k < 6; ++k) a.prof[k] += pt[k];
      a.prof[14] += pt[6] + ((unsigned long long)pt[7] << 32);
      a.prof[15] += pt[8];
      a.prof[6] += (unsigned long long)iterations;
      a.prof[7] += (unsigned long long)ls_evals_total;
      a.prof[8] += (unsigned long long)nctas + ((unsigned long long)G << 32);
      a.prof[9] += 1ull;
      a.prof[11] += (unsigned long long)n_cn + ((unsigned long long)ng << 32);
      a.prof[12] += pt[12];
      a.prof[13] += pt[13];
    }
  }
}

// ---------------------------------------------------------------- setup

constexpr int kSetupThreads = 256;

__device__ __forceinline__ bool same_stencil(const int* __restrict__ cnodes, long long nc_cap,
                                             long long c, long long d) {
  bool same = true;
#pragma unroll 9
  for (int k = 0; k < 27; ++k)
    same &= __ldg(&cnodes[(long long)k * nc_cap + c]) == __ldg(&cnodes[(long long)k * nc_cap + d]);
  return same;
}

__global__ void k_su_heads(const int* __restrict__ nc_dev, long long nc_cap,
                           const int* __restrict__ cnodes, int* __restrict__ head) {
  const long long nc = *nc_dev;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc;
       c += (long long)gridDim.x * blockDim.x)
    head[c] = (c == 0 || !same_stencil(cnodes, nc_cap, c, c - 1)) ? 1 : 0;
}

__global__ void k_su_groups(const int* __restrict__ nc_dev, const int* __restrict__ head,
                            const int* __restrict__ head_off, const int* __restrict__ counts,
                            int* __restrict__ grp_of, int* __restrict__ grp_start) {
  const long long nc = *nc_dev;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc;
       c += (long long)gridDim.x * blockDim.x) {
    const int h = head[c], o = head_off[c];
    grp_of[c] = o + h - 1;
    if (h) grp_start[o] = (int)c;
    if (c == 0) grp_start[counts[0]] = (int)nc;
  }
}

// Per node: (run, slot) entries and the contacts they expand to.
__global__ void k_su_count(const int* __restrict__ counts, long long nc_cap,
                           const int* __restrict__ cnodes, const int* __restrict__ grp_start,
                           int* __restrict__ cnt, int* __restrict__ cnt_exp) {
  const long long np = (long long)counts[0] * 27;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np;
       p += (long long)gridDim.x * blockDim.x) {
    const long long g = p / 27, k = p - g * 27;
    const int c0 = grp_start[g];
    const int node = cnodes[k * nc_cap + c0];
    if (node >= 0) {
      atomicAdd(&cnt[node], 1);
      atomicAdd(&cnt_exp[node], grp_start[g + 1] - c0);
    }
  }
}

__global__ void k_su_fill(const int* __restrict__ counts, long long nc_cap,
                          const int* __restrict__ cnodes, const int* __restrict__ grp_start,
                          const int* __restrict__ off, int* __restrict__ fill,
                          int* __restrict__ ent_tmp) {
  const long long np = (long long)counts[0] * 27;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np;
       p += (long long)gridDim.x * blockDim.x) {
    const long long g = p / 27, k = p - g * 27;
    const int node = cnodes[k * nc_cap + grp_start[g]];
    if (node < 0) continue;
    const int pos = off[node] + atomicAdd(&fill[node], 1);
    ent_tmp[pos] = (int)(((long long)grp_start[g] << 5) | k);
  }
}

// Expand every (run, slot) entry into its contacts at their sorted position
// in the node's segment: the position is the number of contacts of the
// node's runs with a smaller key (keys are unique, runs are disjoint), so
// each node lists (contact << 5 | slot) in ascending contact order.
__global__ void k_su_rank(const int* __restrict__ nd_dev, long long nc_cap,
                          const int* __restrict__ cnodes, const int* __restrict__ grp_of,
                          const int* __restrict__ grp_start, const int* __restrict__ off,
                          const int* __restrict__ off_exp, const int* __restrict__ ent_tmp,
                          int* __restrict__ ent) {
  const long long total = off[*nd_dev];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int key = ent_tmp[e];
    const int c0 = key >> 5, k = key & 31;
    const int node = cnodes[(long long)k * nc_cap + c0];
    const int b = off[node], en = off[node + 1];
    int before = 0;
    for (int p = b; p < en; ++p) {
      const int o = __ldg(&ent_tmp[p]);
      if (o < key) {
        const int oc = o >> 5;
        before += __ldg(&grp_start[__ldg(&grp_of[oc]) + 1]) - oc;
      }
    }
    const int len = grp_start[grp_of[c0] + 1] - c0;
    int* dst = ent + off_exp[node] + before;
    for (int t = 0; t < len; ++t) dst[t] = ((c0 + t) << 5) | k;
  }
}

__global__ void k_su_flag(const int* __restrict__ nd_dev, const int* __restrict__ cnt,
                          int* __restrict__ flag) {
  const long long nd = *nd_dev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nd;
       i += (long long)gridDim.x * blockDim.x)
    flag[i] = cnt[i] > 0 ? 1 : 0;
}

__global__ void k_su_lists(const int* __restrict__ nd_dev, const int* __restrict__ flag,
                           const int* __restrict__ flag_off, const int* __restrict__ off_exp,
                           int* __restrict__ cn, int4* __restrict__ cn_rec,
                           int* __restrict__ fn) {
  const long long nd = *nd_dev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nd;
       i += (long long)gridDim.x * blockDim.x) {
    const int o = flag_off[i];
    if (flag[i]) {
      cn[o] = (int)i;
      cn_rec[o] = make_int4((int)i, off_exp[i], off_exp[i + 1], 0);
    } else {
      fn[i - o] = (int)i;
    }
  }
}

// solver.py:224-256 solve_search_direction: d = -H^-1 g per 3x3 SPD block,
// Cholesky in registers; a block that fails is regularised by +1e-12
// max(tr H, 1) 10^attempt on the diagonal (cumulative, <= 3 times) exactly as
// the reference's batch loop does for its bad blocks.  reg[0] counts the
// regularised blocks (the reference's warning), reg[1] the blocks still not SPD
// after the last attempt (its FloatingPointError).
__global__ void k_search_direction(const double* __restrict__ hb, const double* __restrict__ g,
                                   long long n, double* __restrict__ d, int* __restrict__ reg) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double* H = hb + 9 * i;
    double h[6] = {H[0], H[4], H[8], H[3], H[6], H[7]};  // 00 11 22 10 20 21 (lower)
    double l11 = 0, l21 = 0, l31 = 0, l22 = 0, l32 = 0, l33 = 0;
    bool good = false;
    for (int attempt = 0; attempt < 4; ++attempt) {
      l11 = sqrt(h[0]);
      l21 = h[3] / l11;
      l31 = h[4] / l11;
      l22 = sqrt(h[1] - l21 * l21);
      l32 = (h[5] - l31 * l21) / l22;
      l33 = sqrt(h[2] - l31 * l31 - l32 * l32);
      good = isfinite(l11) && isfinite(l22) && isfinite(l33) && l11 > 0.0 && l22 > 0.0 &&
             l33 > 0.0;
      if (good || attempt == 3) break;
      if (attempt == 0) atomicAdd(&reg[0], 1);
      const double tr = h[0] + h[1] + h[2];
      const double bump = 1e-12 * fmax(tr, 1.0) * (attempt == 0 ? 1.0 : (attempt == 1 ? 10.0 : 100.0));
      h[0] += bump;
      h[1] += bump;
      h[2] += bump;
    }
    if (!good) atomicAdd(&reg[1], 1);
    const double* gi = g + 3 * i;
    const double y1 = -gi[0] / l11;
    const double y2 = (-gi[1] - l21 * y1) / l22;
    const double y3 = (-gi[2] - l31 * y1 - l32 * y2) / l33;
    const double x3 = y3 / l33;
    const double x2 = (y2 - l32 * x3) / l22;
    const double x1 = (y1 - l21 * x2 - l31 * x3) / l11;
    d[3 * i] = x1;
    d[3 * i + 1] = x2;
    d[3 * i + 2] = x3;
  }
}

unsigned su_grid(long long cap) {
  long long b = (cap + kSetupThreads - 1) / kSetupThreads;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (unsigned)b;
}

}  // namespace

int launch_solver_setup(Ctx& c, const int* nd_dev, const int* nc_dev, long long nd_cap,
                        long long nc_cap, const int* cnodes, const SolverSetup& su,
                        DevBuf& tiles) {
  // adjacency entries pack (contact << 5 | slot) into an int32
  if (nc_cap >= (1LL << 26))
    return set_error(MPMRB_E_INVALID, "contact capacity %lld exceeds 2^26", nc_cap);
  MPMRB_CUDA_OK(cudaMemsetAsync(su.cnt, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(su.cnt_exp, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(su.fill, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(su.flag, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(su.counts, 0, sizeof(int) * 2, c.stream));
  const long long ncc = nc_cap > 0 ? nc_cap : 1;
  k_su_heads<<<su_grid(ncc), kSetupThreads, 0, c.stream>>>(nc_dev, nc_cap, cnodes, su.head);
  int rc = scan_exclusive_i32(c, su.head, su.head_off, ncc, nc_dev, su.counts + 0, tiles);
  if (rc) return rc;
  k_su_groups<<<su_grid(ncc), kSetupThreads, 0, c.stream>>>(nc_dev, su.head, su.head_off,
                                                            su.counts, su.grp_of, su.grp_start);
  k_su_count<<<su_grid(27 * ncc), kSetupThreads, 0, c.stream>>>(su.counts, nc_cap, cnodes,
                                                                 su.grp_start, su.cnt, su.cnt_exp);
  c.launches += 3;
  // exclusive scan over nd_cap+1 entries (cnt is zero past nd: off[nd] = total)
  rc = scan_exclusive_i32(c, su.cnt, su.off, nd_cap + 1, nullptr, nullptr, tiles);
  if (rc) return rc;
  rc = scan_exclusive_i32(c, su.cnt_exp, su.off_exp, nd_cap + 1, nullptr, nullptr, tiles);
  if (rc) return rc;
  k_su_fill<<<su_grid(27 * ncc), kSetupThreads, 0, c.stream>>>(su.counts, nc_cap, cnodes,
                                                                su.grp_start, su.off, su.fill,
                                                                su.ent_tmp);
  k_su_rank<<<su_grid(27 * ncc), kSetupThreads, 0, c.stream>>>(nd_dev, nc_cap, cnodes,
                                                                su.grp_of, su.grp_start, su.off,
                                                                su.off_exp, su.ent_tmp, su.ent);
  k_su_flag<<<su_grid(nd_cap + 1), kSetupThreads, 0, c.stream>>>(nd_dev, su.cnt, su.flag);
  c.launches += 3;
  rc = scan_exclusive_i32(c, su.flag, su.flag_off, nd_cap + 1, nullptr, su.counts + 1, tiles);
  if (rc) return rc;
  k_su_lists<<<su_grid(nd_cap + 1), kSetupThreads, 0, c.stream>>>(
      nd_dev, su.flag, su.flag_off, su.off_exp, su.cn, su.cn_rec, su.fn);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_search_direction(Ctx& c, const double* h, const double* g, long long n, double* d,
                            int* reg) {
  MPMRB_CUDA_OK(cudaMemsetAsync(reg, 0, 2 * sizeof(int), c.stream));
  if (n == 0) return MPMRB_OK;
  k_search_direction<<<su_grid(n), kSetupThreads, 0, c.stream>>>(h, g, n, d, reg);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas) {
  // Grid: one 256-thread CTA per SM (255 registers), cooperative so that all
  // CTAs are co-resident for the in-kernel barriers.  Measured and rejected:
  // clusters with DSMEM line-search reductions (1.2 vs 0.9 us per reduction
  // on 12-16 CTAs, tools/reduce_bench.cu).
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    MPMRB_CUDA_OK(cudaGetDevice(&dev));
    MPMRB_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (sms > kMaxSolverCtas) sms = kMaxSolverCtas;
  }
  int g = sms;
  if (grid_ctas > 0 && grid_ctas < g) g = grid_ctas;
  if (a.force_ctas > 1) g = a.force_ctas < sms ? a.force_ctas : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(kThreads);
  static bool smem_set = false;
  const int dyn = (int)(sizeof(double) * kWarps * 27 * kSwStride);
  if (!smem_set) {
    MPMRB_CUDA_OK(cudaFuncSetAttribute(k_qn_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    smem_set = true;
  }
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MPMRB_CUDA_OK(cudaLaunchKernelEx(&cfg, k_qn_solve, a));
  c.launches++;
  return MPMRB_OK;
}

}  // namespace mpmrb
