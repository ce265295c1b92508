// Globally convergent quasi-Newton convex contact solve on sm_100a
// (solver.py:197-382), run entirely on the device as ONE persistent
// cooperative kernel: no host round trip per iteration or per line-search
// evaluation.
//
// Layout.  The problem is restricted to active nodes (solver.py:197-221).
// Per-contact stencils are slot-major [27][nc_cap].  A node->(contact, slot)
// CSR adjacency (built once per solve, entries sorted) turns the J^T scatters
// of the gradient and of the block-diagonal Hessian (solver.py:127-167) into
// per-node gathers: no atomics and a fixed summation order, so a solve is
// bitwise reproducible run to run.  Nodes with adjacency ("contact nodes",
// typically a thin layer) are gathered by one warp each from a compacted
// list; all other nodes take the cheap thread-per-node path.
//
// Phases per iteration (solver.py:338-357), each a grid-stride loop:
//   N  nodes:    jt = J^T g_c, H_ii = m I + sum w^2 R^T G R (gathers), g,
//                residual / norms / mass energy, 3x3 Cholesky -> dv, and the
//                line-search coefficients a1, a2                    [reduce]
//   D  contacts: dvc = R J dv, phi'(0) contact term                   [reduce]
//   LS contacts: <= ls_max evaluations of phi'(a), phi''(a), contact
//                data held in registers                        [reduce each]
//   U  nodes v += a dv; contacts vc += a dvc, then g_c -> R^T g_c, G ->
//      R^T G R and the contact energy for the next N               [grid sync]
// Grid synchronisation is cooperative_groups::this_grid().sync() (measured
// ~2 us per reduction on B200, flat in CTA count; tools/barrier_bench.cu).
// Every CTA sums the per-CTA partials in the same fixed order, so all CTAs
// take identical convergence and line-search decisions.
//
// vc is advanced as vc + a dvc (= R J (v + a dv) + b exactly in real
// arithmetic) instead of being re-gathered from v; the difference is roundoff.
#include <cooperative_groups.h>

#include "common.cuh"
#include "contact.cuh"
#include "internal.h"
#include "solver.cuh"

namespace cg = cooperative_groups;

namespace mpmrb {

namespace {

constexpr int kThreads = kSolverThreads;
constexpr int kMaxRed = 8;  // reduction lanes per call
constexpr int kJR = 2;      // contacts per thread cached in registers

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Sync {
  double* partials;  // [2][kMaxRed][kMaxSolverCtas]
  int nctas;
  unsigned long long* prof;  // CTA 0 / thread 0 only: [10] time inside grid syncs
  __device__ __forceinline__ void operator()() const {
    if (nctas == 1) {
      __syncthreads();
      return;
    }
    unsigned long long t0 = prof ? gtime() : 0ull;
    cg::this_grid().sync();
    if (prof) atomicAdd(prof + 10, gtime() - t0);
  }
};

// Sum K values over all threads of all participating CTAs; every thread
// receives the totals.  Partials are double-buffered: a CTA racing into the
// next reduction writes the other half while slower CTAs still read this one,
// and the grid sync inside the next reduction closes the window.
template <int K>
__device__ void reduce_all(const Sync& sync, int& parity, double (&v)[K], double (&out)[K],
                           double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* part = sync.partials + parity * (kMaxRed * kMaxSolverCtas);
  parity ^= 1;
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
      if (lane == 0) {
        if (sync.nctas == 1) sm[32 * kMaxRed + k] = x;
        else part[k * kMaxSolverCtas + blockIdx.x] = x;
      }
    }
  }
  if (sync.nctas > 1) {
    sync();
    if (wid == 0) {
      // all K x ceil(nctas/32) loads issued before the first add: one L2
      // round trip instead of one per 32 CTAs per value
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

__device__ __forceinline__ void load_frame(const double* fr, long long c, double* R) {
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(fr + 9 * c + k);
}

// R (sum_k w_k u[node_k])
__device__ __forceinline__ void gather_contact(const SolverArgs& a, long long c,
                                               const double* __restrict__ u, const double* R,
                                               double* out) {
  double up[3] = {0.0, 0.0, 0.0};
#pragma unroll 9
  for (int k = 0; k < 27; ++k) {
    int nd = __ldg(&a.cnodes[(long long)k * a.nc_cap + c]);
    double w = __ldg(&a.cw[(long long)k * a.nc_cap + c]);
#pragma unroll
    for (int d = 0; d < 3; ++d) up[d] += w * (*(&u[3 * nd + d]));
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) out[r] = R[3 * r] * up[0] + R[3 * r + 1] * up[1] + R[3 * r + 2] * up[2];
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
  // GR = G @ R with G = [[G0,G3,0],[G3,G1,0],[0,0,G2]]
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

// Per-node part of phase N given the gathered jt (3) and Hessian sums hs (6):
// gradient, residual/norm/energy partials, regularised 3x3 Cholesky
// (solver.py:224-256), direction dv and the line-search coefficients.
struct NodeIn {
  double m, v[3], vs[3];
};

__device__ __forceinline__ NodeIn load_node(const SolverArgs& a, long long i) {
  NodeIn n;
  n.m = a.m[i];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    n.v[d] = (*(&a.v[3 * i + d]));
    n.vs[d] = a.v_star[3 * i + d];
  }
  return n;
}

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

// Contact group: the CTAs that own the contacts.  With a cluster launch it is
// cluster 0 (DSMEM reductions + hardware cluster barrier, ~0.7 us); without
// clusters it is the whole grid (grid reductions, ~1.7 us).
struct Group {
  bool member;     // this CTA owns contacts
  int rank;        // rank within the group
  int size;        // CTAs in the group
  bool cluster;    // reductions go through the cluster
};

// Sum K values over the contact group (members only).  Cluster path: each CTA
// publishes its block sum in its own shared slot, cluster barrier, then every
// CTA reads the size partials over DSMEM in rank order.  Slots are
// double-buffered by parity (same argument as reduce_all).
template <int K>
__device__ void group_reduce(const Group& gr, const Sync& sync, int& parity, int& cparity,
                             double (&v)[K], double (&out)[K], double* sm,
                             double (*cslot)[kMaxRed]) {
  if (!gr.cluster) {
    reduce_all<K>(sync, parity, v, out, sm);
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sm[k * 32 + wid] = x;
  }
  __syncthreads();
  const int par = cparity;
  cparity ^= 1;
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = (lane < kThreads / 32) ? sm[k * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) cslot[par][k] = x;
    }
  }
  cg::this_cluster().sync();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = 0.0;
      if (lane < gr.size) x = *cg::this_cluster().map_shared_rank(&cslot[par][k], lane);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) sm[32 * kMaxRed + k] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = sm[32 * kMaxRed + k];
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) k_qn_solve(SolverArgs a) {
  __shared__ double sm[32 * kMaxRed + kMaxRed];
  __shared__ double cslot[2][kMaxRed];
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
    }
    return;
  }
  // The whole cooperative grid participates (cg grid sync spans every CTA);
  // a problem small enough for one CTA runs on CTA 0 with __syncthreads only.
  int nctas = (int)gridDim.x;
  if (a.force_ctas == 0 && nc <= 1024 && nd <= 8192) nctas = 1;
  if (a.force_ctas == 1) nctas = 1;
  if (nctas == 1 && blockIdx.x != 0) return;
  Sync sync{a.partials, nctas,
            (a.prof && blockIdx.x == 0 && threadIdx.x == 0) ? a.prof : nullptr};
  const int csize = (nctas > 1) ? (int)cg::this_cluster().num_blocks() : 1;
  Group gr;
  if (nctas == 1) {
    gr = Group{true, 0, 1, false};
  } else if (csize > 1) {
    gr = Group{(int)blockIdx.x < csize, (int)blockIdx.x, csize, true};
  } else {
    gr = Group{true, (int)blockIdx.x, nctas, false};
  }
  int parity = 0, cparity = 0;
  const long long tid = (long long)blockIdx.x * kThreads + threadIdx.x;
  const long long nthr = (long long)nctas * kThreads;
  const int lane = threadIdx.x & 31;
  const long long gwarp = tid >> 5, nwarps = nthr >> 5;
  const ContactModel cm{a.K, a.den, a.eps_v};
  const bool prof = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
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
  const int n_cn = *a.adj.n_cn;
  const int n_hn = *a.adj.n_hn;
  const int n_fn = nd - n_cn - n_hn;

  // Contacts are owned by the contact group, interleaved at warp granularity
  // across its CTAs (each warp's 32 contacts consecutive -> coalesced
  // slot-major loads).  A thread's first kJR contacts live in registers
  // (fully unrolled j, never spilled); further ones go through memory.
  const long long cthr = (long long)gr.size * kThreads;
  const long long ctid =
      ((long long)(threadIdx.x >> 5) * gr.size + gr.rank) * 32 + (threadIdx.x & 31);
#define FOR_OWNED_CONTACTS(...)                                         \
  if (gr.member) {                                                      \
    _Pragma("unroll") for (int j = 0; j < kJR; ++j) {                  \
      const long long c = ctid + (long long)j * cthr;                  \
      constexpr bool inreg = true;                                      \
      if (c < nc) { __VA_ARGS__ }                                       \
    }                                                                   \
    for (long long c = ctid + (long long)kJR * cthr; c < nc; c += cthr) { \
      constexpr int j = 0;                                              \
      constexpr bool inreg = false;                                     \
      __VA_ARGS__                                                       \
    }                                                                   \
  }

  // ---- init: v = v0; per contact vc = R J v0 + b, the per-solve constants
  // vhat = -phi/(dt+tau_d) and mu*gamma_lag, and the contact terms
  for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
    for (int d = 0; d < 3; ++d) v[3 * i + d] = a.v0[3 * i + d];
  }
  double vcr[kJR][3], dvcr[kJR][3];
  double e_acc = 0.0;
  FOR_OWNED_CONTACTS({
    double R[9], vc[3], gw[3], rgr[6];
    load_frame(a.frames, c, R);
    gather_contact(a, c, a.v0, R, vc);
#pragma unroll
    for (int d = 0; d < 3; ++d) vc[d] += a.bias[3 * c + d];
    const double vhat = -a.phi[c] / cm.den;
    const double mug = a.mu[c] * a.gamma_lag[c];
    a.cvhat[c] = vhat;
    a.cmug[c] = mug;
    e_acc += contact_terms(cm, vc, vhat, mug, R, gw, rgr);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      a.vc[3 * c + d] = vc[d];
      a.gw[3 * c + d] = gw[d];
      if (inreg) vcr[j][d] = vc[d];
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) a.rgr[6 * c + e] = rgr[e];
  })
  sync();
  lap(0);

  int iterations = 0, ls_evals_total = 0, status = 0;
  bool converged = false;
  double alpha_prev = 0.0;  // pending v += alpha dv, applied by each node's owner in N
  for (int it = 0;; ++it) {
    // ---- N: pending update, node gathers, gradient, residual, Hessian, direction
    double red[8] = {0, 0, 0, 0, e_acc, 0, 0, 0};
    int reg_count = 0;
    auto take_node = [&](long long i) -> NodeIn {
      NodeIn nin = load_node(a, i);
      if (it > 0) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          nin.v[d] = nin.v[d] + alpha_prev * a.dv[3 * i + d];
          v[3 * i + d] = nin.v[d];
        }
      }
      return nin;
    };
    // (a1) heavy contact nodes (> kHeavyNode entries): one warp each
    for (long long t = gwarp; t < n_hn; t += nwarps) {
      const long long i = a.adj.hn[t];
      const int e0 = a.adj.hn_e[2 * t], e1 = a.adj.hn_e[2 * t + 1];
      NodeIn nin{};
      if (lane == 0) nin = take_node(i);
      double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
      for (int e = e0 + lane; e < e1; e += 32) {
        const long long c = __ldg(&a.adj.ent[e]) >> 5;
        const double w = __ldg(&a.adj.w[e]);
        const double w2 = w * w;
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[d] += w * a.gw[3 * c + d];
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[3 + q] += w2 * a.rgr[6 * c + q];
      }
#pragma unroll
      for (int q = 0; q < 9; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
      if (lane == 0) node_finish(a, i, nin, acc, acc + 3, red, reg_count);
    }
    // (a2) light contact nodes: 8-lane groups, four nodes in flight per warp
    {
      const int grp = lane >> 3, gl = lane & 7;
      for (long long t0 = gwarp * 4; t0 < n_cn; t0 += nwarps * 4) {
        const long long t = t0 + grp;
        const bool live = t < n_cn;
        const long long i = live ? a.adj.cn[t] : 0;
        const int e0 = live ? a.adj.cn_e[2 * t] : 0, e1 = live ? a.adj.cn_e[2 * t + 1] : 0;
        NodeIn nin{};
        if (live && gl == 0) nin = take_node(i);
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
        for (int e = e0 + gl; e < e1; e += 8) {
          const long long c = __ldg(&a.adj.ent[e]) >> 5;
          const double w = __ldg(&a.adj.w[e]);
          const double w2 = w * w;
#pragma unroll
          for (int d = 0; d < 3; ++d) acc[d] += w * a.gw[3 * c + d];
#pragma unroll
          for (int q = 0; q < 6; ++q) acc[3 + q] += w2 * a.rgr[6 * c + q];
        }
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (live && gl == 0) node_finish(a, i, nin, acc, acc + 3, red, reg_count);
      }
    }
    if (prof) {
      unsigned long long t = gtime();
      pt[12] += t - tmark;
      tmark = t;
    }
    // (b) nodes without contacts: thread per node
    {
      const double zero[6] = {0, 0, 0, 0, 0, 0};
      for (long long t = tid; t < n_fn; t += nthr) {
        const long long i = a.adj.fn[t];
        node_finish(a, i, take_node(i), zero, zero, red, reg_count);
      }
    }
    if (reg_count) atomicAdd(&a.out->regularized, reg_count);
    if (prof) {
      unsigned long long t = gtime();
      pt[13] += t - tmark;
      tmark = t;
    }
    double s[8];
    reduce_all<8>(sync, parity, red, s, sm);
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
    double alpha_final = 0.0;
    if (gr.member) {
      // ---- D: dvc = R J dv and the phi'(0) contact term (solver.py:305-310, 269)
      double r0[1] = {0.0};
      FOR_OWNED_CONTACTS({
        double R[9], dvc[3], vc[3], g[3];
        load_frame(a.frames, c, R);
        gather_contact(a, c, a.dv, R, dvc);
#pragma unroll
        for (int d = 0; d < 3; ++d) vc[d] = inreg ? vcr[j][d] : a.vc[3 * c + d];
        double Gd[4];
        cm_eval(cm, vc, a.cvhat[c], a.cmug[c], g, Gd);
        r0[0] += g[0] * dvc[0] + g[1] * dvc[1] + g[2] * dvc[2];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          if (inreg) dvcr[j][d] = dvc[d];
          else a.dvc[3 * c + d] = dvc[d];
        }
      })
      double d0s[1];
      group_reduce<1>(gr, sync, parity, cparity, r0, d0s, sm, cslot);
      lap(2);
      const double d0 = a1 + d0s[0];
      if (!isfinite(d0) || d0 >= 0.0) {
        status = MPMRB_E_NOT_DESCENT;
      } else {
        // ---- LS: exact line search (solver.py:266-298)
        double lo = 0.0, hi = INFINITY, alpha = 1.0;
        alpha_final = -1.0;
        int evals = 0;
        for (int ev = 1; ev <= a.ls_max; ++ev) {
          double rr[2] = {0.0, 0.0};
          FOR_OWNED_CONTACTS({
            double vc[3], dvc[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              dvc[d] = inreg ? dvcr[j][d] : a.dvc[3 * c + d];
              vc[d] = (inreg ? vcr[j][d] : a.vc[3 * c + d]) + alpha * dvc[d];
            }
            double g[3], G[4];
            cm_eval(cm, vc, a.cvhat[c], a.cmug[c], g, G);
            rr[0] += g[0] * dvc[0] + g[1] * dvc[1] + g[2] * dvc[2];
            rr[1] += dvc[0] * (G[0] * dvc[0] + G[3] * dvc[1]) +
                     dvc[1] * (G[3] * dvc[0] + G[1] * dvc[1]) + dvc[2] * (G[2] * dvc[2]);
          })
          double ss[2];
          group_reduce<2>(gr, sync, parity, cparity, rr, ss, sm, cslot);
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
        lap(3);
        // ---- U (contacts): vc += alpha dvc and the contact terms for the next N
        e_acc = 0.0;
        FOR_OWNED_CONTACTS({
          double vc[3], R[9], gw[3], rgr[6];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if (inreg) vc[d] = vcr[j][d] = vcr[j][d] + alpha_final * dvcr[j][d];
            else vc[d] = a.vc[3 * c + d] + alpha_final * a.dvc[3 * c + d];
            a.vc[3 * c + d] = vc[d];
          }
          load_frame(a.frames, c, R);
          e_acc += contact_terms(cm, vc, a.cvhat[c], a.cmug[c], R, gw, rgr);
#pragma unroll
          for (int d = 0; d < 3; ++d) a.gw[3 * c + d] = gw[d];
#pragma unroll
          for (int q = 0; q < 6; ++q) a.rgr[6 * c + q] = rgr[q];
        })
      }
      // publish the step (and the status) to the CTAs outside the group
      if (gr.rank == 0 && threadIdx.x == 0) {
        a.ls_out[0] = alpha_final;
        a.ls_out[1] = (double)status;
        if (a.tr_alpha && status == 0) a.tr_alpha[it] = alpha_final;
      }
    }
    sync();  // gw/rgr, alpha and status visible grid-wide
    if (!gr.member || gr.cluster) {
      alpha_final = __ldcg(&a.ls_out[0]);
      status = (int)__ldcg(&a.ls_out[1]);
    }
    lap(4);
    if (status) break;
    alpha_prev = alpha_final;
    ++iterations;
  }
  // The last N applied every pending update, so v is final here (grid synced).
  // ---- epilogue: impulses gamma = -g_c(vc) (solver.py:363-365)
  bool finite_v = true;
  for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double vi = v[3 * i + d];
      finite_v &= isfinite(vi);
      if (a.v_next_full) a.v_next_full[3 * (long long)a.act[i] + d] = vi;
    }
  }
  FOR_OWNED_CONTACTS({
    double vc[3], g[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) vc[d] = inreg ? vcr[j][d] : a.vc[3 * c + d];
    double Gd[4];
    cm_eval(cm, vc, a.cvhat[c], a.cmug[c], g, Gd);
#pragma unroll
    for (int d = 0; d < 3; ++d) a.gamma[3 * c + d] = -g[d];
  })
#undef FOR_OWNED_CONTACTS
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  if (!finite_v) s_flag = 1;
  __syncthreads();
  if (s_flag && threadIdx.x == 0) atomicOr(&a.out->status_flags, 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out->converged = converged ? 1 : 0;
    a.out->iterations = iterations;
    a.out->ls_evals = ls_evals_total;
    a.out->status = status;
    a.out->n_contacts = nc;
    a.out->n_dofs = 3 * nd;
    if (prof) {
      lap(5);
      for (int k = 0; k < 6; ++k) a.prof[k] += pt[k];
      a.prof[6] += (unsigned long long)iterations;
      a.prof[7] += (unsigned long long)ls_evals_total;
      a.prof[8] += (unsigned long long)nctas + ((unsigned long long)gr.size << 32);
      a.prof[9] += 1ull;
      a.prof[11] += (unsigned long long)n_cn + ((unsigned long long)n_hn << 32);
      a.prof[12] += pt[12];
      a.prof[13] += pt[13];
    }
  }
}

// ---------------------------------------------------------------- adjacency

__global__ void k_adj_count(const int* __restrict__ nc_dev, long long nc_cap,
                            const int* __restrict__ cnodes, const double* __restrict__ cw,
                            int* __restrict__ cnt) {
  const long long nc = *nc_dev;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nc * 27) return;
  const long long k = e / nc, c = e - k * nc;
  if (cw[k * nc_cap + c] != 0.0) atomicAdd(&cnt[cnodes[k * nc_cap + c]], 1);
}

__global__ void k_adj_fill(const int* __restrict__ nc_dev, long long nc_cap,
                           const int* __restrict__ cnodes, const double* __restrict__ cw,
                           const int* __restrict__ off, int* __restrict__ fill,
                           int* __restrict__ ent) {
  const long long nc = *nc_dev;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nc * 27) return;
  const long long k = e / nc, c = e - k * nc;
  if (cw[k * nc_cap + c] == 0.0) return;
  const int node = cnodes[k * nc_cap + c];
  const int pos = off[node] + atomicAdd(&fill[node], 1);
  ent[pos] = (int)((c << 5) | k);
}

// Place every entry at its sorted position inside its node's segment: the
// rank is the number of smaller keys in the same segment (keys are unique),
// so the gathers sum in (contact, slot) order regardless of the atomic fill
// order.  Entry-parallel: O(L) work per entry, no serial per-node sort.
__global__ void k_adj_rank(const int* __restrict__ nd_dev, long long nc_cap,
                           const int* __restrict__ cnodes, const double* __restrict__ cw,
                           const int* __restrict__ off, const int* __restrict__ ent_u,
                           int* __restrict__ ent, double* __restrict__ wout) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int total = off[*nd_dev];
  if (e >= total) return;
  const int key = ent_u[e];
  const long long c = key >> 5, k = key & 31;
  const int node = cnodes[k * nc_cap + c];
  const int b = off[node], en = off[node + 1];
  int rank = 0;
  for (int p = b; p < en; ++p) rank += (__ldg(&ent_u[p]) < key) ? 1 : 0;
  ent[b + rank] = key;
  wout[b + rank] = cw[k * nc_cap + c];
}

__global__ void k_adj_flag(const int* __restrict__ nd_dev, const int* __restrict__ off,
                           int* __restrict__ flag, int* __restrict__ hflag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= *nd_dev) return;
  const int L = off[i + 1] - off[i];
  flag[i] = (L > 0 && L <= kHeavyNode) ? 1 : 0;
  hflag[i] = (L > kHeavyNode) ? 1 : 0;
}

__global__ void k_adj_lists(const int* __restrict__ nd_dev, SolverAdjacency adj) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= *nd_dev) return;
  const int o = adj.flag_off[i], ho = adj.hflag_off[i];
  if (adj.flag[i]) {
    adj.cn[o] = (int)i;
    adj.cn_e[2 * o] = adj.off[i];
    adj.cn_e[2 * o + 1] = adj.off[i + 1];
  } else if (adj.hflag[i]) {
    adj.hn[ho] = (int)i;
    adj.hn_e[2 * ho] = adj.off[i];
    adj.hn_e[2 * ho + 1] = adj.off[i + 1];
  } else {
    adj.fn[i - o - ho] = (int)i;
  }
}

}  // namespace

int launch_solver_adjacency(Ctx& c, const int* nd_dev, const int* nc_dev, long long nd_cap,
                            long long nc_cap, const int* cnodes, const double* cw,
                            const SolverAdjacency& adj, DevBuf& tiles) {
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.cnt, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.fill, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.flag, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.hflag, 0, sizeof(int) * (nd_cap + 1), c.stream));
  const long long ne = nc_cap * 27;
  if (ne > 0) {
    k_adj_count<<<grid_for(ne, 256), 256, 0, c.stream>>>(nc_dev, nc_cap, cnodes, cw, adj.cnt);
    c.launches++;
  }
  // exclusive scan over nd+1 entries (the trailing zero makes off[nd] the total)
  int rc = scan_exclusive_i32(c, adj.cnt, adj.off, nd_cap + 1, nullptr, nullptr, tiles);
  if (rc) return rc;
  if (ne > 0) {
    k_adj_fill<<<grid_for(ne, 256), 256, 0, c.stream>>>(nc_dev, nc_cap, cnodes, cw, adj.off,
                                                        adj.fill, adj.ent_tmp);
    k_adj_rank<<<grid_for(ne, 256), 256, 0, c.stream>>>(nd_dev, nc_cap, cnodes, cw, adj.off,
                                                        adj.ent_tmp, adj.ent, adj.w);
    c.launches += 2;
  }
  if (nd_cap > 0) {
    k_adj_flag<<<grid_for(nd_cap, 256), 256, 0, c.stream>>>(nd_dev, adj.off, adj.flag,
                                                            adj.hflag);
    c.launches++;
  }
  rc = scan_exclusive_i32(c, adj.flag, adj.flag_off, nd_cap + 1, nullptr, adj.n_cn, tiles);
  if (rc) return rc;
  rc = scan_exclusive_i32(c, adj.hflag, adj.hflag_off, nd_cap + 1, nullptr, adj.n_hn, tiles);
  if (rc) return rc;
  if (nd_cap > 0) {
    k_adj_lists<<<grid_for(nd_cap, 256), 256, 0, c.stream>>>(nd_dev, adj);
    c.launches++;
  }
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas) {
  // Grid: one CTA per SM (launch bounds + 128 registers).  Preferred launch:
  // clusters of 8 (the contact group is cluster 0) as many as co-reside.
  static int sms = -1, cluster_grid = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms > kMaxSolverCtas) sms = kMaxSolverCtas;
    cluster_grid = 0;
    // Opt-in: measured on the 256k sand pile (17.5k contacts) the 8-CTA
    // contact cluster loses to grid-wide ownership (6.5 vs 4.8 us per
    // line-search evaluation: the fp64 divide/sqrt work of 17.5k contacts on
    // 8 SMs outweighs the cheaper cluster barrier).
    const char* env = getenv("MPMRB_SOLVER_CLUSTER");
    if (env && atoi(env) > 0) {
      cudaLaunchConfig_t q = {};
      q.blockDim = dim3(kThreads);
      q.gridDim = dim3(kSolverCluster);
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = kSolverCluster;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k_qn_solve, &q) == cudaSuccess && ncl > 0) {
        cluster_grid = ncl * kSolverCluster;
        if (cluster_grid > kMaxSolverCtas) cluster_grid = (kMaxSolverCtas / kSolverCluster) * kSolverCluster;
      }
      cudaGetLastError();
    }
  }
  int g = sms;
  bool use_cluster = cluster_grid > 0;
  if (use_cluster) g = cluster_grid;
  if (grid_ctas > 0 && grid_ctas < g) {
    g = grid_ctas;
    use_cluster = false;
  }
  if (a.force_ctas > 1) {
    g = a.force_ctas < sms ? a.force_ctas : sms;
    use_cluster = false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = use_cluster ? kSolverCluster : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_cluster ? 2 : 1;
  MPMRB_CUDA_OK(cudaLaunchKernelEx(&cfg, k_qn_solve, a));
  c.launches++;
  return MPMRB_OK;
}

}  // namespace mpmrb
