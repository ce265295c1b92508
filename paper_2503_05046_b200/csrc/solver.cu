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
    for (int d = 0; d < 3; ++d) up[d] += w * __ldcg(&u[3 * nd + d]);
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
__device__ __forceinline__ void node_finish(const SolverArgs& a, long long i, const double* jt,
                                            const double* hs, double* red, int& reg_count) {
  const double m = a.m[i];
  const double inv_m = 1.0 / m;
  double dvs[3], g[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double vi = __ldcg(&a.v[3 * i + d]);
    dvs[d] = vi - a.v_star[3 * i + d];
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

__global__ void __launch_bounds__(kThreads, 1) k_qn_solve(SolverArgs a) {
  __shared__ double sm[32 * kMaxRed + kMaxRed];
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
  int parity = 0;
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
  const int n_fn = nd - n_cn;

  // Contacts are interleaved across CTAs (consecutive contacts on different
  // SMs) so the fp64 divide/sqrt work of the line search spreads over the
  // whole GPU.  A thread's first kJR contacts live in registers (fully
  // unrolled j, so the arrays never spill); any further ones go through
  // global memory.
  const long long ctid = (long long)threadIdx.x * nctas + blockIdx.x;
#define FOR_OWNED_CONTACTS(...)                                         \
  _Pragma("unroll") for (int j = 0; j < kJR; ++j) {                    \
    const long long c = ctid + (long long)j * nthr;                    \
    constexpr bool inreg = true;                                        \
    if (c < nc) { __VA_ARGS__ }                                         \
  }                                                                     \
  for (long long c = ctid + (long long)kJR * nthr; c < nc; c += nthr) { \
    constexpr int j = 0;                                                \
    constexpr bool inreg = false;                                       \
    __VA_ARGS__                                                         \
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
  for (int it = 0;; ++it) {
    // ---- N: node gathers, gradient, residual, Hessian block, direction
    double red[8] = {0, 0, 0, 0, e_acc, 0, 0, 0};
    int reg_count = 0;
    // (a) contact nodes: one warp per node over its CSR entries
    for (long long t = gwarp; t < n_cn; t += nwarps) {
      const long long i = a.adj.cn[t];
      const int e0 = a.adj.off[i], e1 = a.adj.off[i + 1];
      double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 2
      for (int e = e0 + lane; e < e1; e += 32) {
        const long long c = __ldg(&a.adj.ent[e]) >> 5;
        const double w = __ldg(&a.adj.w[e]);
        const double w2 = w * w;
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[d] += w * __ldcg(&a.gw[3 * c + d]);
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[3 + q] += w2 * __ldcg(&a.rgr[6 * c + q]);
      }
#pragma unroll
      for (int q = 0; q < 9; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
      if (lane == 0) node_finish(a, i, acc, acc + 3, red, reg_count);
    }
    // (b) nodes without contacts: thread per node
    {
      const double zero[6] = {0, 0, 0, 0, 0, 0};
      for (long long t = tid; t < n_fn; t += nthr) node_finish(a, a.adj.fn[t], zero, zero, red,
                                                               reg_count);
    }
    if (reg_count) atomicAdd(&a.out->regularized, reg_count);
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
    // ---- D: dvc = R J dv and the phi'(0) contact term (solver.py:305-310, 269)
    double r0[1] = {0.0};
    FOR_OWNED_CONTACTS({
      double R[9], dvc[3], vc[3], g[3];
      load_frame(a.frames, c, R);
      gather_contact(a, c, a.dv, R, dvc);
#pragma unroll
      for (int d = 0; d < 3; ++d) vc[d] = inreg ? vcr[j][d] : __ldcg(&a.vc[3 * c + d]);
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
    reduce_all<1>(sync, parity, r0, d0s, sm);
    lap(2);
    const double d0 = a1 + d0s[0];
    if (!isfinite(d0) || d0 >= 0.0) {
      status = MPMRB_E_NOT_DESCENT;
      break;
    }
    // ---- LS: exact line search (solver.py:266-298)
    double lo = 0.0, hi = INFINITY, alpha = 1.0, alpha_final = -1.0;
    int evals = 0;
    for (int ev = 1; ev <= a.ls_max; ++ev) {
      double rr[2] = {0.0, 0.0};
      FOR_OWNED_CONTACTS({
        double vc[3], dvc[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          dvc[d] = inreg ? dvcr[j][d] : __ldcg(&a.dvc[3 * c + d]);
          vc[d] = (inreg ? vcr[j][d] : __ldcg(&a.vc[3 * c + d])) + alpha * dvc[d];
        }
        double g[3], G[4];
        cm_eval(cm, vc, a.cvhat[c], a.cmug[c], g, G);
        rr[0] += g[0] * dvc[0] + g[1] * dvc[1] + g[2] * dvc[2];
        rr[1] += dvc[0] * (G[0] * dvc[0] + G[3] * dvc[1]) + dvc[1] * (G[3] * dvc[0] + G[1] * dvc[1]) +
                 dvc[2] * (G[2] * dvc[2]);
      })
      double ss[2];
      reduce_all<2>(sync, parity, rr, ss, sm);
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
    // ---- U: v += alpha dv; vc += alpha dvc and the contact terms at the new iterate
    for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
      for (int d = 0; d < 3; ++d) v[3 * i + d] = __ldcg(&v[3 * i + d]) + alpha_final * a.dv[3 * i + d];
    }
    e_acc = 0.0;
    FOR_OWNED_CONTACTS({
      double vc[3], R[9], gw[3], rgr[6];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (inreg) vc[d] = vcr[j][d] = vcr[j][d] + alpha_final * dvcr[j][d];
        else vc[d] = __ldcg(&a.vc[3 * c + d]) + alpha_final * __ldcg(&a.dvc[3 * c + d]);
        a.vc[3 * c + d] = vc[d];
      }
      load_frame(a.frames, c, R);
      e_acc += contact_terms(cm, vc, a.cvhat[c], a.cmug[c], R, gw, rgr);
#pragma unroll
      for (int d = 0; d < 3; ++d) a.gw[3 * c + d] = gw[d];
#pragma unroll
      for (int q = 0; q < 6; ++q) a.rgr[6 * c + q] = rgr[q];
    })
    ++iterations;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.tr_alpha) a.tr_alpha[it] = alpha_final;
    sync();
    lap(4);
  }
  // ---- epilogue: impulses gamma = -g_c(vc) (solver.py:363-365)
  bool finite_v = true;
  for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double vi = __ldcg(&v[3 * i + d]);
      finite_v &= isfinite(vi);
      if (a.v_next_full) a.v_next_full[3 * (long long)a.act[i] + d] = vi;
    }
  }
  FOR_OWNED_CONTACTS({
    double vc[3], g[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) vc[d] = inreg ? vcr[j][d] : __ldcg(&a.vc[3 * c + d]);
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
      a.prof[8] += (unsigned long long)nctas;
      a.prof[9] += 1ull;
      a.prof[11] += (unsigned long long)n_cn;
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
                           int* __restrict__ flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= *nd_dev) return;
  flag[i] = off[i + 1] > off[i] ? 1 : 0;
}

__global__ void k_adj_lists(const int* __restrict__ nd_dev, const int* __restrict__ flag,
                            const int* __restrict__ flag_off, int* __restrict__ cn,
                            int* __restrict__ fn) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= *nd_dev) return;
  const int o = flag_off[i];
  if (flag[i]) cn[o] = (int)i;
  else fn[i - o] = (int)i;
}

}  // namespace

int launch_solver_adjacency(Ctx& c, const int* nd_dev, const int* nc_dev, long long nd_cap,
                            long long nc_cap, const int* cnodes, const double* cw,
                            const SolverAdjacency& adj, DevBuf& tiles) {
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.cnt, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.fill, 0, sizeof(int) * (nd_cap + 1), c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(adj.flag, 0, sizeof(int) * (nd_cap + 1), c.stream));
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
    k_adj_flag<<<grid_for(nd_cap, 256), 256, 0, c.stream>>>(nd_dev, adj.off, adj.flag);
    c.launches++;
  }
  rc = scan_exclusive_i32(c, adj.flag, adj.flag_off, nd_cap + 1, nullptr, adj.n_cn, tiles);
  if (rc) return rc;
  if (nd_cap > 0) {
    k_adj_lists<<<grid_for(nd_cap, 256), 256, 0, c.stream>>>(nd_dev, adj.flag, adj.flag_off,
                                                             adj.cn, adj.fn);
    c.launches++;
  }
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas) {
  static int max_ctas = -1;
  if (max_ctas < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_qn_solve, kThreads, 0);
    max_ctas = per_sm > 0 ? sms : 1;
    if (max_ctas > kMaxSolverCtas) max_ctas = kMaxSolverCtas;
  }
  int g = max_ctas;
  if (grid_ctas > 0 && grid_ctas < g) g = grid_ctas;
  if (a.force_ctas > 1 && a.force_ctas < g) g = a.force_ctas;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
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
