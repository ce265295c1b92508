// Globally convergent quasi-Newton convex contact solve on sm_100a
// (solver.py:197-382), run entirely on the device as ONE persistent kernel:
// no host round trip per iteration or per line-search evaluation.
//
// Layout: the problem is restricted to active nodes (solver.py:197-221);
// per-contact stencils are slot-major [27][nc_cap] (coalesced across
// contacts).  Each phase is a grid-stride loop over nodes or contacts followed
// by a barrier.  With a single CTA the barrier is __syncthreads(); with several
// CTAs it is a sense-reversing grid barrier (all CTAs are co-resident: the
// grid never exceeds one CTA per SM).  Reductions (residual, norms, line
// search phi'/phi'') are summed per CTA, then every CTA sums the per-CTA
// partials in the same fixed order, so all CTAs take identical branch
// decisions (convergence test, line-search bracketing).
//
// Phases per iteration (solver.py:338-357):
//   P_grad   contacts: g_c(vc) -> J^T scatter (3 ch)                [barrier]
//   P_node   nodes: g = M(v-v*) + J^T g_c; residual, norms, energy [reduce]
//   P_hess   contacts: w^2 R^T G R scatter (6 ch)                   [barrier]
//   P_dir    nodes: 3x3 Cholesky, dv; a1, a2                       [reduce]
//   P_dvc    contacts: dvc = R J dv; phi'(0) contact term           [reduce]
//   P_ls     <= ls_max evaluations of phi'(a), phi''(a)             [reduce each]
//   P_upd    nodes: v += a dv                                      [barrier]
//   P_vc     contacts: vc = R J v + b                               [barrier]
#include "common.cuh"
#include "contact.cuh"
#include "internal.h"
#include "solver.cuh"

namespace mpmrb {

namespace {

constexpr int kThreads = kSolverThreads;
constexpr int kMaxRed = 8;  // reduction lanes per call

struct Sync {
  unsigned* bar;   // [0] count, [1] generation
  int nctas;
  __device__ __forceinline__ void operator()() const {
    if (nctas == 1) {
      __syncthreads();
      return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      volatile unsigned* gen = bar + 1;
      unsigned g = *gen;
      __threadfence();
      if (atomicAdd(bar, 1u) == (unsigned)nctas - 1u) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicExch(bar + 1, g + 1u);
      } else {
        while (*gen == g) __nanosleep(20);
      }
      __threadfence();
    }
    __syncthreads();
  }
};

// Sum K values over all threads of all active CTAs; result in out[] of every
// thread.  Deterministic order given nctas.
// partials is double-buffered: a CTA that races into the next reduction
// writes the other half while slower CTAs still read this one; the barrier
// inside the next call closes the window before the half is reused.
template <int K>
__device__ void reduce_all(const Sync& sync, double* partials_base, int& parity,
                           double (&v)[K], double (&out)[K],
                           double* sm /*32*kMaxRed + kMaxRed*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* partials = partials_base + parity * (kMaxRed * kMaxSolverCtas);
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
        else partials[k * kMaxSolverCtas + blockIdx.x] = x;
      }
    }
  }
  if (sync.nctas > 1) {
    sync();
    if (wid == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double x = 0.0;
        for (int c = lane; c < sync.nctas; c += 32) x += __ldcg(&partials[k * kMaxSolverCtas + c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) sm[32 * kMaxRed + k] = x;
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
  for (int k = 0; k < 9; ++k) R[k] = __ldcg(fr + 9 * c + k);
}

// R (sum_k w_k u[node_k]) (+ bias)
__device__ __forceinline__ void gather_contact(const SolverArgs& a, long long c,
                                               const double* __restrict__ u, const double* R,
                                               bool add_bias, double* out) {
  double up[3] = {0.0, 0.0, 0.0};
#pragma unroll 3
  for (int k = 0; k < 27; ++k) {
    int nd = a.cnodes[(long long)k * a.nc_cap + c];
    double w = a.cw[(long long)k * a.nc_cap + c];
#pragma unroll
    for (int d = 0; d < 3; ++d) up[d] += w * __ldcg(&u[3 * nd + d]);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    out[r] = R[3 * r] * up[0] + R[3 * r + 1] * up[1] + R[3 * r + 2] * up[2];
    if (add_bias) out[r] += a.bias[3 * c + r];
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
      a.out->regularized = 0;
      a.out->status = 0;
      a.out->n_contacts = 0;
      a.out->n_dofs = 3 * nd;
    }
    return;
  }
  // active CTA count from the problem size (identical in every CTA)
  int want = max((nc + 255) / 256, (nd + 4095) / 4096);
  int nctas = min(max(want, 1), (int)gridDim.x);
  if (a.force_ctas > 0) nctas = min(a.force_ctas, (int)gridDim.x);
  if ((int)blockIdx.x >= nctas) return;
  Sync sync{a.bar, nctas};
  const long long tid = (long long)blockIdx.x * kThreads + threadIdx.x;
  const long long nthr = (long long)nctas * kThreads;
  const ContactModel cm{a.K, a.den, a.eps_v};
  double* v = a.v;

  // ---- init: v = v0, vc = R J v + b, zero scatter targets
  for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      v[3 * i + d] = a.v0[3 * i + d];
      a.jt[3 * i + d] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) a.H6[6 * i + k] = 0.0;
  }
  sync();
  for (long long c = tid; c < nc; c += nthr) {
    double R[9], vc[3];
    load_frame(a.frames, c, R);
    gather_contact(a, c, v, R, true, vc);
#pragma unroll
    for (int d = 0; d < 3; ++d) a.vc[3 * c + d] = vc[d];
  }
  sync();

  int iterations = 0, ls_evals_total = 0, status = 0;
  int red_parity = 0;
  bool converged = false;
  double residual = 0.0, threshold = 0.0;
  for (int it = 0;; ++it) {
    // ---- P_grad: contact gradient scatter J^T g_c (solver.py:127-140)
    for (long long c = tid; c < nc; c += nthr) {
      double vc[3] = {__ldcg(&a.vc[3 * c]), __ldcg(&a.vc[3 * c + 1]), __ldcg(&a.vc[3 * c + 2])};
      double g[3];
      cm_gradient(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], g);
      double R[9];
      load_frame(a.frames, c, R);
      double gw[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) gw[j] = g[0] * R[j] + g[1] * R[3 + j] + g[2] * R[6 + j];
      for (int k = 0; k < 27; ++k) {
        double w = a.cw[(long long)k * a.nc_cap + c];
        if (w == 0.0) continue;
        int ndx = a.cnodes[(long long)k * a.nc_cap + c];
#pragma unroll
        for (int d = 0; d < 3; ++d) atomicAdd(&a.jt[3 * ndx + d], w * gw[d]);
      }
    }
    sync();
    // ---- P_node: total gradient, residual/threshold, objective (solver.py:111-119,188-194)
    double red[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (long long i = tid; i < nd; i += nthr) {
      double m = a.m[i];
      double inv_m = 1.0 / m;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double vi = __ldcg(&v[3 * i + d]);
        double dvs = vi - a.v_star[3 * i + d];
        double jt = __ldcg(&a.jt[3 * i + d]);
        double g = m * dvs + jt;
        a.g[3 * i + d] = g;
        a.jt[3 * i + d] = 0.0;  // ready for the next scatter
        red[0] += g * g * inv_m;
        red[1] += m * vi * vi;
        red[2] += jt * jt * inv_m;
        red[3] += m * dvs * dvs;
      }
    }
    for (long long c = tid; c < nc; c += nthr) {
      double vc[3] = {__ldcg(&a.vc[3 * c]), __ldcg(&a.vc[3 * c + 1]), __ldcg(&a.vc[3 * c + 2])};
      red[4] += cm_energy(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c]);
    }
    double sums[5];
    reduce_all<5>(sync, a.partials, red_parity, red, sums, sm);
    residual = sqrt(sums[0]);
    double p_norm = sqrt(sums[1]), j_norm = sqrt(sums[2]);
    threshold = a.eps_a + a.eps_r * fmax(p_norm, j_norm);
    double objective = 0.5 * sums[3] + sums[4];
    if (blockIdx.x == 0 && threadIdx.x == 0 && it <= a.max_iters) {
      if (a.tr_obj) a.tr_obj[it] = objective;
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
    // ---- P_hess: block-diagonal Hessian scatter (solver.py:151-167)
    for (long long c = tid; c < nc; c += nthr) {
      double vc[3] = {__ldcg(&a.vc[3 * c]), __ldcg(&a.vc[3 * c + 1]), __ldcg(&a.vc[3 * c + 2])};
      double G[4];
      cm_hessian(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], G);
      double R[9];
      load_frame(a.frames, c, R);
      // GR = G @ R with G = [[G0,G3,0],[G3,G1,0],[0,0,G2]]; rgr = R^T GR
      double GR[9];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        GR[j] = G[0] * R[j] + G[3] * R[3 + j];
        GR[3 + j] = G[3] * R[j] + G[1] * R[3 + j];
        GR[6 + j] = G[2] * R[6 + j];
      }
      // entries used by the Cholesky: 00, 11, 22, 10, 20, 21
      double rgr[6];
      const int ri[6] = {0, 1, 2, 1, 2, 2}, rj[6] = {0, 1, 2, 0, 0, 1};
#pragma unroll
      for (int e = 0; e < 6; ++e)
        rgr[e] = R[ri[e]] * GR[rj[e]] + R[3 + ri[e]] * GR[3 + rj[e]] + R[6 + ri[e]] * GR[6 + rj[e]];
      for (int k = 0; k < 27; ++k) {
        double w = a.cw[(long long)k * a.nc_cap + c];
        if (w == 0.0) continue;
        double w2 = w * w;
        int ndx = a.cnodes[(long long)k * a.nc_cap + c];
#pragma unroll
        for (int e = 0; e < 6; ++e) atomicAdd(&a.H6[6 * ndx + e], w2 * rgr[e]);
      }
    }
    sync();
    // ---- P_dir: d = -H^{-1} g per node, a1, a2 (solver.py:224-256, 305-307)
    double red2[3] = {0.0, 0.0, 0.0};
    int bad_any = 0, reg_count = 0;
    for (long long i = tid; i < nd; i += nthr) {
      double m = a.m[i];
      double h[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        h[e] = __ldcg(&a.H6[6 * i + e]);
        a.H6[6 * i + e] = 0.0;
      }
      h[0] = m + h[0];
      h[1] = m + h[1];
      h[2] = m + h[2];
      double l11, l21, l31, l22, l32, l33;
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
        if (good) break;
        if (attempt == 3) break;
        ++reg_count;
        double tr = h[0] + h[1] + h[2];
        double bump = 1e-12 * fmax(tr, 1.0) * pow(10.0, (double)attempt);
        h[0] += bump;
        h[1] += bump;
        h[2] += bump;
      }
      if (!good) bad_any = 1;
      double g0 = a.g[3 * i], g1 = a.g[3 * i + 1], g2 = a.g[3 * i + 2];
      double y1 = -g0 / l11;
      double y2 = (-g1 - l21 * y1) / l22;
      double y3 = (-g2 - l31 * y1 - l32 * y2) / l33;
      double x3 = y3 / l33;
      double x2 = (y2 - l32 * x3) / l22;
      double x1 = (y1 - l21 * x2 - l31 * x3) / l11;
      double dvv[3] = {x1, x2, x3};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        a.dv[3 * i + d] = dvv[d];
        double vi = __ldcg(&v[3 * i + d]);
        double mdv = m * dvv[d];
        red2[0] += (vi - a.v_star[3 * i + d]) * mdv;
        red2[1] += dvv[d] * mdv;
      }
    }
    red2[2] = (double)bad_any;
    double s2[3];
    reduce_all<3>(sync, a.partials, red_parity, red2, s2, sm);
    if (reg_count) atomicAdd(&a.out->regularized, reg_count);
    if (s2[2] > 0.0) {
      status = MPMRB_E_NONFINITE;  // "Hessian block not SPD after regularization"
      break;
    }
    const double a1 = s2[0], a2 = s2[1];
    // ---- P_dvc: dvc = R J dv and the phi'(0) contact term (solver.py:308-310, 269)
    double r0[1] = {0.0};
    for (long long c = tid; c < nc; c += nthr) {
      double R[9], dvc[3];
      load_frame(a.frames, c, R);
      gather_contact(a, c, a.dv, R, false, dvc);
#pragma unroll
      for (int d = 0; d < 3; ++d) a.dvc[3 * c + d] = dvc[d];
      double vc[3] = {__ldcg(&a.vc[3 * c]), __ldcg(&a.vc[3 * c + 1]), __ldcg(&a.vc[3 * c + 2])};
      double g[3];
      cm_gradient(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], g);
      r0[0] += g[0] * dvc[0] + g[1] * dvc[1] + g[2] * dvc[2];
    }
    double d0s[1];
    reduce_all<1>(sync, a.partials, red_parity, r0, d0s, sm);
    const double d0 = a1 + d0s[0];
    if (!isfinite(d0) || d0 >= 0.0) {
      status = MPMRB_E_NOT_DESCENT;
      break;
    }
    // ---- P_ls: exact line search (solver.py:266-298)
    double lo = 0.0, hi = INFINITY, alpha = 1.0, dcur = d0;
    double alpha_final = -1.0;
    int evals = 0;
    for (int ev = 1; ev <= a.ls_max; ++ev) {
      double rr[2] = {0.0, 0.0};
      for (long long c = tid; c < nc; c += nthr) {
        double dvc[3] = {__ldcg(&a.dvc[3 * c]), __ldcg(&a.dvc[3 * c + 1]), __ldcg(&a.dvc[3 * c + 2])};
        double vc[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) vc[d] = __ldcg(&a.vc[3 * c + d]) + alpha * dvc[d];
        double g[3], G[4];
        cm_gradient(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], g);
        cm_hessian(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], G);
        rr[0] += g[0] * dvc[0] + g[1] * dvc[1] + g[2] * dvc[2];
        double Gd0 = G[0] * dvc[0] + G[3] * dvc[1];
        double Gd1 = G[3] * dvc[0] + G[1] * dvc[1];
        double Gd2 = G[2] * dvc[2];
        rr[1] += dvc[0] * Gd0 + dvc[1] * Gd1 + dvc[2] * Gd2;
      }
      double ss[2];
      reduce_all<2>(sync, a.partials, red_parity, rr, ss, sm);
      evals = ev;
      double d = a1 + a2 * alpha + ss[0];
      double dd = a2 + ss[1];
      dcur = d;
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
    (void)dcur;
    ls_evals_total += evals;
    // ---- P_upd: v += alpha dv
    for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
      for (int d = 0; d < 3; ++d) v[3 * i + d] = __ldcg(&v[3 * i + d]) + alpha_final * a.dv[3 * i + d];
    }
    ++iterations;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.tr_alpha) a.tr_alpha[it] = alpha_final;
    sync();
    // ---- P_vc: recompute contact velocities at the new iterate
    for (long long c = tid; c < nc; c += nthr) {
      double R[9], vc[3];
      load_frame(a.frames, c, R);
      gather_contact(a, c, v, R, true, vc);
#pragma unroll
      for (int d = 0; d < 3; ++d) a.vc[3 * c + d] = vc[d];
    }
    sync();
  }
  // ---- epilogue: impulses gamma = -g_c(vc) (solver.py:363-365, 141-144)
  bool finite_v = true;
  for (long long i = tid; i < nd; i += nthr) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double vi = __ldcg(&v[3 * i + d]);
      finite_v &= isfinite(vi);
      if (a.v_next_full) a.v_next_full[3 * (long long)a.act[i] + d] = vi;
    }
  }
  for (long long c = tid; c < nc; c += nthr) {
    double vc[3] = {__ldcg(&a.vc[3 * c]), __ldcg(&a.vc[3 * c + 1]), __ldcg(&a.vc[3 * c + 2])};
    double g[3];
    cm_gradient(cm, vc, a.phi[c], a.gamma_lag[c], a.mu[c], g);
#pragma unroll
    for (int d = 0; d < 3; ++d) a.gamma[3 * c + d] = -g[d];
  }
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  if (!finite_v) s_flag = 1;
  __syncthreads();
  if (s_flag) atomicOr(&a.out->status_flags, 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out->converged = converged ? 1 : 0;
    a.out->iterations = iterations;
    a.out->ls_evals = ls_evals_total;
    a.out->status = status;
    a.out->n_contacts = nc;
    a.out->n_dofs = 3 * nd;
  }
}

}  // namespace

int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas) {
  static int max_ctas = -1;
  if (max_ctas < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_qn_solve, kThreads, 0);
    max_ctas = sms * (per_sm > 0 ? 1 : 0);
    if (max_ctas > kMaxSolverCtas) max_ctas = kMaxSolverCtas;
    if (max_ctas < 1) max_ctas = 1;
  }
  int g = grid_ctas > 0 ? (grid_ctas < max_ctas ? grid_ctas : max_ctas) : max_ctas;
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
