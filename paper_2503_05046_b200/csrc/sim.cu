// Fused substep pipeline (coupling.py:115-219) on sm_100a.
//
// One substep = grid build -> P2G -> grid update -> active compaction ->
// contact detection -> contact stencils / gamma_lag -> device-side QN solve
// -> reaction accumulation -> G2P, all sizes resolved on the device, captured
// once as a CUDA graph and replayed N times per coupling step with no host
// synchronisation.  The host (coupling.py's scheduler) only syncs once per
// step, in mpmrb_sim_end_step.
#include <nvtx3/nvToolsExt.h>

#include <cstring>
#include <vector>

#include "common.cuh"
#include "contact.cuh"
#include "internal.h"
#include "sim.h"
#include "solver.cuh"

namespace mpmrb {

namespace {

constexpr int kMaxBodies = 32;

struct NvtxRange {  // host-side range for nsys / ncu --nvtx
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

__global__ void k_emit_active(long long n_cap, const unsigned char* __restrict__ active,
                              const int* __restrict__ woff, const double* __restrict__ mass,
                              const double* __restrict__ v_star, const double* __restrict__ v_k,
                              int* __restrict__ act, int* __restrict__ remap,
                              double* __restrict__ m_c, double* __restrict__ vstar_c,
                              double* __restrict__ vk_c) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool a = (i < n_cap) && active[i];
  unsigned b = __ballot_sync(0xffffffffu, a);
  if (i >= n_cap) return;
  if (!a) {
    remap[i] = -1;
    return;
  }
  int lane = threadIdx.x & 31;
  int idx = woff[i >> 5] + __popc(b & ((1u << lane) - 1u));
  act[idx] = (int)i;
  remap[i] = idx;
  m_c[idx] = mass[i];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    vstar_c[3 * idx + d] = v_star[3 * i + d];
    vk_c[3 * idx + d] = v_k[3 * i + d];
  }
}

// Per contact: stencil of its particle, restricted to active nodes
// (solver.py:207-213), the substep-start contact velocity at v_k and the lagged
// normal impulse (coupling.py:131-133, contact_model.py:50-55).
__global__ void k_contact_prepare(GridDev g, const double* __restrict__ x,
                                  const int* __restrict__ nc_dev, long long nc_cap,
                                  const int* __restrict__ cpart, const double* __restrict__ frames,
                                  const double* __restrict__ bias, const double* __restrict__ phi,
                                  const double* __restrict__ v_k, const int* __restrict__ remap,
                                  double K, double den, int* __restrict__ cnodes,
                                  double* __restrict__ cw, double* __restrict__ gamma_lag,
                                  DevStatus* st) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nc = *nc_dev;
  if (nc > nc_cap) nc = nc_cap;
  if (c >= nc) return;
  long long p = cpart[c];
  double xp[3] = {x[3 * p], x[3 * p + 1], x[3 * p + 2]};
  Stencil1 s;
  make_stencil1(xp, g.h, s);
  StencilBlocks sb;
  if (!resolve_blocks(s, g.hkeys, g.hvals, g.mask, sb)) {
    raise_status(st, MPMRB_E_ALLOCATION, 50, c);
    return;
  }
  double vp[3] = {0.0, 0.0, 0.0};
  int k = 0;
  for (int ox = 0; ox < 3; ++ox)
    for (int oy = 0; oy < 3; ++oy)
      for (int oz = 0; oz < 3; ++oz, ++k) {
        double w = (s.w[0][ox] * s.w[1][oy]) * s.w[2][oz];
        int node = stencil_node(s, sb, ox, oy, oz);
#pragma unroll
        for (int d = 0; d < 3; ++d) vp[d] += w * v_k[3 * node + d];
        const int r = remap[node];
        const bool dead = r < 0 || w == 0.0;  // dead slot: w = 0, no node (solver.py:207-213)
        cnodes[(long long)k * nc_cap + c] = dead ? -1 : r;
        cw[(long long)k * nc_cap + c] = dead ? 0.0 : w;
      }
  const double* R = frames + 9 * c;
  double vn = (R[6] * vp[0] + R[7] * vp[1] + R[8] * vp[2]) + bias[3 * c + 2];
  double vhat = -phi[c] / den;
  gamma_lag[c] = K * fmax(0.0, vhat - vn);
}


// Reactions on bodies (coupling.py:58-66, 141-144), pass 1: gamma_world =
// gamma^T R per contact and per-CTA partial sums of -gamma_world and
// -arm x gamma_world per body (grid-stride over the device contact count).
constexpr int kReactCtas = 148;
constexpr int kReactThreads = 256;
constexpr int kReactBodies = 4;  // bodies accumulated per pass over the contacts

__global__ void __launch_bounds__(kReactThreads) k_reactions(
    const int* __restrict__ counters /*nb, n_act, nc*/, const double* __restrict__ gamma,
    const double* __restrict__ frames, const double* __restrict__ witness,
    const int* __restrict__ cbody, const mpmrb_geom* __restrict__ geoms, int ngeom, int nbody,
    long long nc_cap, double* __restrict__ gamma_world, double* __restrict__ partial) {
  __shared__ double wsum[kReactThreads / 32][kReactBodies * 6];
  __shared__ double body_pos[kMaxBodies][3];
  const long long nc = min((long long)counters[2], nc_cap);
  for (int gi = threadIdx.x; gi < ngeom; gi += blockDim.x) {
    int b = geoms[gi].body;
    if (b < kMaxBodies)
      for (int d = 0; d < 3; ++d) body_pos[b][d] = geoms[gi].body_pos[d];
  }
  __syncthreads();
  const int nb = nbody < kMaxBodies ? nbody : kMaxBodies;
  // bodies in passes of kReactBodies: each pass reads every contact once and
  // accumulates the 6 wrench components of those bodies in registers, then
  // reduces them all with one shared-memory exchange
  for (int b0 = 0; b0 < nb; b0 += kReactBodies) {
    double acc[kReactBodies][6];
#pragma unroll
    for (int j = 0; j < kReactBodies; ++j)
#pragma unroll
      for (int e = 0; e < 6; ++e) acc[j][e] = 0.0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc;
         c += (long long)gridDim.x * blockDim.x) {
      const double* R = frames + 9 * c;
      const double* gm = gamma + 3 * c;
      double gw[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) gw[j] = gm[0] * R[j] + gm[1] * R[3 + j] + gm[2] * R[6 + j];
      if (b0 == 0)
#pragma unroll
        for (int j = 0; j < 3; ++j) gamma_world[3 * c + j] = gw[j];
      const int bj = cbody[c] - b0;
      if (bj < 0 || bj >= kReactBodies) continue;
      const double arm[3] = {witness[3 * c] - body_pos[cbody[c]][0],
                             witness[3 * c + 1] - body_pos[cbody[c]][1],
                             witness[3 * c + 2] - body_pos[cbody[c]][2]};
      const double v6[6] = {gw[0], gw[1], gw[2], arm[1] * gw[2] - arm[2] * gw[1],
                            arm[2] * gw[0] - arm[0] * gw[2], arm[0] * gw[1] - arm[1] * gw[0]};
#pragma unroll
      for (int j = 0; j < kReactBodies; ++j)
        if (j == bj)
#pragma unroll
          for (int e = 0; e < 6; ++e) acc[j][e] += v6[e];
    }
    // warp sums, then warp 0 adds the warps' sums in warp order
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kReactBodies; ++j)
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        double x = acc[j][e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) wsum[wid][j * 6 + e] = x;
      }
    __syncthreads();
    if (threadIdx.x < kReactBodies * 6) {
      const int j = threadIdx.x / 6, e = threadIdx.x % 6;
      double x = 0.0;
      for (int w = 0; w < kReactThreads / 32; ++w) x += wsum[w][threadIdx.x];
      if (b0 + j < nb) partial[((long long)(b0 + j) * 6 + e) * kReactCtas + blockIdx.x] = x;
    }
    __syncthreads();
  }
}

struct SubstepStat {
  int nb, n_act, nc, iters, converged, ls_evals, regularized, status;
};

// Pass 2 (one warp): accumulate the partials in CTA order into the step's
// impulse accumulator, plus the per-substep statistics record.
__global__ void k_substep_end(const int* __restrict__ counters, const SolveOut* __restrict__ so,
                              const double* __restrict__ partial, int nbody,
                              double* __restrict__ accum, int* __restrict__ substep_idx,
                              SubstepStat* __restrict__ stats, int max_substeps, DevStatus* st) {
  // one warp per wrench component (all components' partial loads in flight
  // at once), each summing the kReactCtas partials in a fixed order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nb = nbody < kMaxBodies ? nbody : kMaxBodies;
  const bool any = counters[2] > 0;
  for (int q = wid; q < nb * 6; q += nw) {
    double x = 0.0;
    if (any)
      for (int k = lane; k < kReactCtas; k += 32) x += partial[(long long)q * kReactCtas + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) accum[q] -= x;
  }
  if (threadIdx.x == 0) {
    int k = *substep_idx;
    if (k < max_substeps) {
      SubstepStat r;
      r.nb = counters[0];
      r.n_act = counters[1];
      r.nc = counters[2];
      r.iters = so->iterations;
      r.converged = so->converged;
      r.ls_evals = so->ls_evals;
      r.regularized = so->regularized;
      r.status = so->status;
      stats[k] = r;
    }
    *substep_idx = k + 1;
    const int nc = counters[2];
    if (nc > 0 && so->status) raise_status(st, so->status, 60, k);
    if (nc > 0 && (so->status_flags & 1)) raise_status(st, MPMRB_E_NONFINITE, 61, k);
  }
}

__global__ void k_reset_solveout(SolveOut* so) {
  if (threadIdx.x == 0) {
    so->converged = 0;
    so->iterations = 0;
    so->ls_evals = 0;
    so->regularized = 0;
    so->status = 0;
    so->status_flags = 0;
  }
}

__global__ void k_set_solveout(SolveOut* so, int converged, int iterations, int ls_evals,
                               int regularized) {
  if (threadIdx.x == 0) {
    so->converged = converged;
    so->iterations = iterations;
    so->ls_evals = ls_evals;
    so->regularized = regularized;
    so->status = 0;
    so->status_flags = 0;
  }
}

long long next_pow2(long long v) {
  long long p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

// --------------------------------------------------------------------------

int Sim::reserve(long long n, long long nb_needed) {
  long long nb_cap_new = nb_needed * 2 + 64;
  bool grow = nb_cap_new > nb_cap || n != n_particles || ngeom * n > nc_cap;
  if (!grow) return MPMRB_OK;
  if (nb_cap_new < nb_cap) nb_cap_new = nb_cap;
  if (graph_exec) {
    cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
  }
  nb_cap = nb_cap_new;
  hash_cap = next_pow2(4 * nb_cap);
  long long N = nb_cap * kNodesPerBlock;
  long long nc = (long long)(ngeom > 0 ? ngeom : 1) * (n > 0 ? n : 1);
  nc_cap = nc;
  if (bias_n != n || bias_geoms < ngeom) {
    // new particle count or more geoms: cache slots restart empty
    if (b_bias_stamp.grow(sizeof(int) * (size_t)(ngeom > 0 ? ngeom : 1) * (n > 0 ? n : 1)) ||
        b_bias_store.grow(sizeof(double) * 3 * (size_t)(ngeom > 0 ? ngeom : 1) * (n > 0 ? n : 1)))
      return MPMRB_E_CUDA;
    MPMRB_CUDA_OK(cudaMemsetAsync(b_bias_stamp.p, 0, b_bias_stamp.bytes, ctx->stream));
    bias_n = n;
    bias_geoms = ngeom;
  }
  n_particles = n;
  int rc = 0;
  {
    const long long nn = n > 0 ? n : 1;
    rc |= b_qd.grow(8 * 27 * nn);
    rc |= b_qmid.grow(8 * nn);
    rc |= b_perm.grow(4 * nn);
    rc |= b_skeys.grow(4 * 2 * nn);
    rc |= b_svals.grow(4 * 2 * nn);
    rc |= b_cpart_user.grow(4 * (long long)(ngeom > 0 ? ngeom : 1) * nn);
    rc |= b_taucache.grow(8 * 6 * nn);
    rc |= b_tauvalid.grow(64);
    if (rc) return MPMRB_E_CUDA;
    double* d = b_qd.as<double>();
    q.x = d;
    q.v = d + 3 * nn;
    q.f = d + 6 * nn;
    q.c = d + 15 * nn;
    q.mass = d + 24 * nn;
    q.vol0 = d + 25 * nn;
    q.plastic = d + 26 * nn;
    q.mid = b_qmid.as<long long>();
    q.n = n;
    q.tau_cache = b_taucache.as<double>();
    q.tau_valid = b_tauvalid.as<int>();
    if (prec == MPMRB_PREC_F32) {
      if (b_qf.grow(4 * 30 * nn)) return MPMRB_E_CUDA;
      float* fp = b_qf.as<float>();
      q32.x = q.x;
      q32.v = fp;
      q32.f = fp + 3 * nn;
      q32.c = fp + 12 * nn;
      q32.mass = fp + 21 * nn;
      q32.vol0 = fp + 22 * nn;
      q32.plastic = fp + 23 * nn;
      q32.tau_cache = fp + 24 * nn;
      q32.mid = q.mid;
      q32.n = n;
      q32.tau_valid = q.tau_valid;
    }
  }
  rc |= b_hkeys.grow(8 * hash_cap);
  rc |= b_hvals.grow(4 * hash_cap);
  rc |= b_ukeys.grow(8 * nb_cap);
  rc |= b_bkeys.grow(8 * nb_cap);
  rc |= b_mass.grow(8 * N);
  rc |= b_mom.grow(8 * 6 * N);  // mom_apic (3N) followed by mom_force (3N)
  rc |= b_vk.grow(8 * 3 * N);
  rc |= b_vstar.grow(8 * 3 * N);
  rc |= b_vnext.grow(8 * 3 * N);
  rc |= b_active.grow(N);
  rc |= b_wcount.grow(4 * (N / 32 + 1));
  rc |= b_woff.grow(4 * (N / 32 + 1));
  rc |= b_act.grow(4 * N);
  rc |= b_remap.grow(4 * N);
  rc |= b_mc.grow(8 * N);
  rc |= b_vstarc.grow(8 * 3 * N);
  rc |= b_vkc.grow(8 * 3 * N);
  rc |= b_cnt.grow(4 * (n + 1));
  rc |= b_offs.grow(4 * (n + 1));
  rc |= b_cpart.grow(4 * nc_cap);
  rc |= b_cbody.grow(4 * nc_cap);
  rc |= b_cphi.grow(8 * nc_cap);
  rc |= b_cmu.grow(8 * nc_cap);
  rc |= b_cgl.grow(8 * nc_cap);
  rc |= b_cnormal.grow(8 * 3 * nc_cap);
  rc |= b_cwit.grow(8 * 3 * nc_cap);
  rc |= b_cbias.grow(8 * 3 * nc_cap);
  rc |= b_cframes.grow(8 * 9 * nc_cap);
  rc |= b_cnodes.grow(4 * 27 * nc_cap);
  rc |= b_cw.grow(8 * 27 * nc_cap);
  rc |= b_sv.grow(8 * 3 * N);
  rc |= b_sdv.grow(8 * 3 * N);
  rc |= b_svc.grow(8 * 5 * nc_cap);  // vc (3), vhat, mu*gamma_lag
  rc |= b_sdvc.grow(8 * 3 * nc_cap);
  rc |= b_su_c.grow(4 * 4 * (nc_cap + 2));  // head, head_off, grp_of, grp_start
  rc |= b_su_n.grow(4 * 14 * (N + 2) + 64);  // cnt, fill, off, flag, flag_off, cn, fn, counts, cn_rec (4), cnt_exp, off_exp
  rc |= b_su_ent.grow(2 * 4 * 27 * nc_cap);  // entries + tmp
  rc |= b_cellsum.grow(8 * kCellSumStride * nc_cap);  // per-contact records
  rc |= b_gamma.grow(8 * 3 * nc_cap);
  rc |= b_gworld.grow(8 * 3 * nc_cap);
  long long scan_n = (N + 1) > (n + 1) ? (N + 1) : (n + 1);
  rc |= b_tiles.grow(8 * (scan_n / 2048 + 2));
  if (rc) return MPMRB_E_CUDA;
  return MPMRB_OK;
}

int Sim::capture_or_launch(int part_lo, int part_hi) {
  Ctx& c = *ctx;
  // parts (mpmrb_sim_substep_part): 0 grid + P2G, 1 grid update + contacts,
  // 2 contact solve, 3 reactions + G2P
  auto in = [&](int k) { return part_lo <= k && k <= part_hi; };
  long long N = nb_cap * kNodesPerBlock;
  int* counters = b_counters.as<int>();  // [0] nb, [1] n_act, [2] nc, [3] substep idx
  GridDev g{b_hkeys.as<unsigned long long>(), b_hvals.as<int>(), (unsigned)(hash_cap - 1), h};
  int rc;
  double* mom_apic = b_mom.as<double>();
  double* mom_force = mom_apic + 3 * N;
  ContactArrays ca{};
  ca.particle = b_cpart.as<int>();
  ca.body = b_cbody.as<int>();
  ca.phi = b_cphi.as<double>();
  ca.normal = b_cnormal.as<double>();
  ca.witness = b_cwit.as<double>();
  ca.frames = b_cframes.as<double>();
  ca.bias = b_cbias.as<double>();
  ca.mu = b_cmu.as<double>();
  if (in(0)) {
  mark(0);
  // 1. grid (grid.py:71-103)
  rc = launch_grid_build(c, q.x, n_particles, h, b_bkeys.as<long long>(), nb_cap,
                         b_hkeys.as<unsigned long long>(), b_hvals.as<int>(), hash_cap,
                         b_ukeys.as<long long>(), counters + 0);
  if (rc) return rc;
  mark(1);
  // 2. P2G (mpm.py:66-99)
  MPMRB_CUDA_OK(cudaMemsetAsync(b_mass.p, 0, 8 * N, c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(b_mom.p, 0, 8 * 6 * N, c.stream));
  if (cloth.ne > 0) {  // cloth forces before the transfer (cloth.cu)
    rc = launch_cloth_forces(c, cloth, q, b_mats.as<mpmrb_material>(), nmat);
    if (rc) return rc;
  }
  rc = (prec == MPMRB_PREC_F32)
           ? launch_p2g(c, g, q32, b_mats.as<mpmrb_material>(), nmat, dt_s, b_mass.as<double>(),
                        mom_apic, mom_force)
           : launch_p2g(c, g, q, b_mats.as<mpmrb_material>(), nmat, dt_s, b_mass.as<double>(),
                        mom_apic, mom_force);
  if (rc) return rc;
  }
  if (in(1)) {
  mark(2);
  // 3. grid update + ordered active compaction (mpm.py:102-115, solver.py:203-205)
  rc = launch_grid_update(c, N, counters + 0, b_mass.as<double>(), mom_apic, mom_force, gravity[0],
                          gravity[1], gravity[2], dt_s, b_active.as<unsigned char>(),
                          b_vk.as<double>(), b_vstar.as<double>(), b_vnext.as<double>(),
                          b_wcount.as<int>());
  if (rc) return rc;
  rc = scan_exclusive_i32(c, b_wcount.as<int>(), b_woff.as<int>(), N / 32, nullptr, counters + 1,
                          b_tiles);
  if (rc) return rc;
  k_emit_active<<<grid_for(N, 256), 256, 0, c.stream>>>(
      N, b_active.as<unsigned char>(), b_woff.as<int>(), b_mass.as<double>(), b_vstar.as<double>(),
      b_vk.as<double>(), b_act.as<int>(), b_remap.as<int>(), b_mc.as<double>(),
      b_vstarc.as<double>(), b_vkc.as<double>());
  c.launches++;
  mark(3);
  // 4. contacts (collision.py:88-132)
  rc = launch_detect(c, q.x, n_particles, b_geoms.as<mpmrb_geom>(), ngeom, margin,
                     b_cnt.as<int>(), b_offs.as<int>(), counters + 2, b_tiles, nc_cap,
                     b_bias_stamp.as<int>(), b_bias_store.as<double>(), b_dyn.as<int>(), ca);
  if (rc) return rc;
  k_contact_prepare<<<grid_for(nc_cap, 128), 128, 0, c.stream>>>(
      g, q.x, counters + 2, nc_cap, ca.particle, ca.frames, ca.bias, ca.phi, b_vk.as<double>(),
      b_remap.as<int>(), K, den, b_cnodes.as<int>(), b_cw.as<double>(), b_cgl.as<double>(),
      c.status);
  c.launches++;
  }
  if (in(2)) {
  mark(4);
  // 5. quasi-Newton solve on the device (solver.py:328-382)
  k_reset_solveout<<<1, 32, 0, c.stream>>>(b_solveout.as<SolveOut>());
  c.launches++;
  SolverSetup su{};
  {
    int* ci = b_su_c.as<int>();
    su.head = ci;
    su.head_off = ci + (nc_cap + 2);
    su.grp_of = ci + 2 * (nc_cap + 2);
    su.grp_start = ci + 3 * (nc_cap + 2);
    int* ni = b_su_n.as<int>();
    su.cnt = ni;
    su.fill = ni + (N + 2);
    su.off = ni + 2 * (N + 2);
    su.flag = ni + 3 * (N + 2);
    su.flag_off = ni + 4 * (N + 2);
    su.cn = ni + 5 * (N + 2);
    su.fn = ni + 6 * (N + 2);
    su.counts = ni + 7 * (N + 2);
    su.cn_rec = reinterpret_cast<int4*>(ni + 8 * (N + 2));
    su.cnt_exp = ni + 12 * (N + 2);
    su.off_exp = ni + 13 * (N + 2);
    su.ent = b_su_ent.as<int>();
    su.ent_tmp = su.ent + 27 * nc_cap;
  }
  rc = launch_solver_setup(c, counters + 1, counters + 2, N, nc_cap, b_cnodes.as<int>(), su,
                           b_tiles);
  if (rc) return rc;
  SolverArgs a{};
  a.nd_dev = counters + 1;
  a.nc_dev = counters + 2;
  a.nc_cap = nc_cap;
  a.nd_cap = N;
  a.su = su;
  a.prof = c.solver_prof;
  a.m = b_mc.as<double>();
  a.v_star = b_vstarc.as<double>();
  a.v0 = b_vkc.as<double>();
  a.cnodes = b_cnodes.as<int>();
  a.cw = b_cw.as<double>();
  a.frames = ca.frames;
  a.bias = ca.bias;
  a.phi = ca.phi;
  a.mu = ca.mu;
  a.gamma_lag = b_cgl.as<double>();
  a.K = K;
  a.den = den;
  a.eps_v = eps_v;
  a.eps_a = sp.eps_a;
  a.eps_r = sp.eps_r;
  a.ls_tol = sp.ls_tol;
  a.max_iters = sp.max_iters;
  a.ls_max = sp.ls_max_iters;
  a.skip_if_no_contacts = 1;
  a.force_ctas = force_ctas;
  a.force_ls_ctas = force_ls_ctas;
  a.ext_free[0] = a.ext_free[1] = a.ext_free[2] = 0.0;
  a.p_out = nullptr;
  a.v = b_sv.as<double>();
  a.dv = b_sdv.as<double>();
  a.vc = b_svc.as<double>();
  a.cvhat = b_svc.as<double>() + 3 * nc_cap;
  a.cmug = b_svc.as<double>() + 4 * nc_cap;
  a.dvc = b_sdvc.as<double>();
  a.partials = b_partials.as<double>();
  a.cellsum = b_cellsum.as<double>();
  a.slots = b_slots.as<unsigned long long>();
  a.chan = reinterpret_cast<unsigned*>(b_slots.as<char>() + 8 * kSolverSlotWords);
  a.bar = reinterpret_cast<unsigned*>(b_slots.as<char>() + 8 * kSolverSlotWords + 64);
  a.gamma = b_gamma.as<double>();
  a.out = b_solveout.as<SolveOut>();
  a.act = b_act.as<int>();
  a.v_next_full = b_vnext.as<double>();
  rc = launch_qn_solve(c, a, 0);
  if (rc) return rc;
  }
  if (in(3)) {
  mark(5);
  k_reactions<<<kReactCtas, kReactThreads, 0, c.stream>>>(
      counters, b_gamma.as<double>(), ca.frames, ca.witness, ca.body, b_geoms.as<mpmrb_geom>(),
      ngeom, nbody, nc_cap, b_gworld.as<double>(), b_react.as<double>());
  k_substep_end<<<1, 256, 0, c.stream>>>(counters, b_solveout.as<SolveOut>(),
                                       b_react.as<double>(), nbody, b_accum.as<double>(),
                                       counters + 3, b_stats.as<SubstepStat>(), max_substeps,
                                       c.status);
  c.launches += 2;
  mark(6);
  // 6. G2P (mpm.py:118-138)
  rc = (prec == MPMRB_PREC_F32)
           ? launch_g2p(c, g, q32, b_mats.as<mpmrb_material>(), nmat, b_vnext.as<double>(), dt_s,
                        b_misc.as<unsigned long long>(), b_misc.as<int>() + 2)
           : launch_g2p(c, g, q, b_mats.as<mpmrb_material>(), nmat, b_vnext.as<double>(), dt_s,
                        b_misc.as<unsigned long long>(), b_misc.as<int>() + 2);
  if (rc) return rc;
  if (cloth.ne > 0) {  // d3 advection, return map, element particles to centroids
    rc = (prec == MPMRB_PREC_F32)
             ? launch_cloth_post(c, cloth, q32, b_mats.as<mpmrb_material>(), nmat, dt_s)
             : launch_cloth_post(c, cloth, q, b_mats.as<mpmrb_material>(), nmat, dt_s);
    if (rc) return rc;
  }
  mark(7);
  }
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

// Stage boundaries: CUDA events for bench.py's live per-stage timing (direct
// launches), and NVTX ranges named after the pipeline stages (nsys / ncu
// --nvtx; while a graph is captured they bracket the capture).
void Sim::mark(int k) {
  static const char* kStage[kProfEvents - 1] = {"mpmrb grid build", "mpmrb P2G",
                                                "mpmrb grid update", "mpmrb contacts",
                                                "mpmrb contact solve", "mpmrb reactions",
                                                "mpmrb G2P"};
  if (prof_on) cudaEventRecord(prof_ev[k], ctx->stream);
  if (k > 0) nvtxRangePop();
  if (k < kProfEvents - 1) nvtxRangePushA(kStage[k]);
}

// One substep with direct launches and events between the pipeline stages
// (bench.py's live per-kernel timing; graph replays cannot be bracketed).
int Sim::profile_substep(float* stage_ms, int* sizes) {
  Ctx& c = *ctx;
  if (!prof_ev[0])
    for (int k = 0; k < kProfEvents; ++k) MPMRB_CUDA_OK(cudaEventCreate(&prof_ev[k]));
  prof_on = true;
  int rc = capture_or_launch();
  prof_on = false;
  if (rc) return rc;
  MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
  for (int k = 0; k + 1 < kProfEvents; ++k)
    MPMRB_CUDA_OK(cudaEventElapsedTime(&stage_ms[k], prof_ev[k], prof_ev[k + 1]));
  int hc[4] = {0, 0, 0, 0};
  MPMRB_CUDA_OK(cudaMemcpy(hc, b_counters.p, sizeof(hc), cudaMemcpyDeviceToHost));
  sizes[0] = hc[0];
  sizes[1] = hc[1];
  sizes[2] = hc[2];
  SolveOut so{};
  MPMRB_CUDA_OK(cudaMemcpy(&so, b_solveout.p, sizeof(so), cudaMemcpyDeviceToHost));
  sizes[3] = so.iterations;
  sizes[4] = so.ls_evals;
  return MPMRB_OK;
}

int Sim::begin_step(long long epoch, int n_substeps) {
  NvtxRange r("mpmrb begin_step");
  Ctx& c = *ctx;
  if (!have_particles) return set_error(MPMRB_E_INVALID, "sim: particles not set");
  if (!have_params) return set_error(MPMRB_E_INVALID, "sim: params not set");
  // size the grid for the current positions (one host sync per step)
  if (b_counters.grow(64) || b_misc.grow(64) || b_solveout.grow(sizeof(SolveOut)) ||
      b_bar.grow(4096) || b_partials.grow(sizeof(double) * (2 * 8 * kMaxSolverCtas + 8)) ||
      b_dyn.grow(64) || b_accum.grow(sizeof(double) * 6 * kMaxBodies) ||
      b_react.grow(sizeof(double) * 6 * kMaxBodies * kReactCtas) ||
      b_slots.grow(kSolverSyncBytes))
    return MPMRB_E_CUDA;
  if (!slots_init) {
    // slot tags start at 0 and channel tags at 1, so no stale slot matches
    MPMRB_CUDA_OK(cudaMemsetAsync(b_slots.p, 0, kSolverSyncBytes, c.stream));
    unsigned ch[4] = {1u, 1u, 1u, 0u};
    MPMRB_CUDA_OK(cudaMemcpyAsync(b_slots.as<char>() + 8 * kSolverSlotWords, ch, sizeof(ch),
                                  cudaMemcpyHostToDevice, c.stream));
    MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
    slots_init = true;
  }
  if (!bar_init) {
    MPMRB_CUDA_OK(cudaMemsetAsync(b_bar.p, 0, 64, c.stream));
    bar_init = true;
  }
  long long nb_probe_cap = nb_cap > 0 ? nb_cap : 1024;
  long long probe_hcap = 0;
  int nb_probe = 0;
  for (int attempt = 0; attempt < 8; ++attempt) {
    long long hcap = next_pow2(4 * nb_probe_cap);
    probe_hcap = hcap;
    if (b_probe_hk.grow(8 * hcap) || b_probe_hv.grow(4 * hcap) || b_probe_uk.grow(8 * nb_probe_cap) ||
        b_probe_bk.grow(8 * nb_probe_cap))
      return MPMRB_E_CUDA;
    // particle health first (coupling.py:171 checks before the plan)
    MPMRB_CUDA_OK(cudaMemsetAsync(b_counters.as<int>() + 8, 0, 4, c.stream));
    int rc = launch_health(c, p.x, p.v, p.n, h, b_counters.as<int>() + 8);
    if (rc) return rc;
    int hbad[9] = {0};
    MPMRB_CUDA_OK(cudaMemcpyAsync(hbad, b_counters.p, sizeof(hbad), cudaMemcpyDeviceToHost,
                                  c.stream));
    MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
    if (hbad[8])
      return set_error(MPMRB_E_DIVERGED, "non-finite or out-of-range particle state");
    rc = launch_grid_build(c, p.x, p.n, h, b_probe_bk.as<long long>(), nb_probe_cap,
                           b_probe_hk.as<unsigned long long>(), b_probe_hv.as<int>(), hcap,
                           b_probe_uk.as<long long>(), b_counters.as<int>());
    if (rc) return rc;
    int nb_host = 0;
    MPMRB_CUDA_OK(cudaMemcpyAsync(&nb_host, b_counters.p, sizeof(int), cudaMemcpyDeviceToHost,
                                  c.stream));
    MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
    int st = c.check_status("sim_begin_step");
    if (st == MPMRB_E_CAPACITY) {
      nb_probe_cap = (long long)nb_host * 2 + 64;
      continue;
    }
    if (st) return st;
    int rc2 = reserve(p.n, nb_host);
    if (rc2) return rc2;
    nb_probe = nb_host;
    break;
  }
  if (b_tauvalid.p) MPMRB_CUDA_OK(cudaMemsetAsync(b_tauvalid.p, 0, sizeof(int), c.stream));
  // sim-internal particle order for this step: sorted by (block, cell) of the
  // step-start positions, gathered from the user's arrays (scattered back in
  // end_step)
  if (p.n > 0) {
    int rc = launch_particle_sort(c, p.x, p.n, h, b_probe_hk.as<unsigned long long>(),
                                  b_probe_hv.as<int>(), probe_hcap, nb_probe > 0 ? nb_probe : 1,
                                  b_skeys.as<unsigned>(), b_svals.as<int>(), b_perm.as<int>());
    if (rc) return rc;
    const int* perm = b_perm.as<int>();
    rc = launch_particle_gather(c, perm, p.n, p.x, 3, q.x);
    if (prec == MPMRB_PREC_F32) {
      if (!rc) rc = launch_particle_gather_f32(c, perm, p.n, p.v, 3, q32.v);
      if (!rc) rc = launch_particle_gather_f32(c, perm, p.n, p.f, 9, q32.f);
      if (!rc) rc = launch_particle_gather_f32(c, perm, p.n, p.c, 9, q32.c);
      if (!rc) rc = launch_particle_gather_f32(c, perm, p.n, p.mass, 1, const_cast<float*>(q32.mass));
      if (!rc) rc = launch_particle_gather_f32(c, perm, p.n, p.vol0, 1, const_cast<float*>(q32.vol0));
      if (!rc) {
        if (p.plastic) rc = launch_particle_gather_f32(c, perm, p.n, p.plastic, 1, q32.plastic);
        else MPMRB_CUDA_OK(cudaMemsetAsync(q32.plastic, 0, 4 * p.n, c.stream));
      }
    } else {
      if (!rc) rc = launch_particle_gather(c, perm, p.n, p.v, 3, q.v);
      if (!rc) rc = launch_particle_gather(c, perm, p.n, p.f, 9, q.f);
      if (!rc) rc = launch_particle_gather(c, perm, p.n, p.c, 9, q.c);
      if (!rc) rc = launch_particle_gather(c, perm, p.n, p.mass, 1, const_cast<double*>(q.mass));
      if (!rc) rc = launch_particle_gather(c, perm, p.n, p.vol0, 1, const_cast<double*>(q.vol0));
      if (!rc) {
        if (p.plastic) rc = launch_particle_gather(c, perm, p.n, p.plastic, 1, q.plastic);
        else MPMRB_CUDA_OK(cudaMemsetAsync(q.plastic, 0, 8 * p.n, c.stream));
      }
    }
    if (!rc) rc = launch_gather_i64(c, perm, p.n, p.mid, const_cast<long long*>(q.mid));
    if (rc) return rc;
    if (cloth.ne > 0) {
      if (b_invperm.grow(4 * p.n) || b_qrole.grow(p.n) || b_qtau.grow(8 * 9 * p.n) ||
          b_qfext.grow(8 * 3 * p.n))
        return MPMRB_E_CUDA;
      if (q.role != b_qrole.as<signed char>() || q.tau != b_qtau.as<double>() ||
          q.fext != b_qfext.as<double>()) {
        q.role = b_qrole.as<signed char>();
        q.tau = b_qtau.as<double>();
        q.fext = b_qfext.as<double>();
        invalidate();
      }
      if (cloth.inv_perm != b_invperm.as<int>()) {
        cloth.inv_perm = b_invperm.as<int>();
        invalidate();
      }
      rc = launch_inverse_perm(c, perm, p.n, b_invperm.as<int>());
      if (!rc) rc = launch_gather_i8(c, cloth_role_user, perm, p.n, b_qrole.as<signed char>());
      if (rc) return rc;
      MPMRB_CUDA_OK(cudaMemsetAsync(q.tau, 0, 8 * 9 * p.n, c.stream));
    } else if (q.role) {
      q.role = nullptr;
      q.tau = nullptr;
      q.fext = nullptr;
      invalidate();
    }
    // the fp32 layout shares the cloth roles, element stresses and vertex
    // forces (float64) with the float64 one
    if (q32.role != q.role || q32.tau != q.tau || q32.fext != q.fext) {
      q32.role = q.role;
      q32.tau = q.tau;
      q32.fext = q.fext;
      invalidate();
    }
  }
  if (max_substeps < n_substeps || !b_stats.p) {
    max_substeps = n_substeps > max_substeps ? n_substeps : max_substeps;
    if (b_stats.grow(sizeof(SubstepStat) * (max_substeps + 1))) return MPMRB_E_CUDA;
    if (graph_exec) {
      cudaGraphExecDestroy(graph_exec);
      graph_exec = nullptr;
    }
  }
  steps_substeps = n_substeps;
  // per-step resets: accumulator, counters, bias-cache epoch (coupling.py:175-176)
  // bias-cache stamp: a private per-step counter (never the user's epoch, so
  // restarting a scene from step 0 cannot resurrect stale first-sight biases)
  (void)epoch;
  int dyn[2] = {++bias_stamp_counter, 0};
  MPMRB_CUDA_OK(cudaMemcpyAsync(b_dyn.p, dyn, sizeof(dyn), cudaMemcpyHostToDevice, c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(b_accum.p, 0, b_accum.bytes, c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(b_misc.p, 0, 64, c.stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(b_counters.p, 0, 64, c.stream));
  // Morton keys at step start for plan staleness (coupling.py:173, 212)
  if (b_plankeys.grow(2 * (p.n + 1))) return MPMRB_E_CUDA;
  if (p.n > 0) {
    long long* dummy_perm = nullptr;
    (void)dummy_perm;
    int rc = launch_morton_only(c, p.x, p.n, h, b_plankeys.as<uint16_t>());
    if (rc) return rc;
  }
  // bias-cache slots of this step are stamped with epoch+1; memcpy above is
  // ordered before every substep on the stream.
  // MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
  return MPMRB_OK;
}

int Sim::substep() {
  Ctx& c = *ctx;
  if (!use_graph || c.stream == nullptr) return capture_or_launch();
  if (!graph_exec) {
    cudaGraph_t graph = nullptr;
    long long before = c.launches;
    MPMRB_CUDA_OK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
    int rc = capture_or_launch();
    cudaError_t e = cudaStreamEndCapture(c.stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      use_graph = false;  // capture unsupported: direct launches
      c.launches = before;
      return capture_or_launch();
    }
    kernels_per_substep = c.launches - before;
    c.launches = before;
    e = cudaGraphInstantiate(&graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      cudaGetLastError();
      graph_exec = nullptr;
      use_graph = false;
      return capture_or_launch();
    }
  }
  NvtxRange r("mpmrb substep (graph)");
  MPMRB_CUDA_OK(cudaGraphLaunch(graph_exec, c.stream));
  c.launches += kernels_per_substep;
  return MPMRB_OK;
}

int Sim::substep_part(int part) {
  if (part < 0 || part > 3) return set_error(MPMRB_E_INVALID, "substep part must be 0..3");
  NvtxRange r("mpmrb substep part");
  return capture_or_launch(part, part);
}

int Sim::set_solve_result(int converged, int iterations, int ls_evals, int regularized) {
  k_set_solveout<<<1, 32, 0, ctx->stream>>>(b_solveout.as<SolveOut>(), converged, iterations,
                                            ls_evals, regularized);
  ctx->launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int Sim::end_step(mpmrb_step_stats* out, double* impulses_host) {
  NvtxRange r("mpmrb end_step");
  Ctx& c = *ctx;
  std::vector<SubstepStat> st(steps_substeps > 0 ? steps_substeps : 1);
  unsigned long long misc[4] = {0, 0, 0, 0};
  if (steps_substeps > 0)
    MPMRB_CUDA_OK(cudaMemcpyAsync(st.data(), b_stats.p, sizeof(SubstepStat) * steps_substeps,
                                  cudaMemcpyDeviceToHost, c.stream));
  MPMRB_CUDA_OK(cudaMemcpyAsync(misc, b_misc.p, sizeof(misc), cudaMemcpyDeviceToHost, c.stream));
  double acc[6 * kMaxBodies];
  MPMRB_CUDA_OK(cudaMemcpyAsync(acc, b_accum.p, sizeof(double) * 6 * kMaxBodies,
                                cudaMemcpyDeviceToHost, c.stream));
  unsigned long long changed = 0;
  if (p.n > 0) {
    // internal order -> the user's arrays (reference order)
    const int* perm = b_perm.as<int>();
    int rc = launch_particle_scatter(c, perm, p.n, q.x, 3, p.x);
    if (prec == MPMRB_PREC_F32) {
      if (!rc) rc = launch_particle_scatter_f32(c, perm, p.n, q32.v, 3, p.v);
      if (!rc) rc = launch_particle_scatter_f32(c, perm, p.n, q32.f, 9, p.f);
      if (!rc) rc = launch_particle_scatter_f32(c, perm, p.n, q32.c, 9, p.c);
      if (!rc && p.plastic)
        rc = launch_particle_scatter_f32(c, perm, p.n, q32.plastic, 1, p.plastic);
    } else {
      if (!rc) rc = launch_particle_scatter(c, perm, p.n, q.v, 3, p.v);
      if (!rc) rc = launch_particle_scatter(c, perm, p.n, q.f, 9, p.f);
      if (!rc) rc = launch_particle_scatter(c, perm, p.n, q.c, 9, p.c);
      if (!rc && p.plastic) rc = launch_particle_scatter(c, perm, p.n, q.plastic, 1, p.plastic);
    }
    if (rc) return rc;
  }
  if (p.n > 0) {
    int rc = launch_staleness(c, b_plankeys.as<uint16_t>(), p.x, p.n, h,
                              b_misc.as<unsigned long long>() + 4);
    if (rc) return rc;
    MPMRB_CUDA_OK(cudaMemcpyAsync(&changed, b_misc.as<unsigned long long>() + 4, 8,
                                  cudaMemcpyDeviceToHost, c.stream));
  }
  MPMRB_CUDA_OK(cudaStreamSynchronize(c.stream));
  // device status (first error of the step)
  DevStatus ds{};
  MPMRB_CUDA_OK(cudaMemcpy(&ds, c.status, sizeof(DevStatus), cudaMemcpyDeviceToHost));
  MPMRB_CUDA_OK(cudaMemset(c.status, 0, sizeof(DevStatus)));
  std::memset(out, 0, sizeof(*out));
  out->substeps = steps_substeps;
  out->all_converged = 1;
  long long it_sum = 0, nc_sum = 0, act_sum = 0;
  for (int k = 0; k < steps_substeps; ++k) {
    const SubstepStat& s = st[k];
    int conv = (s.nc == 0) ? 1 : s.converged;
    out->all_converged &= conv ? 1 : 0;
    if (!conv) {
      out->substeps_unconverged += 1;
      out->iterations_unconverged += s.iters;
    }
    it_sum += s.iters;
    nc_sum += s.nc;
    act_sum += s.n_act;
    if (s.iters > out->iterations_max) out->iterations_max = s.iters;
    if (s.nc > out->n_contacts_max) out->n_contacts_max = s.nc;
    out->ls_evals += s.ls_evals;
    out->regularized += s.regularized;
  }
  out->iterations_total = it_sum;
  if (steps_substeps > 0) {
    out->iterations_mean = (double)it_sum / steps_substeps;
    out->n_contacts_mean = (double)nc_sum / steps_substeps;
    out->n_active_mean = (double)act_sum / steps_substeps;
  }
  out->clamped = (long long)misc[0];
  int health = (int)(misc[1] & 0xffffffffu);
  out->status = ds.code;
  out->status_detail = ds.detail;
  out->status_aux = ds.aux;
  if (!out->status && health) out->status = MPMRB_E_DIVERGED;
  staleness = p.n > 0 ? (double)changed / (double)p.n : 0.0;
  if (impulses_host) std::memcpy(impulses_host, acc, sizeof(double) * 6 * (nbody < kMaxBodies ? nbody : kMaxBodies));
  return MPMRB_OK;
}

Sim::~Sim() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  for (int k = 0; k < kProfEvents; ++k)
    if (prof_ev[k]) cudaEventDestroy(prof_ev[k]);
}

}  // namespace mpmrb
