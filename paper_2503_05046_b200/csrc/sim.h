// Fused-substep simulation context (host side).
#pragma once

#include <cuda_runtime.h>

#include "internal.h"

namespace mpmrb {

int launch_morton_only(Ctx& c, const double* x, long long n, double h, uint16_t* keys);

struct Sim {
  Ctx* ctx = nullptr;
  ParticlesDev p{};  // user arrays (reference order)
  ParticlesDev q{};  // sim-internal copy sorted by (block, cell), used by the substeps
  ParticlesF32 q32{};  // its float32 layout (fp32 performance mode; x is q.x)
  int prec = MPMRB_PREC_F64;
  bool have_particles = false;
  bool have_params = false;
  int nmat = 0;
  int ngeom = 0;
  int nbody = 0;
  double h = 0.0, dt_s = 0.0, gravity[3] = {0.0, 0.0, 0.0};
  double K = 0.0, den = 1.0, eps_v = 1e-4, margin = 0.0;
  mpmrb_solver_params sp{};
  int force_ctas = 0;
  int force_ls_ctas = 0;
  long long nb_cap = 0, hash_cap = 0, nc_cap = 0, n_particles = -1;
  long long bias_n = -1;
  int bias_geoms = -1;
  int max_substeps = 0;
  int steps_substeps = 0;
  int bias_stamp_counter = 0;
  double staleness = 0.0;
  bool use_graph = true;
  bool bar_init = false;
  cudaGraphExec_t graph_exec = nullptr;
  long long kernels_per_substep = 0;

  DevBuf b_mats, b_geoms, b_counters, b_misc, b_solveout, b_bar, b_partials, b_dyn, b_accum;
  DevBuf b_probe_hk, b_probe_hv, b_probe_uk, b_probe_bk, b_plankeys, b_stats;
  DevBuf b_hkeys, b_hvals, b_ukeys, b_bkeys;
  DevBuf b_mass, b_mom, b_vk, b_vstar, b_vnext, b_active, b_wcount, b_woff, b_act, b_remap;
  DevBuf b_mc, b_vstarc, b_vkc;
  DevBuf b_cnt, b_offs, b_cpart, b_cbody, b_cphi, b_cmu, b_cgl, b_cnormal, b_cwit, b_cbias,
      b_cframes, b_cnodes, b_cw;
  DevBuf b_sv, b_sdv, b_svc, b_sdvc, b_gamma, b_gworld, b_tiles;
  // solver setup (groups + node adjacency), cellsum, reduction slots
  DevBuf b_su_c, b_su_n, b_su_ent, b_cellsum, b_slots;
  // sorted particle state: x, v (3n) f, c (9n) mass, vol0, plastic (n) doubles; mid (n) int64
  DevBuf b_qd, b_qmid, b_perm, b_skeys, b_svals, b_cpart_user;
  DevBuf b_qf;  // float32 particle state (fp32 mode): v 3n, f 9n, c 9n, mass, vol0, plastic n, tau 6n
  DevBuf b_react;  // per-CTA reaction partials
  // codimensional cloth (cloth.cu): mesh in user order + per-step internal views
  ClothDev cloth{};
  const signed char* cloth_role_user = nullptr;
  DevBuf b_invperm, b_qrole, b_qtau, b_qfext;
  DevBuf b_taucache, b_tauvalid;  // sand: Hencky stress cached by G2P for P2G
  bool slots_init = false;
  DevBuf b_bias_stamp, b_bias_store;

  static constexpr int kProfEvents = 8;
  cudaEvent_t prof_ev[kProfEvents] = {};
  bool prof_on = false;
  void mark(int k);
  int profile_substep(float* stage_ms, int* sizes);
  int reserve(long long n, long long nb_needed);
  int capture_or_launch(int part_lo = 0, int part_hi = 3);
  int substep_part(int part);
  int set_solve_result(int converged, int iterations, int ls_evals, int regularized);
  int begin_step(long long epoch, int n_substeps);
  int substep();
  int end_step(mpmrb_step_stats* out, double* impulses_host);
  void invalidate() {
    if (graph_exec) {
      cudaGraphExecDestroy(graph_exec);
      graph_exec = nullptr;
    }
  }
  ~Sim();
};

}  // namespace mpmrb
