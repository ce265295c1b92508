// Arguments of the persistent quasi-Newton solve kernel (solver.cu).
#pragma once

#include "internal.h"

namespace mpmrb {

constexpr int kSolverThreads = 512;
constexpr int kMaxSolverCtas = 160;

struct SolveOut {
  int converged;
  int iterations;
  int ls_evals;
  int regularized;
  int status;
  int status_flags;  // bit 0: non-finite solution
  int n_contacts;
  int n_dofs;
};

struct SolverArgs {
  // sizes (device)
  const int* nd_dev;
  const int* nc_dev;
  long long nc_cap;
  // problem on active nodes (solver.py:75-110)
  const double* m;
  const double* v_star;
  const double* v0;
  const int* cnodes;   // [27][nc_cap]
  const double* cw;    // [27][nc_cap]
  const double* frames;
  const double* bias;
  const double* phi;
  const double* mu;
  const double* gamma_lag;
  double K, den, eps_v;
  // solver parameters (solver.py:35-49)
  double eps_a, eps_r, ls_tol;
  int max_iters, ls_max;
  int skip_if_no_contacts;
  int force_ctas;  // 0 = automatic
  // work (device)
  double* v;
  double* g;
  double* jt;
  double* H6;
  double* dv;
  double* vc;
  double* dvc;
  double* partials;  // [kMaxRed][kMaxSolverCtas]
  unsigned* bar;     // 2 words, zero-initialised once
  // outputs
  double* gamma;
  double* tr_obj;
  double* tr_res;
  double* tr_thr;
  double* tr_alpha;
  SolveOut* out;
  // fused epilogue: scatter v into the full grid
  const int* act;
  double* v_next_full;
};

int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas);

}  // namespace mpmrb
