// Arguments of the persistent quasi-Newton solve kernel (solver.cu).
#pragma once

#include "internal.h"

namespace mpmrb {

constexpr int kSolverThreads = 512;
constexpr int kMaxSolverCtas = 160;
constexpr int kSolverCluster = 8;  // CTAs of the contact-owning cluster
constexpr int kSolverProf = 16;  // phase timers (ns), see solver.cu

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

// Node -> (contact, slot) adjacency of one solve (built by
// launch_solver_adjacency from the contact stencils).
struct SolverAdjacency {
  int* cnt;      // (nd_cap+1) scratch
  int* fill;     // (nd_cap+1) scratch
  int* off;      // (nd_cap+1) CSR offsets
  int* ent;      // (27 nc_cap) packed (c << 5) | k, ascending within a node
  int* ent_tmp;  // (27 nc_cap) scratch: entries in atomic fill order
  double* w;     // (27 nc_cap) stencil weight of each entry
  int* flag;     // (nd_cap+1) scratch: node has 1..kHeavy entries
  int* flag_off; // (nd_cap+1) scan of flag
  int* hflag;    // (nd_cap+1) scratch: node has > kHeavy entries
  int* hflag_off;// (nd_cap+1) scan of hflag
  int* cn;       // (nd_cap) light contact nodes (8-lane groups)
  int* cn_e;     // (2 nd_cap) CSR bounds of each light contact node
  int* hn;       // (nd_cap) heavy contact nodes (one warp each)
  int* hn_e;     // (2 nd_cap) CSR bounds of each heavy contact node
  int* fn;       // (nd_cap) nodes without entries
  int* n_cn;     // device count of light contact nodes
  int* n_hn;     // device count of heavy contact nodes
};

constexpr int kHeavyNode = 64;  // entries above which a node gets a whole warp

struct SolverArgs {
  // sizes (device)
  const int* nd_dev;
  const int* nc_dev;
  long long nc_cap;
  long long nd_cap;
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
  SolverAdjacency adj;
  // solver parameters (solver.py:35-49)
  double eps_a, eps_r, ls_tol;
  int max_iters, ls_max;
  int skip_if_no_contacts;
  int force_ctas;  // 0 = automatic
  // work (device)
  double* v;
  double* dv;
  double* vc;
  double* dvc;
  double* gw;        // (nc,3) R^T g_c
  double* rgr;       // (nc,6) R^T G R (00,11,22,10,20,21)
  double* cvhat;     // (nc,) -phi/(dt+tau_d), per solve
  double* cmug;      // (nc,) mu*gamma_lag, per solve
  double* partials;  // 2 x [kMaxRed][kMaxSolverCtas]
  double* ls_out;    // (2,) line-search step and status published by the contact group
  // outputs
  double* gamma;
  double* tr_obj;
  double* tr_res;
  double* tr_thr;
  double* tr_alpha;
  SolveOut* out;
  unsigned long long* prof;  // optional [kSolverProf] phase times (ns)
  // fused epilogue: scatter v into the full grid
  const int* act;
  double* v_next_full;
};

// Build the adjacency from cnodes/cw (w != 0 slots only).
int launch_solver_adjacency(Ctx& c, const int* nd_dev, const int* nc_dev, long long nd_cap,
                            long long nc_cap, const int* cnodes, const double* cw,
                            const SolverAdjacency& adj, DevBuf& tiles);
int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas);

}  // namespace mpmrb
