// Arguments of the persistent quasi-Newton solve kernel (solver.cu).
#pragma once

#include "internal.h"

namespace mpmrb {

constexpr int kSolverThreads = 256;
constexpr int kMaxSolverCtas = 160;
constexpr int kSolverProf = 16;  // phase timers (ns), see solver.cu
// + per-CTA work time (ns) of the N, D and U phases: [16 + phase*kMaxSolverCtas + cta]
constexpr int kSolverProfWords = 16 + 5 * 160;
constexpr int kCellSumStride = 10;  // per-contact record: R^T g (3), R^T G R (6), padded to 80 B

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

// Per-solve structure built by launch_solver_setup from the contact stencils.
//
// Contact groups: maximal runs of consecutive contacts with identical stencil
// node lists (the contacts of one grid cell share all 27 nodes); they make
// the node adjacency cheap to build.  Each contact owner writes one record per
// iteration (R^T g, R^T G R); each contact node gathers, through a node ->
// (contact, slot) CSR sorted by contact, the records weighted by the slot
// weight: a fixed summation order (ascending contact id per node), no atomics.
struct SolverSetup {
  int* head;       // (nc_cap+1) scratch: contact starts a group
  int* head_off;   // (nc_cap+1) exclusive scan of head
  int* grp_of;     // (nc_cap) group of each contact
  int* grp_start;  // (nc_cap+1) first contact of each group, [ng] = nc
  int* cnt;        // (nd_cap+1) scratch: entries per node
  int* fill;       // (nd_cap+1) scratch
  int* off;        // (nd_cap+1) CSR offsets
  int* cnt_exp;    // (nd_cap+1) scratch: contacts per node
  int* off_exp;    // (nd_cap+1) CSR offsets of the expanded entries
  int* ent_tmp;    // (27 nc_cap) scratch: (run, slot) entries in atomic fill order
  int* ent;        // (27 nc_cap) (contact << 5 | slot), ascending contact within a node
  int* flag;       // (nd_cap+1) scratch: node has entries
  int* flag_off;   // (nd_cap+1) exclusive scan of flag
  int* cn;         // (nd_cap) contact nodes (ascending)
  int* fn;         // (nd_cap) free nodes (ascending)
  int4* cn_rec;    // (nd_cap) per contact node: (node, expanded CSR begin, end, 0)
  int* counts;     // device [0] n_groups, [1] n_contact_nodes
};

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
  const int* cnodes;   // [27][nc_cap], -1 on dead (w = 0) slots
  const double* cw;    // [27][nc_cap]
  const double* frames;
  const double* bias;
  const double* phi;
  const double* mu;
  const double* gamma_lag;
  double K, den, eps_v;
  SolverSetup su;
  // solver parameters (solver.py:35-49)
  double eps_a, eps_r, ls_tol;
  int max_iters, ls_max;
  int skip_if_no_contacts;
  int force_ctas;  // 0 = automatic
  int force_ls_ctas;  // 0 = automatic
  // free nodes held outside this problem (slab decomposition, slab.py): their
  // sums S0 = sum m |v0 - v*|^2, Q0 = sum m |v*|^2, Q1 = sum m v*.(v0 - v*),
  // added to the problem's own; the final P = prod(1 - alpha) goes to p_out
  double ext_free[3];
  double* p_out;      // device, optional
  // work (device)
  double* v;         // (nd,3) solution (contact nodes during the solve, all at the end)
  double* dv;        // (nd,3)
  double* vc;        // (nc,3) contact velocities
  double* dvc;       // (nc,3)
  double* cvhat;     // (nc,) -phi/(dt+tau_d)
  double* cmug;      // (nc,) mu*gamma_lag
  double* cellsum;   // (nc_cap, kCellSumStride) per-contact records
  double* partials;  // [2][8][kMaxSolverCtas] grid reductions
  unsigned long long* slots;  // self-validating reduction slots (see solver.cu)
  unsigned* chan;    // [4] channel tags carried across solves ([3]: barrier generation)
  unsigned* bar;     // grid barrier words: [0] count, [32] generation (zeroed once)
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

// words of the self-validating slot area (solver.cu)
constexpr long long kSolverSlotWords = 2LL * kMaxSolverCtas * 6 + 2LL * kMaxSolverCtas * 4 + 2 * 4 + 2 * 4;
// the slot buffer is followed by chan[4] (64 B) and the barrier words (256 B)
constexpr long long kSolverSyncBytes = 8 * kSolverSlotWords + 64 + 256;

// Build groups + node adjacency from cnodes/cw.
int launch_solver_setup(Ctx& c, const int* nd_dev, const int* nc_dev, long long nd_cap,
                        long long nc_cap, const int* cnodes, const SolverSetup& su,
                        DevBuf& tiles);
int launch_qn_solve(Ctx& c, const SolverArgs& a, int grid_ctas);
// solver.py:224-256 (reg[2] device: regularised blocks, blocks still not SPD)
int launch_search_direction(Ctx& c, const double* h, const double* g, long long n, double* d,
                            int* reg);

}  // namespace mpmrb
