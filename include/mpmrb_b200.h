/*
 * mpmrb_b200 — C ABI of the B200-native (sm_100a) MPM–rigid coupling substep.
 *
 * Drop-in boundary for the hot path of the reference package `mpmrb`
 * (/root/reference/pkg/src/mpmrb).  The reference has no FFI of its own; its
 * boundary is the Python API listed in SURVEY.md §8(b).  Each entry point
 * below names the reference function it replaces (file:line).  The Python
 * package `paper_2503_05046_b200` binds these with ctypes (see INTEGRATION.md
 * for the binding a maintainer of the reference would add).
 *
 * Conventions
 *  - every array argument is a DEVICE pointer (cudaMalloc'd / torch CUDA
 *    tensor storage) unless the name ends in `_host`;
 *  - float64 everywhere the reference uses float64 (all physics), int64 where
 *    the reference returns int64 indices, uint16 for Morton keys;
 *  - (n,3) and (n,3,3) arrays are row-major and contiguous, exactly the
 *    layout of the reference's NumPy arrays;
 *  - calls are asynchronous on the context's stream unless documented as
 *    returning a host-visible count (those synchronise the stream);
 *  - return value: MPMRB_OK or an error code; `mpmrb_last_error()` gives the
 *    message.  Error codes map one-to-one onto the reference's exceptions.
 */
#ifndef MPMRB_B200_H
#define MPMRB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPMRB_ABI_VERSION 2

/* error codes -> reference exceptions */
enum {
  MPMRB_OK = 0,
  MPMRB_E_ALLOCATION = 1,   /* grid.AllocationError        grid.py:22,29-30,78,119-120 */
  MPMRB_E_PLAN_EPOCH = 2,   /* transfer.PlanEpochError     transfer.py:40,159-160       */
  MPMRB_E_INVALID = 3,      /* ValueError (shape/mode/range) transfer.py:58-59,161-170  */
  MPMRB_E_NOT_DESCENT = 4,  /* line-search ValueError      solver.py:274-275            */
  MPMRB_E_NONFINITE = 5,    /* FloatingPointError          solver.py:243,364            */
  MPMRB_E_DIVERGED = 6,     /* coupling.SimulationDiverged coupling.py:158-165          */
  MPMRB_E_CUDA = 7,         /* (new) CUDA runtime failure                                */
  MPMRB_E_CAPACITY = 8      /* (new) preallocated capacity too small; retry larger       */
};

/* material models */
enum { MPMRB_MAT_ELASTIC = 0, /* fixed corotated, materials.py:113-122 */
       MPMRB_MAT_SAND = 1,    /* Drucker–Prager (new; parity unpinned)  */
       MPMRB_MAT_CLOTH = 2 }; /* codimensional cloth, Jiang et al. 2017 (new; parity unpinned) */

/* per-particle cloth roles (mpmrb_sim_set_cloth) */
enum { MPMRB_CLOTH_NONE = 0, MPMRB_CLOTH_VERTEX = 1, MPMRB_CLOTH_ELEMENT = 2 };

/* geometry primitives (geometry.py) */
enum { MPMRB_GEOM_HALFSPACE = 0, MPMRB_GEOM_SPHERE = 1, MPMRB_GEOM_BOX = 2,
       MPMRB_GEOM_CAPSULE = 3 };

typedef struct mpmrb_ctx mpmrb_ctx;

/* A material table entry (materials.py:24-46 plus the sand extension). */
typedef struct {
  int32_t kind;          /* MPMRB_MAT_* */
  int32_t pad_;
  double mu, lam;        /* Lame parameters (materials.py:40-46) */
  double dp_alpha;       /* Drucker–Prager alpha for sand, else 0 */
  double k_normal;       /* cloth: transverse compression stiffness */
  double gamma_shear;    /* cloth: transverse shear stiffness */
  double friction;       /* cloth: cloth-cloth friction coefficient */
} mpmrb_material;

/* One rigid geometry in WORLD pose, flattened in (body, geom) order
 * (collision.py:98-104).  `rot` is R_geom = R_body @ R(geom.quat), row-major;
 * `pos` is the geom origin in world.  params: halfspace (nx,ny,nz,offset),
 * sphere (r), box (hx,hy,hz), capsule (r, half_length). */
typedef struct {
  int32_t kind;          /* MPMRB_GEOM_* */
  int32_t body;          /* body index */
  int32_t geom;          /* geom index within the body */
  int32_t pad_;
  double rot[9];
  double pos[3];
  double params[4];
  double mu;             /* friction vs particles (bodies.py:25) */
  double body_pos[3];    /* body.position (arm origin, collision.py:114) */
  double body_v[3];      /* body.v */
  double body_omega[3];  /* body.omega */
} mpmrb_geom;

/* Particle state views (particles.py:12-64), all length n. */
typedef struct {
  double* x;       /* (n,3) */
  double* v;       /* (n,3) */
  double* f;       /* (n,3,3) */
  double* c;       /* (n,3,3) */
  const double* mass;     /* (n,) */
  const double* volume0;  /* (n,) */
  const int64_t* material_id;  /* (n,) */
  double* plastic;  /* (n,) accumulated plastic strain (sand), may be NULL */
  int64_t n;
} mpmrb_particles;

/* Block-sparse grid lookup structure produced by mpmrb_grid_allocate. */
typedef struct {
  const int64_t* block_keys;      /* (nb,) sorted packed keys (grid.py:42) */
  const uint64_t* hash_keys;      /* (hash_cap,) open-addressing slots */
  const int32_t* hash_vals;       /* (hash_cap,) block index per slot */
  int64_t n_blocks;
  int64_t hash_cap;               /* power of two */
  double h;
} mpmrb_grid_view;

/* Contact problem restricted to active nodes (solver.py:75-110). */
typedef struct {
  int64_t n_nodes;      /* active nodes nd */
  int64_t n_contacts;   /* nc */
  const double* m;      /* (nd,) */
  const double* v_star; /* (nd,3) */
  const double* v_init; /* (nd,3) */
  const int64_t* nodes; /* (nc,27) restricted indices, dead slots -> 0 */
  const double* w;      /* (nc,27), 0 on dead slots */
  const double* frames; /* (nc,3,3) */
  const double* bias;   /* (nc,3) */
  const double* phi;    /* (nc,) */
  const double* mu;     /* (nc,) */
  const double* gamma_lag; /* (nc,) */
  double stiffness, tau_d, eps_v, dt;  /* contact_model.py:26-39 */
} mpmrb_problem;

typedef struct {
  double eps_a, eps_r;
  int32_t max_iters, ls_max_iters;
  double ls_tol;
} mpmrb_solver_params;   /* solver.py:35-49 */

typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t ls_evals;          /* total line-search derivative evaluations */
  int32_t regularized;       /* Hessian blocks regularised (solver.py:244 warning) */
  int32_t status;            /* MPMRB_OK / NOT_DESCENT / NONFINITE */
  int32_t pad_;
} mpmrb_solve_report;

/* Per-step statistics for advance_step's StepSummary (coupling.py:70-84). */
typedef struct {
  int32_t substeps;
  int32_t all_converged;
  int32_t iterations_max;
  int32_t n_contacts_max;
  double iterations_mean;
  double n_contacts_mean;
  double n_active_mean;
  int64_t clamped;
  int64_t ls_evals;
  int64_t regularized;
  int32_t status;           /* first error of the step (MPMRB_E_*) */
  int32_t status_detail;
  int64_t status_aux;
  /* contact solves of the step that stopped at max_iters without meeting the
   * residual test (solver.py:358-362) and the iterations they spent */
  int32_t substeps_unconverged;
  int32_t reserved;
  int64_t iterations_total;
  int64_t iterations_unconverged;
} mpmrb_step_stats;

/* ------------------------------------------------------------------ lifecycle */
int mpmrb_abi_version(void);
const char* mpmrb_last_error(void);
int mpmrb_create(int device, mpmrb_ctx** out);
int mpmrb_destroy(mpmrb_ctx* ctx);
int mpmrb_set_stream(mpmrb_ctx* ctx, void* cuda_stream);
/* Synchronise the stream and raise any device-side error recorded so far. */
int mpmrb_sync(mpmrb_ctx* ctx);
/* Number of kernel launches this context has issued (for bench accounting). */
int64_t mpmrb_launch_count(mpmrb_ctx* ctx);

/* ------------------------------------------------------------------ binning */
/* transfer.py:85-102 build_sort_plan (stable 10-bit Morton counting sort).
 * bin_keys must hold 1024, bin_starts 1025 entries; *n_bins_host is set
 * (synchronises).  Range errors -> MPMRB_E_INVALID (transfer.py:58-59). */
int mpmrb_sort_plan(mpmrb_ctx* ctx, const double* x, int64_t n, double h, uint16_t* keys,
                    int64_t* perm, int64_t* inv_perm, uint16_t* bin_keys,
                    int64_t* bin_starts, int64_t* bin_of, int64_t* n_bins_host);
/* transfer.py:105-113 plan_staleness; result written to *out_host (synchronises). */
int mpmrb_plan_staleness(mpmrb_ctx* ctx, const uint16_t* plan_keys, const double* x,
                         int64_t n, double h, double* out_host);
/* grid.py:34-36 base_cells -> (n,3) int64 */
int mpmrb_base_cells(mpmrb_ctx* ctx, const double* x, int64_t n, double h, int64_t* cells);
/* grid.py:71-103 SparseGrid.allocate.  Writes sorted unique block keys and a
 * hash table (hash_cap must be a power of two >= 2*block_cap).  *n_blocks_host
 * always receives the true block count; if it exceeds block_cap the call
 * returns MPMRB_E_CAPACITY and the caller retries with more room. */
int mpmrb_grid_allocate(mpmrb_ctx* ctx, const double* x, int64_t n, double h,
                        int64_t* block_keys, int64_t block_cap, uint64_t* hash_keys,
                        int32_t* hash_vals, int64_t hash_cap, int64_t* n_blocks_host);
/* grid.py:105-122 SparseGrid.node_ids; misses -> MPMRB_E_ALLOCATION. */
int mpmrb_node_ids(mpmrb_ctx* ctx, const mpmrb_grid_view* grid, const int64_t* coords,
                   int64_t m, int64_t* ids);
/* mpm.py:39-53 build_stencil: weights (n,27), nodes (n,27), dpos (n,27,3). */
int mpmrb_build_stencil(mpmrb_ctx* ctx, const mpmrb_grid_view* grid, const double* x,
                        int64_t n, double* weights, int64_t* nodes, double* dpos);

/* particles.py:97-136 seed_box on the GPU: the jittered lattice of cells
 * [lo, hi) with per_axis^3 points per cell, jitter drawn exactly as
 * numpy.random.default_rng(seed).uniform (PCG64 jump-ahead; state4_host =
 * bit_generator state hi, lo, inc hi, lo), kept where |x - center| <= half.
 * Bit-identical to the reference's NumPy seeding.  x_out may be NULL to count;
 * *n_host receives the count (synchronises); MPMRB_E_CAPACITY if cap is too
 * small. */
int mpmrb_seed_box(mpmrb_ctx* ctx, const int64_t* lo_host, const int64_t* hi_host,
                   int32_t per_axis, double jitter, double h, const double* center_host,
                   const double* half_host, const uint64_t* state4_host, double* x_out,
                   int64_t cap, int64_t* n_host);

/* ------------------------------------------------------------------ transfer */
/* transfer.py:148-248 scatter_reduce: out (n_out, nch) = sum over (rows,k). */
int mpmrb_scatter_reduce(mpmrb_ctx* ctx, const int64_t* node_ids, const double* values,
                         int64_t rows, int64_t k, int64_t nch, int64_t n_out, double* out);
/* transfer.py:135-145,178-187 scatter_reduce(mode="deterministic"): the same
 * sums as mpmrb_scatter_reduce, each (node, channel) folded left to right in
 * flattened (row, slot) order from 0.0 -- the reference's np.bincount order,
 * so the result is bitwise identical to the reference's for the same inputs
 * and independent of any sort plan.  rows * k and n_out must be < 2^31. */
int mpmrb_scatter_reduce_ordered(mpmrb_ctx* ctx, const int64_t* node_ids, const double* values,
                                 int64_t rows, int64_t k, int64_t nch, int64_t n_out,
                                 double* out);
/* mpm.py:56-63 compute_stresses (Kirchhoff tau per particle). */
int mpmrb_compute_stresses(mpmrb_ctx* ctx, const double* f, const int64_t* material_id,
                           int64_t n, const mpmrb_material* mats_host, int32_t n_mats,
                           double* tau);
/* mpm.py:66-99 particle_to_grid; outputs are overwritten (n_nodes = 64*nb). */
int mpmrb_p2g(mpmrb_ctx* ctx, const mpmrb_grid_view* grid, const mpmrb_particles* p,
              const mpmrb_material* mats_host, int32_t n_mats, double dt, double* mass,
              double* mom_apic, double* mom_force);
/* mpm.py:66-99 particle_to_grid(mode="deterministic"): the reference's
 * (n, 27, 7) contributions summed with the ordered scatter
 * (mpmrb_scatter_reduce_ordered): every node channel is folded in particle-id
 * / slot order, so the grid is bitwise reproducible and independent of the
 * particle order's plan.  Same arguments as mpmrb_p2g. */
int mpmrb_p2g_ordered(mpmrb_ctx* ctx, const mpmrb_grid_view* grid, const mpmrb_particles* p,
                      const mpmrb_material* mats_host, int32_t n_mats, double dt, double* mass,
                      double* mom_apic, double* mom_force);
/* mpm.py:102-115 grid_update. */
int mpmrb_grid_update(mpmrb_ctx* ctx, int64_t n_nodes, const double* mass,
                      const double* mom_apic, const double* mom_force,
                      const double* gravity_host, double dt, uint8_t* active, double* v_k,
                      double* v_star);
/* mpm.py:118-138 grid_to_particle (+ materials.py:86-110 clamp, + sand return
 * map).  Updates p->x, v, c, f (and plastic) in place; *n_clamped_host set
 * (synchronises). */
int mpmrb_g2p(mpmrb_ctx* ctx, const mpmrb_grid_view* grid, const mpmrb_particles* p,
              const mpmrb_material* mats_host, int32_t n_mats, const double* v_next,
              double dt, int64_t* n_clamped_host);

/* materials.py:86-110 clamp_degenerate: f_out = repaired F; *n_bad_host set. */
int mpmrb_clamp_degenerate(mpmrb_ctx* ctx, const double* f, int64_t n, double* f_out,
                           int64_t* n_bad_host);

/* ------------------------------------------------------------------ contacts */
/* contact_model.py:62-111 contact_energy / contact_gradient / contact_hessian,
 * evaluated by the same device functions the solver kernel uses.  Any of the
 * outputs may be NULL; hess is (n,3,3). */
int mpmrb_contact_model(mpmrb_ctx* ctx, const double* vc, const double* phi,
                        const double* gamma_lag, const double* mu, int64_t n, double stiffness,
                        double tau_d, double eps_v, double dt, double* energy, double* grad,
                        double* hess);
/* materials.py:70-83 polar_rotation of n 3x3 matrices (device arrays), the
 * Higham iteration with a per-matrix stop at max|dR| <= 1e-13 (the reference
 * stops on the batch-wide maximum; the extra iterations change R only at
 * roundoff). */
int mpmrb_polar_rotation(mpmrb_ctx* ctx, const double* f, int64_t n, double* r);
/* Exclusive prefix sum of n int32 device values into out (device); *total
 * (device, may be NULL) receives the sum.  The offsets behind the reference's
 * compactions and counting sorts: np.flatnonzero in collision.py:105 (contact
 * selection) and solver.py:202 (active nodes), the stable integer argsort of
 * transfer.py:89.  Single pass (decoupled look-back) for n <= 2^25, in the
 * context's stream; does not synchronise. */
int mpmrb_scan_exclusive_i32(mpmrb_ctx* ctx, const int32_t* in, int64_t n, int32_t* out,
                             int32_t* total);
/* materials.py:57-67 inverse_transpose3 via the adjugate. */
int mpmrb_inverse_transpose3(mpmrb_ctx* ctx, const double* m, int64_t n, double* out);
/* solver.py:224-256 solve_search_direction: d = -H^-1 g for n SPD 3x3 blocks
 * h (n,3,3) and g (n,3), device arrays; blocks that fail the Cholesky are
 * regularised like the reference.  *n_regularized_host counts them (the
 * reference's warning); MPMRB_E_NONFINITE if any block is still not SPD after
 * the last attempt (the reference's FloatingPointError).  Synchronises. */
int mpmrb_search_direction(mpmrb_ctx* ctx, const double* h, const double* g, int64_t n,
                           double* d, int32_t* n_regularized_host);
/* geometry.py:162-169 query_signed_distance for one geom in its LOCAL frame. */
int mpmrb_sdf_query(mpmrb_ctx* ctx, const mpmrb_geom* geom_host, const double* points,
                    int64_t n, double* phi, double* normal, double* witness);
/* geometry.py:186-189 contact_frames. */
int mpmrb_contact_frames(mpmrb_ctx* ctx, const double* normals, int64_t n, double* frames);
/* collision.py:88-132 detect_contacts with the BiasCache (collision.py:55-85)
 * as per-(geom, particle) slots: bias_stamp (n_geoms*n int32) and bias_store
 * (n_geoms*n*3); a slot is valid when stamp == epoch_stamp.  Outputs are
 * SoA arrays of capacity `cap`; *n_contacts_host is set (synchronises) and
 * MPMRB_E_CAPACITY returned if cap is too small. */
int mpmrb_detect_contacts(mpmrb_ctx* ctx, const double* x, int64_t n,
                          const mpmrb_geom* geoms_host, int32_t n_geoms, double margin,
                          int32_t* bias_stamp, double* bias_store, int32_t epoch_stamp,
                          int64_t cap, int64_t* particle, int64_t* body, int64_t* geom,
                          double* phi, double* normal, double* witness, double* frames,
                          double* bias, double* mu, int64_t* n_contacts_host);
/* collision.py:135-143 contact_velocities for stencils (nc,27). */
int mpmrb_contact_velocities(mpmrb_ctx* ctx, const int64_t* nodes, const double* w,
                             const double* frames, const double* bias, int64_t nc,
                             const double* v_grid, double* vc);

/* ------------------------------------------------------------------ solver */
/* solver.py:379-382 quasi_newton_solve.  v (nd,3) receives the solution,
 * gamma (nc,3) the impulses; traces (may be NULL) have max_iters+1 entries
 * each: objective, residual, threshold, and max_iters entries of alpha. */
int mpmrb_qn_solve(mpmrb_ctx* ctx, const mpmrb_problem* prob_host,
                   const mpmrb_solver_params* params_host, const double* v0, double* v,
                   double* gamma, double* objective, double* residual, double* threshold,
                   double* alpha, mpmrb_solve_report* report_host);
/* The same solve with free nodes held outside the problem (slab domain
 * decomposition: the contact problem is gathered to one rank, every rank keeps
 * its contact-free active nodes).  ext_free_host[3] = the external nodes'
 * S0 = sum m |v0 - v*|^2, Q0 = sum m |v*|^2, Q1 = sum m v*.(v0 - v*); they
 * enter every reduction in closed form (their g = m (v - v*), H = m I), and
 * *p_host receives P = prod(1 - alpha) so that each rank finishes its free
 * nodes as v = v* + P (v0 - v*).  No reference counterpart: the reference is
 * single-process. */
int mpmrb_qn_solve_ext(mpmrb_ctx* ctx, const mpmrb_problem* prob_host,
                       const mpmrb_solver_params* params_host, const double* v0,
                       const double* ext_free_host, double* v, double* gamma, double* objective,
                       double* residual, double* threshold, double* alpha, double* p_host,
                       mpmrb_solve_report* report_host);

/* Solver phase timers (globaltimer ns, accumulated over solves since the last
 * reset) when the context was created with MPMRB_SOLVER_PROF=1, else zeros:
 * [0] init [1] node phase [2] dvc phase [3] line search [4] update
 * [5] epilogue [6] iterations [7] line-search evals [8] sum of CTAs [9] solves. */
int mpmrb_solver_profile(mpmrb_ctx* ctx, uint64_t* out_host /*16*/, int32_t reset);
/* Per-CTA time (ns) of the node (N), direction (D), update (U) phases and of
 * the node-phase grid reduction, accumulated like mpmrb_solver_profile:
 * out_host[phase * 160 + cta], 800 words (diagnostics of load balance across
 * the cooperative grid). */
int mpmrb_solver_profile_cta(mpmrb_ctx* ctx, uint64_t* out_host /*800*/);

/* ------------------------------------------------------------------ fused substep */
/* coupling.py:115-219 as a device pipeline: one CUDA graph per substep. */
typedef struct mpmrb_sim mpmrb_sim;
int mpmrb_sim_create(mpmrb_ctx* ctx, mpmrb_sim** out);
int mpmrb_sim_destroy(mpmrb_sim* sim);
/* Bind particle arrays (kept by pointer; rebind after reallocation). */
int mpmrb_sim_set_particles(mpmrb_sim* sim, const mpmrb_particles* p);
int mpmrb_sim_set_materials(mpmrb_sim* sim, const mpmrb_material* mats_host, int32_t n);
/* Body poses are frozen per coupling step (coupling.py:1-8): set before each step. */
int mpmrb_sim_set_geoms(mpmrb_sim* sim, const mpmrb_geom* geoms_host, int32_t n_geoms,
                        int32_t n_bodies);
int mpmrb_sim_set_params(mpmrb_sim* sim, double h, double dt_substep,
                         const double* gravity_host, double stiffness, double tau_d,
                         double eps_v, double margin, const mpmrb_solver_params* solver);
/* Precision of the fused substep's particle state and arithmetic (north_star
 * "fp64 oracle mode; fp32 performance mode").  MPMRB_PREC_F64 (default) is the
 * reference's float64 everywhere.  MPMRB_PREC_F32 keeps the sim-internal
 * copy of v, F, C, mass, volume, plastic strain and the cached sand stress in
 * float32 and does the per-particle arithmetic (stress, SVD, return map, P2G
 * contributions, G2P) in float32; positions, grid channels, contacts and the
 * contact solve stay float64, and the user's arrays stay float64 (converted
 * at begin/end_step).  Not combinable with cloth (MPMRB_E_INVALID).  No
 * reference counterpart (the reference is float64 only). */
enum { MPMRB_PREC_F64 = 0, MPMRB_PREC_F32 = 1 };
int mpmrb_sim_set_precision(mpmrb_sim* sim, int32_t precision);
/* Codimensional cloth (new): triangles with vertex particles
 * and one element particle each.  All arrays are device arrays in the user's
 * (reference) particle order: tri (ne,3) and epart (ne,) particle indices,
 * dm_inv (ne,2,2) rest inverse, vol (ne,) rest volume, d3 (ne,3) transverse
 * direction (state, updated in place every substep), role (n,) int8
 * MPMRB_CLOTH_*.  Pass ne = 0 to remove the cloth. */
int mpmrb_sim_set_cloth(mpmrb_sim* sim, int64_t n_elements, const int32_t* tri,
                        const int32_t* epart, const double* dm_inv, const double* vol,
                        double* d3, const int8_t* role);
/* coupling.py:168-182: plan epoch, bias-cache reset, accumulator reset.
 * Sizes the grid/contact capacity for this step (synchronises once). */
int mpmrb_sim_begin_step(mpmrb_sim* sim, int64_t epoch, int32_t n_substeps);
/* coupling.py:115-150, enqueued (no host sync). */
int mpmrb_sim_substep(mpmrb_sim* sim);
/* coupling.py:192-216: reads per-substep stats and the accumulated impulses
 * (n_bodies*6: linear then angular, NOT divided by dt).  Synchronises. */
int mpmrb_sim_end_step(mpmrb_sim* sim, mpmrb_step_stats* stats_host,
                       double* impulses_host);
/* Run ONE substep with direct launches and CUDA events between the 7
 * pipeline stages (grid build, P2G, grid update+compaction, contacts, solve,
 * reactions, G2P): stage_ms_host[7]; sizes_host[5] = nb, n_active, n_contacts,
 * solver iterations, line-search evaluations.  Must be called between
 * begin_step and end_step (it is one of that step's substeps). */
int mpmrb_sim_profile_substep(mpmrb_sim* sim, float* stage_ms_host, int32_t* sizes_host);
/* transfer.py:105-113 plan staleness measured at the last end_step. */
double mpmrb_sim_staleness(mpmrb_sim* sim);
/* Device pointers of the most recent substep's grid (for parity tests). */
int mpmrb_sim_last_grid(mpmrb_sim* sim, int64_t* n_blocks_host, const int64_t** block_keys,
                        const double** mass, const double** v_star, const double** v_next);
/* Number of contacts of the most recent substep and its device arrays. */
int mpmrb_sim_last_contacts(mpmrb_sim* sim, int64_t* n_host, const int32_t** particle,
                            const double** gamma_world);

/* ---------------------------------------------------- slab decomposition hooks
 * slab.py's fused mode runs each substep in parts so that the exchanges of a
 * slab-decomposed scene sit between them: part 0 = grid build + P2G; (P2G
 * halo reduce on the grid channels); part 1 = grid update, active compaction,
 * contact detection and preparation; part 2 = the contact solve, or instead
 * the distributed solve writing v_next and gamma through the views and
 * mpmrb_sim_set_solve_result; part 3 = reactions, substep end, G2P.
 * Parts 0..3 in order are mpmrb_sim_substep with direct launches. */
typedef struct {
  int64_t n_blocks, n_active, n_contacts;   /* device counters, read back */
  int64_t nc_cap;                            /* row stride of cnodes / cw */
  const int64_t* block_keys;  /* (n_blocks,) sorted packed block keys (grid.py:26-31) */
  double* mass;               /* (n_blocks*64,) node = block rank * 64 + (lx*4+ly)*4+lz */
  double* mom_apic;           /* (n_blocks*64, 3) */
  double* mom_force;          /* (n_blocks*64, 3) */
  const double* v_star;       /* (n_blocks*64, 3), valid after part 1 */
  const double* v_k;          /* (n_blocks*64, 3) */
  double* v_next;             /* (n_blocks*64, 3), read by part 3's G2P */
  const int32_t* act;         /* (n_active,) node index of each active node, ascending */
  const double* m_act;        /* (n_active,) m, v*, v_k of the active nodes */
  const double* v_star_act;   /* (n_active, 3) */
  const double* v_k_act;      /* (n_active, 3) */
  const int32_t* cnodes;      /* (27, nc_cap) active index of each stencil slot, -1 dead */
  const double* cw;           /* (27, nc_cap) stencil weight, 0 for dead slots */
  const double* frames;       /* (n_contacts, 3, 3) contact frames */
  const double* bias;         /* (n_contacts, 3) */
  const double* phi;          /* (n_contacts,) */
  const double* mu;           /* (n_contacts,) */
  const double* gamma_lag;    /* (n_contacts,) */
  double* gamma;              /* (n_contacts, 3) contact-frame impulses (part 3 reads) */
} mpmrb_sim_views;
int mpmrb_sim_substep_part(mpmrb_sim* sim, int32_t part);
/* Synchronises the sim's stream and reads the counters back. */
int mpmrb_sim_get_views(mpmrb_sim* sim, mpmrb_sim_views* out);
/* The report of a solve done outside part 2 (iterations, convergence, line-
 * search evaluations) for the step statistics. */
int mpmrb_sim_set_solve_result(mpmrb_sim* sim, const mpmrb_solve_report* report);

#ifdef __cplusplus
}
#endif
#endif /* MPMRB_B200_H */
