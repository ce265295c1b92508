// Host-side internals shared by the .cu translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstddef>
#include <cstdint>

#include "../../include/mpmrb_b200.h"

namespace mpmrb {

struct DevStatus;

int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* expr, const char* file, int line);

// A grow-only device buffer.  Growth frees the old allocation, so it must not
// happen while a captured graph still references it (sim code re-captures).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  int grow(size_t need);  // returns MPMRB_OK or MPMRB_E_CUDA
  void release();
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  DevStatus* status = nullptr;   // device
  DevStatus* status_host = nullptr;  // pinned mirror
  long long launches = 0;
  DevBuf scratch[32];
  // phase timers of the solver kernel (enabled by MPMRB_SOLVER_PROF=1)
  unsigned long long* solver_prof = nullptr;
  // single-pass scan state (scan.cu): [0] ticket | epoch, [1..] tile status;
  // zeroed once at creation, never reset (epoch-tagged), so scans replay
  // inside CUDA graphs
  unsigned long long* scan_state = nullptr;
  int check_status(const char* where);  // sync + read + clear device status
};

// Scratch slot ids for API-level (non-fused) calls.
constexpr int kOnePassMaxTiles = 8192;  // single-pass scans up to 2^25 elements (4096 per tile)

enum ScratchSlot {
  SS_TILE = 0, SS_TILE2, SS_HIST, SS_KEYS, SS_TMP0, SS_TMP1, SS_TMP2, SS_TMP3, SS_COUNT,
  SS_SOLVER0, SS_SOLVER1, SS_SOLVER2, SS_SOLVER3, SS_SOLVER4, SS_SOLVER5, SS_SOLVER6,
  SS_SOLVER7, SS_SOLVER8, SS_MATS, SS_GEOMS, SS_PROBLEM, SS_HOSTINFO,
  // ordered (deterministic) scatter / P2G
  SS_ORD_K, SS_ORD_I, SS_ORD_S, SS_ORD_N, SS_ORD_V, SS_ORD_O,
  SS_DIR  // search-direction counters (mpmrb_search_direction)
};

inline unsigned grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// ---- launchers (each returns MPMRB_OK or an error code) --------------------
// scan.cu
int scan_exclusive_i32(Ctx& c, const int* in, int* out, long long n_cap, const int* n_dev,
                       int* total_dev, DevBuf& tiles);
int scan_exclusive_i64(Ctx& c, const long long* in, long long* out, long long n, long long* total_dev,
                       DevBuf& tiles);

// binning.cu
int launch_base_cells(Ctx& c, const double* x, long long n, double h, long long* cells);
int launch_sort_plan(Ctx& c, const double* x, long long n, double h, uint16_t* keys,
                     long long* perm, long long* inv_perm, uint16_t* bin_keys,
                     long long* bin_starts, long long* bin_of, int* n_bins_dev);
int launch_staleness(Ctx& c, const uint16_t* plan_keys, const double* x, long long n,
                     double h, unsigned long long* changed_dev);
// Block discovery into a hash table; writes sorted keys and hash values.
// counters_dev[0] receives nb.  Capacity overflow raises MPMRB_E_CAPACITY in
// the device status (aux = needed count), range errors MPMRB_E_ALLOCATION.
int launch_grid_build(Ctx& c, const double* x, long long n, double h, long long* block_keys,
                      long long block_cap, unsigned long long* hkeys, int* hvals,
                      long long hash_cap, long long* ukeys_scratch, int* nb_dev);
int launch_node_ids(Ctx& c, const mpmrb_grid_view& g, const long long* coords, long long m,
                    long long* ids);
int launch_build_stencil(Ctx& c, const mpmrb_grid_view& g, const double* x, long long n,
                         double* weights, long long* nodes, double* dpos);

// mpm.cu
int launch_scatter_reduce(Ctx& c, const long long* ids, const double* vals, long long rows,
                          long long k, long long nch, long long n_out, double* out);
int launch_stresses(Ctx& c, const double* f, const long long* mid, long long n,
                    const mpmrb_material* mats_dev, int nmat, double* tau);
// Particle state as the kernels see it.  T is the precision of the
// per-particle state and arithmetic: double (the reference's float64, and the
// user's arrays) or float (the sim-internal copy in the fp32 performance
// mode).  Positions are always float64.
template <class T>
struct ParticlesT {
  double* x;
  T* v;
  T* f;
  T* c;
  const T* mass;
  const T* vol0;
  const long long* mid;
  T* plastic;
  long long n;
  // codimensional cloth (NULL when absent; both precisions): role per
  // particle (MPMRB_CLOTH_*), element stresses written by the cloth kernel,
  // vertex forces
  const signed char* role = nullptr;
  double* tau = nullptr;   // (n,9)
  double* fext = nullptr;  // (n,3)
  // sand: Hencky stress of the post-return-map F written by G2P for the next
  // substep's P2G (symmetric, 6 entries); valid when *tau_valid != 0
  T* tau_cache = nullptr;  // (n,6)
  int* tau_valid = nullptr;
};
using ParticlesDev = ParticlesT<double>;
using ParticlesF32 = ParticlesT<float>;
struct ClothDev {
  long long ne = 0;
  const int* tri = nullptr;
  const int* epart = nullptr;
  const double* dm_inv = nullptr;
  const double* vol = nullptr;
  double* d3 = nullptr;
  const int* inv_perm = nullptr;
};
struct GridDev {
  const unsigned long long* hkeys;
  const int* hvals;
  unsigned mask;
  double h;
};
int launch_p2g(Ctx& c, const GridDev& g, const ParticlesDev& p, const mpmrb_material* mats_dev,
               int nmat, double dt, double* mass, double* mom_apic, double* mom_force);
int launch_grid_update(Ctx& c, long long n_nodes_cap, const int* nb_dev, const double* mass,
                       const double* mom_apic, const double* mom_force, double gx, double gy,
                       double gz, double dt, unsigned char* active, double* v_k, double* v_star,
                       double* v_next_or_null, int* block_active_count_or_null);
int launch_g2p(Ctx& c, const GridDev& g, const ParticlesDev& p, const mpmrb_material* mats_dev,
               int nmat, const double* v_next, double dt, unsigned long long* clamped_dev,
               int* health_dev);
// fp32 performance mode: the same transfers on float32 particle state
int launch_p2g(Ctx& c, const GridDev& g, const ParticlesF32& p, const mpmrb_material* mats_dev,
               int nmat, double dt, double* mass, double* mom_apic, double* mom_force);
int launch_g2p(Ctx& c, const GridDev& g, const ParticlesF32& p, const mpmrb_material* mats_dev,
               int nmat, const double* v_next, double dt, unsigned long long* clamped_dev,
               int* health_dev);

// seed.cu
int launch_seed_box(Ctx& c, const long long* lo, const long long* hi, int per_axis,
                    double jitter, double h, const double* center, const double* half,
                    const unsigned long long* state4, double* x_out, long long cap,
                    long long* n_host);

// cloth.cu
int launch_cloth_forces(Ctx& c, const ClothDev& cl, const ParticlesDev& p,
                        const mpmrb_material* mats_dev, int nmat);
int launch_cloth_post(Ctx& c, const ClothDev& cl, const ParticlesDev& p,
                      const mpmrb_material* mats_dev, int nmat, double dt);
int launch_cloth_post(Ctx& c, const ClothDev& cl, const ParticlesF32& p,
                      const mpmrb_material* mats_dev, int nmat, double dt);
int launch_inverse_perm(Ctx& c, const int* perm, long long n, int* inv);
int launch_gather_i8(Ctx& c, const signed char* src, const int* perm, long long n,
                     signed char* dst);

int launch_clamp(Ctx& c, const double* f, long long n, double* out, unsigned long long* nbad);
int launch_polar(Ctx& c, const double* f, long long n, int inv_t_only, double* out);
int launch_health(Ctx& c, const double* x, const double* v, long long n, double h, int* bad);

// reorder.cu: once-per-step (block, cell) particle order
int sort_pairs_u32(Ctx& c, unsigned* ka, int* va, unsigned* kb, int* vb, long long n, int bits,
                   int* vals_out, unsigned** keys_out);
int launch_p2g_ordered(Ctx& c, const GridDev& g, const ParticlesDev& p,
                       const mpmrb_material* mats_dev, int nmat, double dt, long long n_nodes,
                       double* mass, double* mom_apic, double* mom_force);
int launch_scatter_reduce_ordered(Ctx& c, const long long* ids, const double* vals,
                                  long long rows, long long k, long long nch, long long n_out,
                                  double* out);
int launch_particle_sort(Ctx& c, const double* x, long long n, double h,
                         const unsigned long long* hkeys, const int* hvals, long long hash_cap,
                         long long n_blocks_cap, unsigned* keys2, int* vals2, int* perm_out);
int launch_particle_gather(Ctx& c, const int* perm, long long n, const double* src, int width,
                           double* dst);
int launch_particle_scatter(Ctx& c, const int* perm, long long n, const double* src, int width,
                            double* dst);
// float64 user arrays <-> float32 sim-internal copy (fp32 performance mode)
int launch_particle_gather_f32(Ctx& c, const int* perm, long long n, const double* src, int width,
                               float* dst);
int launch_particle_scatter_f32(Ctx& c, const int* perm, long long n, const float* src, int width,
                                double* dst);
int launch_gather_i64(Ctx& c, const int* perm, long long n, const long long* src, long long* dst);
int launch_map_ids(Ctx& c, const int* ids, const int* perm, const int* n_dev, long long cap,
                   int* out);

// contact.cu
int launch_contact_model(Ctx& c, const double* vc, const double* phi, const double* gl,
                         const double* mu, long long n, double K, double den, double eps_v,
                         double* energy, double* grad, double* hess);
int launch_sdf_query(Ctx& c, const mpmrb_geom* g_dev, const double* pts, long long n, double* phi,
                     double* normal, double* witness);
int launch_frames(Ctx& c, const double* normals, long long n, double* frames);
int launch_contact_velocities(Ctx& c, const long long* nodes, const double* w,
                              const double* frames, const double* bias, long long nc,
                              const double* v_grid, double* vc);

}  // namespace mpmrb
