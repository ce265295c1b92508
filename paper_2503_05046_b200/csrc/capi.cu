// extern "C" boundary of libmpmrb_b200.so (include/mpmrb_b200.h).
#include <cstdio>
#include <cstring>
#include <new>

#include "common.cuh"
#include "contact.cuh"
#include "internal.h"
#include "sim.h"
#include "solver.cuh"

namespace mpmrb {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t e, const char* expr, const char* file, int line) {
  return set_error(MPMRB_E_CUDA, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                   cudaGetErrorString(e), expr, file, line);
}

int DevBuf::grow(size_t need) {
  if (need <= bytes && p) return MPMRB_OK;
  if (need == 0) need = 16;
  size_t nb = need + need / 4 + 256;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, nb);
  if (e != cudaSuccess) {
    set_cuda_error(e, "cudaMalloc", __FILE__, __LINE__);
    return MPMRB_E_CUDA;
  }
  if (p) cudaFree(p);
  p = q;
  bytes = nb;
  return MPMRB_OK;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

static const char* code_name(int code) {
  switch (code) {
    case MPMRB_E_ALLOCATION: return "AllocationError";
    case MPMRB_E_PLAN_EPOCH: return "PlanEpochError";
    case MPMRB_E_INVALID: return "ValueError";
    case MPMRB_E_NOT_DESCENT: return "line search needs a descent direction";
    case MPMRB_E_NONFINITE: return "FloatingPointError";
    case MPMRB_E_DIVERGED: return "SimulationDiverged";
    case MPMRB_E_CAPACITY: return "capacity exceeded";
    default: return "error";
  }
}

int Ctx::check_status(const char* where) {
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaStreamSynchronize", where, 0);
  DevStatus h{};
  e = cudaMemcpy(&h, status, sizeof(DevStatus), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemcpy(status)", where, 0);
  if (h.code == 0) return MPMRB_OK;
  cudaMemset(status, 0, sizeof(DevStatus));
  return set_error(h.code, "%s: %s (site %d, index %lld)", where, code_name(h.code), h.detail,
                   h.aux);
}

}  // namespace mpmrb

using namespace mpmrb;

struct mpmrb_ctx : public Ctx {};
struct mpmrb_sim : public Sim {};

#define CHECK_CTX(c) \
  if (!(c)) return set_error(MPMRB_E_INVALID, "null context")

extern "C" {

int mpmrb_abi_version(void) { return MPMRB_ABI_VERSION; }

const char* mpmrb_last_error(void) { return g_err; }

int mpmrb_create(int device, mpmrb_ctx** out) {
  if (!out) return set_error(MPMRB_E_INVALID, "out is null");
  MPMRB_CUDA_OK(cudaSetDevice(device));
  mpmrb_ctx* c = new (std::nothrow) mpmrb_ctx();
  if (!c) return set_error(MPMRB_E_INVALID, "out of host memory");
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&c->status, sizeof(DevStatus));
  if (e != cudaSuccess) {
    delete c;
    return set_cuda_error(e, "cudaMalloc(status)", __FILE__, __LINE__);
  }
  cudaMemset(c->status, 0, sizeof(DevStatus));
  if (cudaMalloc(&c->scan_state, 8 * (kOnePassMaxTiles + 2)) == cudaSuccess)
    cudaMemset(c->scan_state, 0, 8 * (kOnePassMaxTiles + 2));
  else
    c->scan_state = nullptr;  // scans take the three-kernel path
  const char* prof = getenv("MPMRB_SOLVER_PROF");
  if (prof && atoi(prof) > 0) {
    if (cudaMalloc(&c->solver_prof, 8 * kSolverProfWords) == cudaSuccess)
      cudaMemset(c->solver_prof, 0, 8 * kSolverProfWords);
    else
      c->solver_prof = nullptr;
  }
  *out = c;
  return MPMRB_OK;
}

int mpmrb_solver_profile(mpmrb_ctx* c, uint64_t* out_host, int32_t reset) {
  CHECK_CTX(c);
  if (!c->solver_prof) {
    std::memset(out_host, 0, 8 * kSolverProf);
    return MPMRB_OK;
  }
  MPMRB_CUDA_OK(cudaStreamSynchronize(c->stream));
  MPMRB_CUDA_OK(cudaMemcpy(out_host, c->solver_prof, 8 * kSolverProf, cudaMemcpyDeviceToHost));
  if (reset) MPMRB_CUDA_OK(cudaMemset(c->solver_prof, 0, 8 * kSolverProfWords));
  return MPMRB_OK;
}

int mpmrb_solver_profile_cta(mpmrb_ctx* c, uint64_t* out_host) {
  static_assert(kSolverProfWords - kSolverProf == 800, "profile layout");
  CHECK_CTX(c);
  if (!c->solver_prof) {
    std::memset(out_host, 0, 8 * (kSolverProfWords - kSolverProf));
    return MPMRB_OK;
  }
  MPMRB_CUDA_OK(cudaStreamSynchronize(c->stream));
  MPMRB_CUDA_OK(cudaMemcpy(out_host, c->solver_prof + kSolverProf,
                           8 * (kSolverProfWords - kSolverProf), cudaMemcpyDeviceToHost));
  return MPMRB_OK;
}

int mpmrb_destroy(mpmrb_ctx* c) {
  if (!c) return MPMRB_OK;
  cudaStreamSynchronize(c->stream);
  for (auto& b : c->scratch) b.release();
  if (c->status) cudaFree(c->status);
  if (c->scan_state) cudaFree(c->scan_state);
  if (c->solver_prof) cudaFree(c->solver_prof);
  delete c;
  return MPMRB_OK;
}

int mpmrb_set_stream(mpmrb_ctx* c, void* s) {
  CHECK_CTX(c);
  c->stream = (cudaStream_t)s;
  return MPMRB_OK;
}

int mpmrb_sync(mpmrb_ctx* c) {
  CHECK_CTX(c);
  return c->check_status("mpmrb_sync");
}

int64_t mpmrb_launch_count(mpmrb_ctx* c) { return c ? (int64_t)c->launches : 0; }

// ------------------------------------------------------------------ binning

int mpmrb_sort_plan(mpmrb_ctx* c, const double* x, int64_t n, double h, uint16_t* keys,
                    int64_t* perm, int64_t* inv_perm, uint16_t* bin_keys, int64_t* bin_starts,
                    int64_t* bin_of, int64_t* n_bins_host) {
  CHECK_CTX(c);
  if (n < 0 || !(h > 0)) return set_error(MPMRB_E_INVALID, "bad n or h");
  if (c->scratch[SS_COUNT].grow(64)) return MPMRB_E_CUDA;
  int* nb = c->scratch[SS_COUNT].as<int>();
  int rc = launch_sort_plan(*c, x, n, h, keys, (long long*)perm, (long long*)inv_perm, bin_keys,
                            (long long*)bin_starts, (long long*)bin_of, nb);
  if (rc) return rc;
  int hb = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&hb, nb, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("build_sort_plan");
  if (rc) return rc;
  *n_bins_host = hb;
  return MPMRB_OK;
}

int mpmrb_plan_staleness(mpmrb_ctx* c, const uint16_t* plan_keys, const double* x, int64_t n,
                         double h, double* out_host) {
  CHECK_CTX(c);
  if (c->scratch[SS_COUNT].grow(64)) return MPMRB_E_CUDA;
  unsigned long long* cnt = c->scratch[SS_COUNT].as<unsigned long long>();
  int rc = launch_staleness(*c, plan_keys, x, n, h, cnt);
  if (rc) return rc;
  unsigned long long hc = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&hc, cnt, 8, cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("plan_staleness");
  if (rc) return rc;
  *out_host = n > 0 ? (double)hc / (double)n : 0.0;
  return MPMRB_OK;
}

int mpmrb_base_cells(mpmrb_ctx* c, const double* x, int64_t n, double h, int64_t* cells) {
  CHECK_CTX(c);
  return launch_base_cells(*c, x, n, h, (long long*)cells);
}

int mpmrb_grid_allocate(mpmrb_ctx* c, const double* x, int64_t n, double h, int64_t* block_keys,
                        int64_t block_cap, uint64_t* hash_keys, int32_t* hash_vals,
                        int64_t hash_cap, int64_t* n_blocks_host) {
  CHECK_CTX(c);
  if (!(h > 0)) return set_error(MPMRB_E_INVALID, "grid spacing h must be positive");
  if (hash_cap < 2 || (hash_cap & (hash_cap - 1)) || hash_cap < 2 * block_cap)
    return set_error(MPMRB_E_INVALID, "hash_cap must be a power of two >= 2*block_cap");
  if (c->scratch[SS_KEYS].grow(8 * (block_cap + 1)) || c->scratch[SS_COUNT].grow(64))
    return MPMRB_E_CUDA;
  int* nb = c->scratch[SS_COUNT].as<int>();
  int rc = launch_grid_build(*c, x, n, h, (long long*)block_keys, block_cap,
                             (unsigned long long*)hash_keys, (int*)hash_vals, hash_cap,
                             c->scratch[SS_KEYS].as<long long>(), nb);
  if (rc) return rc;
  int hb = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&hb, nb, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("SparseGrid.allocate");
  *n_blocks_host = hb;
  return rc;
}

int mpmrb_node_ids(mpmrb_ctx* c, const mpmrb_grid_view* g, const int64_t* coords, int64_t m,
                   int64_t* ids) {
  CHECK_CTX(c);
  int rc = launch_node_ids(*c, *g, (const long long*)coords, m, (long long*)ids);
  if (rc) return rc;
  return c->check_status("SparseGrid.node_ids");
}

int mpmrb_build_stencil(mpmrb_ctx* c, const mpmrb_grid_view* g, const double* x, int64_t n,
                        double* weights, int64_t* nodes, double* dpos) {
  CHECK_CTX(c);
  int rc = launch_build_stencil(*c, *g, x, n, weights, (long long*)nodes, dpos);
  if (rc) return rc;
  return c->check_status("build_stencil");
}

// ------------------------------------------------------------------ transfer

int mpmrb_scatter_reduce(mpmrb_ctx* c, const int64_t* node_ids, const double* values,
                         int64_t rows, int64_t k, int64_t nch, int64_t n_out, double* out) {
  CHECK_CTX(c);
  int rc = launch_scatter_reduce(*c, (const long long*)node_ids, values, rows, k, nch, n_out, out);
  if (rc) return rc;
  return c->check_status("scatter_reduce");
}

int mpmrb_scatter_reduce_ordered(mpmrb_ctx* c, const int64_t* node_ids, const double* values,
                                 int64_t rows, int64_t k, int64_t nch, int64_t n_out,
                                 double* out) {
  CHECK_CTX(c);
  int rc = launch_scatter_reduce_ordered(*c, (const long long*)node_ids, values, rows, k, nch,
                                         n_out, out);
  if (rc) return rc;
  return c->check_status("scatter_reduce_ordered");
}

static int upload_mats(Ctx& c, const mpmrb_material* mats_host, int n) {
  if (c.scratch[SS_MATS].grow(sizeof(mpmrb_material) * (n > 0 ? n : 1))) return MPMRB_E_CUDA;
  if (n > 0)
    MPMRB_CUDA_OK(cudaMemcpyAsync(c.scratch[SS_MATS].p, mats_host, sizeof(mpmrb_material) * n,
                                  cudaMemcpyHostToDevice, c.stream));
  return MPMRB_OK;
}

int mpmrb_compute_stresses(mpmrb_ctx* c, const double* f, const int64_t* mid, int64_t n,
                           const mpmrb_material* mats_host, int32_t n_mats, double* tau) {
  CHECK_CTX(c);
  int rc = upload_mats(*c, mats_host, n_mats);
  if (rc) return rc;
  rc = launch_stresses(*c, f, (const long long*)mid, n, c->scratch[SS_MATS].as<mpmrb_material>(),
                       n_mats, tau);
  if (rc) return rc;
  return c->check_status("compute_stresses");
}

static GridDev grid_dev(const mpmrb_grid_view* g) {
  return GridDev{(const unsigned long long*)g->hash_keys, (const int*)g->hash_vals,
                 (unsigned)(g->hash_cap - 1), g->h};
}

static ParticlesDev particles_dev(const mpmrb_particles* p) {
  return ParticlesDev{p->x, p->v, p->f, p->c, p->mass, p->volume0,
                      (const long long*)p->material_id, p->plastic, p->n};
}

int mpmrb_p2g(mpmrb_ctx* c, const mpmrb_grid_view* g, const mpmrb_particles* p,
              const mpmrb_material* mats_host, int32_t n_mats, double dt, double* mass,
              double* mom_apic, double* mom_force) {
  CHECK_CTX(c);
  long long N = g->n_blocks * kNodesPerBlock;
  MPMRB_CUDA_OK(cudaMemsetAsync(mass, 0, 8 * N, c->stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(mom_apic, 0, 24 * N, c->stream));
  MPMRB_CUDA_OK(cudaMemsetAsync(mom_force, 0, 24 * N, c->stream));
  int rc = upload_mats(*c, mats_host, n_mats);
  if (rc) return rc;
  rc = launch_p2g(*c, grid_dev(g), particles_dev(p), c->scratch[SS_MATS].as<mpmrb_material>(),
                  n_mats, dt, mass, mom_apic, mom_force);
  if (rc) return rc;
  return c->check_status("particle_to_grid");
}

int mpmrb_p2g_ordered(mpmrb_ctx* c, const mpmrb_grid_view* g, const mpmrb_particles* p,
                      const mpmrb_material* mats_host, int32_t n_mats, double dt, double* mass,
                      double* mom_apic, double* mom_force) {
  CHECK_CTX(c);
  const long long N = g->n_blocks * kNodesPerBlock;
  int rc = upload_mats(*c, mats_host, n_mats);
  if (rc) return rc;
  rc = launch_p2g_ordered(*c, grid_dev(g), particles_dev(p),
                          c->scratch[SS_MATS].as<mpmrb_material>(), n_mats, dt, N, mass,
                          mom_apic, mom_force);
  if (rc) return rc;
  return c->check_status("p2g_ordered");
}

int mpmrb_grid_update(mpmrb_ctx* c, int64_t n_nodes, const double* mass, const double* mom_apic,
                      const double* mom_force, const double* g, double dt, uint8_t* active,
                      double* v_k, double* v_star) {
  CHECK_CTX(c);
  int rc = launch_grid_update(*c, n_nodes, nullptr, mass, mom_apic, mom_force, g[0], g[1], g[2],
                              dt, active, v_k, v_star, nullptr, nullptr);
  if (rc) return rc;
  return c->check_status("grid_update");
}

int mpmrb_g2p(mpmrb_ctx* c, const mpmrb_grid_view* g, const mpmrb_particles* p,
              const mpmrb_material* mats_host, int32_t n_mats, const double* v_next, double dt,
              int64_t* n_clamped_host) {
  CHECK_CTX(c);
  if (c->scratch[SS_COUNT].grow(64)) return MPMRB_E_CUDA;
  unsigned long long* cl = c->scratch[SS_COUNT].as<unsigned long long>();
  MPMRB_CUDA_OK(cudaMemsetAsync(cl, 0, 8, c->stream));
  int rc = upload_mats(*c, mats_host, n_mats);
  if (rc) return rc;
  rc = launch_g2p(*c, grid_dev(g), particles_dev(p), c->scratch[SS_MATS].as<mpmrb_material>(),
                  n_mats, v_next, dt, cl, nullptr);
  if (rc) return rc;
  unsigned long long h = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&h, cl, 8, cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("grid_to_particle");
  if (n_clamped_host) *n_clamped_host = (int64_t)h;
  return rc;
}

int mpmrb_clamp_degenerate(mpmrb_ctx* c, const double* f, int64_t n, double* f_out,
                           int64_t* n_bad_host) {
  CHECK_CTX(c);
  if (c->scratch[SS_COUNT].grow(64)) return MPMRB_E_CUDA;
  unsigned long long* nb = c->scratch[SS_COUNT].as<unsigned long long>();
  int rc = launch_clamp(*c, f, n, f_out, nb);
  if (rc) return rc;
  unsigned long long h = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&h, nb, 8, cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("clamp_degenerate");
  *n_bad_host = (int64_t)h;
  return rc;
}

// ------------------------------------------------------------------ contacts

int mpmrb_contact_model(mpmrb_ctx* c, const double* vc, const double* phi, const double* gl,
                        const double* mu, int64_t n, double k, double tau_d, double eps_v,
                        double dt, double* energy, double* grad, double* hess) {
  CHECK_CTX(c);
  int rc = launch_contact_model(*c, vc, phi, gl, mu, n, dt * (dt + tau_d) * k, dt + tau_d, eps_v,
                                energy, grad, hess);
  if (rc) return rc;
  return c->check_status("contact_model");
}

int mpmrb_polar_rotation(mpmrb_ctx* c, const double* f, int64_t n, double* r) {
  CHECK_CTX(c);
  int rc = launch_polar(*c, f, n, 0, r);
  if (rc) return rc;
  return c->check_status("polar_rotation");
}

int mpmrb_scan_exclusive_i32(mpmrb_ctx* c, const int32_t* in, int64_t n, int32_t* out,
                             int32_t* total) {
  CHECK_CTX(c);
  if (n < 0 || (n > 0 && (!in || !out))) return set_error(MPMRB_E_INVALID, "scan: bad arguments");
  if (n > (1LL << 31) - 1) return set_error(MPMRB_E_INVALID, "scan: n exceeds int32 range");
  return scan_exclusive_i32(*c, in, out, n, nullptr, total, c->scratch[SS_TILE]);
}

int mpmrb_inverse_transpose3(mpmrb_ctx* c, const double* m, int64_t n, double* out) {
  CHECK_CTX(c);
  int rc = launch_polar(*c, m, n, 1, out);
  if (rc) return rc;
  return c->check_status("inverse_transpose3");
}

int mpmrb_search_direction(mpmrb_ctx* c, const double* h, const double* g, int64_t n, double* d,
                           int32_t* n_reg) {
  CHECK_CTX(c);
  if (c->scratch[SS_DIR].grow(64)) return MPMRB_E_CUDA;
  int* reg = c->scratch[SS_DIR].as<int>();
  int rc = launch_search_direction(*c, h, g, n, d, reg);
  if (rc) return rc;
  int hreg[2] = {0, 0};
  MPMRB_CUDA_OK(cudaMemcpyAsync(hreg, reg, sizeof(hreg), cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("solve_search_direction");
  if (rc) return rc;
  if (n_reg) *n_reg = hreg[0];
  if (hreg[1]) return set_error(MPMRB_E_NONFINITE, "Hessian block not SPD after regularization");
  return MPMRB_OK;
}

int mpmrb_sdf_query(mpmrb_ctx* c, const mpmrb_geom* geom_host, const double* pts, int64_t n,
                    double* phi, double* normal, double* witness) {
  CHECK_CTX(c);
  if (c->scratch[SS_GEOMS].grow(sizeof(mpmrb_geom))) return MPMRB_E_CUDA;
  MPMRB_CUDA_OK(cudaMemcpyAsync(c->scratch[SS_GEOMS].p, geom_host, sizeof(mpmrb_geom),
                                cudaMemcpyHostToDevice, c->stream));
  int rc = launch_sdf_query(*c, c->scratch[SS_GEOMS].as<mpmrb_geom>(), pts, n, phi, normal,
                            witness);
  if (rc) return rc;
  return c->check_status("query_signed_distance");
}

int mpmrb_contact_frames(mpmrb_ctx* c, const double* normals, int64_t n, double* frames) {
  CHECK_CTX(c);
  int rc = launch_frames(*c, normals, n, frames);
  if (rc) return rc;
  return c->check_status("contact_frames");
}

int mpmrb_detect_contacts(mpmrb_ctx* c, const double* x, int64_t n, const mpmrb_geom* geoms_host,
                          int32_t n_geoms, double margin, int32_t* bias_stamp,
                          double* bias_store, int32_t epoch_stamp, int64_t cap,
                          int64_t* particle, int64_t* body, int64_t* geom, double* phi,
                          double* normal, double* witness, double* frames, double* bias,
                          double* mu, int64_t* n_contacts_host) {
  CHECK_CTX(c);
  if (c->scratch[SS_GEOMS].grow(sizeof(mpmrb_geom) * (n_geoms > 0 ? n_geoms : 1)) ||
      c->scratch[SS_TMP0].grow(4 * (n + 1)) || c->scratch[SS_TMP1].grow(4 * (n + 1)) ||
      c->scratch[SS_TMP2].grow(4 * (cap + 1)) || c->scratch[SS_COUNT].grow(64))
    return MPMRB_E_CUDA;
  if (n_geoms > 0)
    MPMRB_CUDA_OK(cudaMemcpyAsync(c->scratch[SS_GEOMS].p, geoms_host,
                                  sizeof(mpmrb_geom) * n_geoms, cudaMemcpyHostToDevice,
                                  c->stream));
  int* cnt_total = c->scratch[SS_COUNT].as<int>();
  int* epoch_dev = cnt_total + 4;
  MPMRB_CUDA_OK(cudaMemcpyAsync(epoch_dev, &epoch_stamp, 4, cudaMemcpyHostToDevice, c->stream));
  ContactArrays ca{};
  ca.particle = c->scratch[SS_TMP2].as<int>();
  ca.particle64 = (long long*)particle;
  ca.body64 = (long long*)body;
  ca.geom64 = (long long*)geom;
  ca.phi = phi;
  ca.normal = normal;
  ca.witness = witness;
  ca.frames = frames;
  ca.bias = bias;
  ca.mu = mu;
  int rc = launch_detect(*c, x, n, c->scratch[SS_GEOMS].as<mpmrb_geom>(), n_geoms, margin,
                         c->scratch[SS_TMP0].as<int>(), c->scratch[SS_TMP1].as<int>(), cnt_total,
                         c->scratch[SS_TILE], cap, bias_stamp, bias_store, epoch_dev, ca);
  if (rc) return rc;
  int tot = 0;
  MPMRB_CUDA_OK(cudaMemcpyAsync(&tot, cnt_total, 4, cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("detect_contacts");
  *n_contacts_host = tot;
  return rc;
}

int mpmrb_seed_box(mpmrb_ctx* c, const int64_t* lo, const int64_t* hi, int32_t per_axis,
                   double jitter, double h, const double* center, const double* half,
                   const uint64_t* state4, double* x_out, int64_t cap, int64_t* n_host) {
  CHECK_CTX(c);
  if (per_axis < 1) return set_error(MPMRB_E_INVALID, "per_axis must be >= 1");
  long long n = 0;
  int rc = launch_seed_box(*c, (const long long*)lo, (const long long*)hi, per_axis, jitter, h,
                           center, half, (const unsigned long long*)state4, x_out, cap, &n);
  *n_host = n;
  if (rc == MPMRB_E_CAPACITY) return set_error(rc, "seed_box: %lld points, capacity %lld", n, (long long)cap);
  if (rc) return rc;
  return c->check_status("seed_box");
}

int mpmrb_contact_velocities(mpmrb_ctx* c, const int64_t* nodes, const double* w,
                             const double* frames, const double* bias, int64_t nc,
                             const double* v_grid, double* vc) {
  CHECK_CTX(c);
  int rc = launch_contact_velocities(*c, (const long long*)nodes, w, frames, bias, nc, v_grid, vc);
  if (rc) return rc;
  return c->check_status("contact_velocities");
}

}  // extern "C"

// ------------------------------------------------------------------ solver

namespace mpmrb {
namespace {
__global__ void k_problem_layout(const long long* __restrict__ nodes, const double* __restrict__ w,
                                 long long nc, int* __restrict__ cnodes, double* __restrict__ cw) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nc * 27) return;
  long long c = e / 27, k = e % 27;
  // dead slots (w = 0, solver.py:207-213) carry no node
  cnodes[k * nc + c] = (w[e] == 0.0) ? -1 : (int)nodes[e];
  cw[k * nc + c] = w[e];
}
}  // namespace
}  // namespace mpmrb

static int qn_solve_impl(mpmrb_ctx* c, const mpmrb_problem* pr, const mpmrb_solver_params* sp,
                         const double* v0, const double* ext_free, double* v, double* gamma,
                         double* objective, double* residual, double* threshold, double* alpha,
                         double* p_host, mpmrb_solve_report* rep);

extern "C" int mpmrb_qn_solve(mpmrb_ctx* c, const mpmrb_problem* pr,
                              const mpmrb_solver_params* sp, const double* v0, double* v,
                              double* gamma, double* objective, double* residual,
                              double* threshold, double* alpha, mpmrb_solve_report* rep) {
  return qn_solve_impl(c, pr, sp, v0, nullptr, v, gamma, objective, residual, threshold, alpha,
                       nullptr, rep);
}

extern "C" int mpmrb_qn_solve_ext(mpmrb_ctx* c, const mpmrb_problem* pr,
                                  const mpmrb_solver_params* sp, const double* v0,
                                  const double* ext_free_host, double* v, double* gamma,
                                  double* objective, double* residual, double* threshold,
                                  double* alpha, double* p_host, mpmrb_solve_report* rep) {
  return qn_solve_impl(c, pr, sp, v0, ext_free_host, v, gamma, objective, residual, threshold,
                       alpha, p_host, rep);
}

static int qn_solve_impl(mpmrb_ctx* c, const mpmrb_problem* pr, const mpmrb_solver_params* sp,
                         const double* v0, const double* ext_free, double* v, double* gamma,
                         double* objective, double* residual, double* threshold, double* alpha,
                         double* p_host, mpmrb_solve_report* rep) {
  CHECK_CTX(c);
  long long nd = pr->n_nodes, nc = pr->n_contacts;
  long long ncc = nc > 0 ? nc : 1, ndd = nd > 0 ? nd : 1;
  int rc = 0;
  rc |= c->scratch[SS_SOLVER0].grow(4 * 27 * ncc);           // cnodes
  rc |= c->scratch[SS_SOLVER1].grow(8 * 27 * ncc);           // cw
  rc |= c->scratch[SS_SOLVER2].grow(8 * 3 * ndd);            // dv
  rc |= c->scratch[SS_SOLVER3].grow(8 * kCellSumStride * ncc);  // contact records
  rc |= c->scratch[SS_SOLVER4].grow(8 * 8 * ncc);            // vc, dvc, vhat, mug
  rc |= c->scratch[SS_SOLVER5].grow(8 * (2 * 8 * kMaxSolverCtas + 8));  // grid partials
  rc |= c->scratch[SS_SOLVER6].grow(4096);                   // sizes, SolveOut
  rc |= c->scratch[SS_SOLVER7].grow(4 * 14 * (ndd + 2) + 64);  // node adjacency ints
  rc |= c->scratch[SS_SOLVER8].grow(2 * 4 * 27 * ncc);       // adjacency entries + tmp
  rc |= c->scratch[SS_PROBLEM].grow(4 * 4 * (ncc + 2));      // contact groups
  rc |= c->scratch[SS_HOSTINFO].grow(kSolverSyncBytes);  // reduction slots, tags, barrier
  if (rc) return MPMRB_E_CUDA;
  char* misc = c->scratch[SS_SOLVER6].as<char>();
  int* sizes = (int*)(misc + 2048);
  SolveOut* so = (SolveOut*)(misc + 2304);
  MPMRB_CUDA_OK(cudaMemsetAsync(misc, 0, 4096, c->stream));
  int hs[2] = {(int)nd, (int)nc};
  MPMRB_CUDA_OK(cudaMemcpyAsync(sizes, hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  unsigned long long* slots = c->scratch[SS_HOSTINFO].as<unsigned long long>();
  unsigned* chan = reinterpret_cast<unsigned*>(slots + kSolverSlotWords);
  {
    MPMRB_CUDA_OK(cudaMemsetAsync(slots, 0, kSolverSyncBytes, c->stream));
    static const unsigned ch[4] = {1u, 1u, 1u, 0u};
    MPMRB_CUDA_OK(cudaMemcpyAsync(chan, ch, sizeof(ch), cudaMemcpyHostToDevice, c->stream));
  }
  if (nc > 0) {
    k_problem_layout<<<grid_for(nc * 27, 256), 256, 0, c->stream>>>(
        (const long long*)pr->nodes, pr->w, nc, c->scratch[SS_SOLVER0].as<int>(),
        c->scratch[SS_SOLVER1].as<double>());
    c->launches++;
  }
  SolverSetup su{};
  {
    int* ni = c->scratch[SS_SOLVER7].as<int>();
    su.cnt = ni;
    su.fill = ni + (ndd + 2);
    su.off = ni + 2 * (ndd + 2);
    su.flag = ni + 3 * (ndd + 2);
    su.flag_off = ni + 4 * (ndd + 2);
    su.cn = ni + 5 * (ndd + 2);
    su.fn = ni + 6 * (ndd + 2);
    su.counts = ni + 7 * (ndd + 2);
    su.cn_rec = reinterpret_cast<int4*>(ni + 8 * (ndd + 2));
    int* ci = c->scratch[SS_PROBLEM].as<int>();
    su.head = ci;
    su.head_off = ci + (ncc + 2);
    su.grp_of = ci + 2 * (ncc + 2);
    su.grp_start = ci + 3 * (ncc + 2);
    su.cnt_exp = ni + 12 * (ndd + 2);
    su.off_exp = ni + 13 * (ndd + 2);
    su.ent = c->scratch[SS_SOLVER8].as<int>();
    su.ent_tmp = su.ent + 27 * ncc;
  }
  rc = launch_solver_setup(*c, sizes, sizes + 1, nd, nc, c->scratch[SS_SOLVER0].as<int>(), su,
                           c->scratch[SS_TILE]);
  if (rc) return rc;
  SolverArgs a{};
  a.nd_dev = sizes;
  a.nc_dev = sizes + 1;
  a.nc_cap = nc;
  a.nd_cap = nd;
  a.su = su;
  a.prof = c->solver_prof;
  a.m = pr->m;
  a.v_star = pr->v_star;
  a.v0 = v0 ? v0 : pr->v_init;
  a.cnodes = c->scratch[SS_SOLVER0].as<int>();
  a.cw = c->scratch[SS_SOLVER1].as<double>();
  a.frames = pr->frames;
  a.bias = pr->bias;
  a.phi = pr->phi;
  a.mu = pr->mu;
  a.gamma_lag = pr->gamma_lag;
  a.K = pr->dt * (pr->dt + pr->tau_d) * pr->stiffness;  // contact_model.py:42-43
  a.den = pr->dt + pr->tau_d;
  a.eps_v = pr->eps_v;
  a.eps_a = sp->eps_a;
  a.eps_r = sp->eps_r;
  a.ls_tol = sp->ls_tol;
  a.max_iters = sp->max_iters;
  a.ls_max = sp->ls_max_iters;
  a.skip_if_no_contacts = 0;
  a.force_ctas = 0;
  a.v = v;
  a.dv = c->scratch[SS_SOLVER2].as<double>();
  a.cellsum = c->scratch[SS_SOLVER3].as<double>();
  a.vc = c->scratch[SS_SOLVER4].as<double>();
  a.dvc = a.vc + 3 * ncc;
  a.cvhat = a.vc + 6 * ncc;
  a.cmug = a.vc + 7 * ncc;
  a.partials = c->scratch[SS_SOLVER5].as<double>();
  a.slots = slots;
  a.chan = chan;
  a.bar = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(slots) + 8 * kSolverSlotWords + 64);
  a.gamma = gamma;
  a.tr_obj = objective;
  a.tr_res = residual;
  a.tr_thr = threshold;
  a.tr_alpha = alpha;
  a.out = so;
  a.act = nullptr;
  a.v_next_full = nullptr;
  const char* force = getenv("MPMRB_SOLVER_CTAS");
  if (force) a.force_ctas = atoi(force);
  const char* force_ls = getenv("MPMRB_SOLVER_LS_CTAS");
  if (force_ls) a.force_ls_ctas = atoi(force_ls);
  for (int k = 0; k < 3; ++k) a.ext_free[k] = ext_free ? ext_free[k] : 0.0;
  double* p_dev = reinterpret_cast<double*>(misc + 2304 + 256);  // after SolveOut
  a.p_out = p_dev;
  rc = launch_qn_solve(*c, a, 0);
  if (rc) return rc;
  SolveOut h{};
  MPMRB_CUDA_OK(cudaMemcpyAsync(&h, so, sizeof(SolveOut), cudaMemcpyDeviceToHost, c->stream));
  if (p_host)
    MPMRB_CUDA_OK(cudaMemcpyAsync(p_host, p_dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  rc = c->check_status("quasi_newton_solve");
  if (rc) return rc;
  rep->converged = h.converged;
  rep->iterations = h.iterations;
  rep->ls_evals = h.ls_evals;
  rep->regularized = h.regularized;
  rep->status = h.status;
  if (h.status == MPMRB_E_NOT_DESCENT)
    return set_error(MPMRB_E_NOT_DESCENT, "line search needs a descent direction");
  if (h.status == MPMRB_E_NONFINITE)
    return set_error(MPMRB_E_NONFINITE, "Hessian block not SPD after regularization");
  if (h.status_flags & 1)
    return set_error(MPMRB_E_NONFINITE, "contact solve produced non-finite velocities");
  return MPMRB_OK;
}

// ------------------------------------------------------------------ sim

extern "C" {

int mpmrb_sim_create(mpmrb_ctx* c, mpmrb_sim** out) {
  CHECK_CTX(c);
  mpmrb_sim* s = new (std::nothrow) mpmrb_sim();
  if (!s) return set_error(MPMRB_E_INVALID, "out of host memory");
  s->ctx = c;
  if (getenv("MPMRB_NO_GRAPH")) s->use_graph = false;
  const char* force = getenv("MPMRB_SOLVER_CTAS");
  if (force) s->force_ctas = atoi(force);
  const char* force_ls = getenv("MPMRB_SOLVER_LS_CTAS");
  if (force_ls) s->force_ls_ctas = atoi(force_ls);
  *out = s;
  return MPMRB_OK;
}

int mpmrb_sim_destroy(mpmrb_sim* s) {
  if (!s) return MPMRB_OK;
  cudaStreamSynchronize(s->ctx->stream);
  // every DevBuf member frees itself (DevBuf::~DevBuf)
  delete s;
  return MPMRB_OK;
}

int mpmrb_sim_set_particles(mpmrb_sim* s, const mpmrb_particles* p) {
  if (!s || !p) return set_error(MPMRB_E_INVALID, "null argument");
  ParticlesDev np = particles_dev(p);
  if (std::memcmp(&np, &s->p, sizeof(np)) != 0) s->invalidate();
  s->p = np;
  s->have_particles = true;
  return MPMRB_OK;
}

int mpmrb_sim_set_cloth(mpmrb_sim* s, int64_t ne, const int32_t* tri, const int32_t* epart,
                        const double* dm_inv, const double* vol, double* d3,
                        const int8_t* role) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  if (ne < 0) return set_error(MPMRB_E_INVALID, "negative element count");
  if (ne > 0 && !(tri && epart && dm_inv && vol && d3 && role))
    return set_error(MPMRB_E_INVALID, "cloth arrays must be non-null");
  const bool changed = (ne > 0) != (s->cloth.ne > 0) || s->cloth.tri != tri ||
                       s->cloth.epart != epart || s->cloth.dm_inv != dm_inv ||
                       s->cloth.vol != vol || s->cloth.d3 != d3 || s->cloth.ne != ne ||
                       s->cloth_role_user != (const signed char*)role;
  s->cloth.ne = ne;
  s->cloth.tri = tri;
  s->cloth.epart = epart;
  s->cloth.dm_inv = dm_inv;
  s->cloth.vol = vol;
  s->cloth.d3 = d3;
  s->cloth_role_user = (const signed char*)role;
  if (changed) s->invalidate();
  return MPMRB_OK;
}

int mpmrb_sim_set_materials(mpmrb_sim* s, const mpmrb_material* mats, int32_t n) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  if (s->b_mats.grow(sizeof(mpmrb_material) * (n > 0 ? n : 1))) return MPMRB_E_CUDA;
  if (n > 0)
    MPMRB_CUDA_OK(cudaMemcpyAsync(s->b_mats.p, mats, sizeof(mpmrb_material) * n,
                                  cudaMemcpyHostToDevice, s->ctx->stream));
  if (n != s->nmat) s->invalidate();
  s->nmat = n;
  return MPMRB_OK;
}

int mpmrb_sim_set_geoms(mpmrb_sim* s, const mpmrb_geom* geoms, int32_t n, int32_t nbody) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  if (nbody > 32) return set_error(MPMRB_E_INVALID, "at most 32 bodies in the fused path");
  void* old = s->b_geoms.p;
  if (s->b_geoms.grow(sizeof(mpmrb_geom) * (n > 0 ? n : 1))) return MPMRB_E_CUDA;
  if (old != s->b_geoms.p || n != s->ngeom || nbody != s->nbody) s->invalidate();
  if (n > 0)
    MPMRB_CUDA_OK(cudaMemcpyAsync(s->b_geoms.p, geoms, sizeof(mpmrb_geom) * n,
                                  cudaMemcpyHostToDevice, s->ctx->stream));
  s->ngeom = n;
  s->nbody = nbody;
  return MPMRB_OK;
}

int mpmrb_sim_set_params(mpmrb_sim* s, double h, double dt_s, const double* g, double k,
                         double tau_d, double eps_v, double margin,
                         const mpmrb_solver_params* sp) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  double K = dt_s * (dt_s + tau_d) * k;
  bool same = s->have_params && s->h == h && s->dt_s == dt_s && s->gravity[0] == g[0] &&
              s->gravity[1] == g[1] && s->gravity[2] == g[2] && s->K == K &&
              s->den == dt_s + tau_d && s->eps_v == eps_v && s->margin == margin &&
              std::memcmp(&s->sp, sp, sizeof(*sp)) == 0;
  if (!same) s->invalidate();
  s->h = h;
  s->dt_s = dt_s;
  s->gravity[0] = g[0];
  s->gravity[1] = g[1];
  s->gravity[2] = g[2];
  s->K = K;
  s->den = dt_s + tau_d;
  s->eps_v = eps_v;
  s->margin = margin;
  s->sp = *sp;
  s->have_params = true;
  return MPMRB_OK;
}

int mpmrb_sim_set_precision(mpmrb_sim* s, int32_t prec) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  if (prec != MPMRB_PREC_F64 && prec != MPMRB_PREC_F32)
    return set_error(MPMRB_E_INVALID, "precision must be MPMRB_PREC_F64 or MPMRB_PREC_F32");
  if (prec != s->prec) {
    s->invalidate();
    s->n_particles = -1;  // re-lay the internal particle copy in reserve()
  }
  s->prec = prec;
  return MPMRB_OK;
}

int mpmrb_sim_begin_step(mpmrb_sim* s, int64_t epoch, int32_t n_substeps) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  return s->begin_step(epoch, n_substeps);
}

int mpmrb_sim_substep(mpmrb_sim* s) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  return s->substep();
}

int mpmrb_sim_substep_part(mpmrb_sim* s, int32_t part) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  return s->substep_part(part);
}

int mpmrb_sim_get_views(mpmrb_sim* s, mpmrb_sim_views* v) {
  if (!s || !v) return set_error(MPMRB_E_INVALID, "null sim or views");
  int hc[3] = {0, 0, 0};
  MPMRB_CUDA_OK(cudaStreamSynchronize(s->ctx->stream));
  MPMRB_CUDA_OK(cudaMemcpy(hc, s->b_counters.p, sizeof(hc), cudaMemcpyDeviceToHost));
  const long long N = s->nb_cap * kNodesPerBlock;
  const long long cap = s->nc_cap;
  v->n_blocks = hc[0];
  v->n_active = hc[1];
  v->n_contacts = hc[2] < cap ? hc[2] : cap;
  v->nc_cap = cap;
  v->block_keys = (const int64_t*)s->b_bkeys.p;
  v->mass = s->b_mass.as<double>();
  v->mom_apic = s->b_mom.as<double>();
  v->mom_force = s->b_mom.as<double>() + 3 * N;
  v->v_star = s->b_vstar.as<double>();
  v->v_k = s->b_vk.as<double>();
  v->v_next = s->b_vnext.as<double>();
  v->act = s->b_act.as<int>();
  v->m_act = s->b_mc.as<double>();
  v->v_star_act = s->b_vstarc.as<double>();
  v->v_k_act = s->b_vkc.as<double>();
  v->cnodes = s->b_cnodes.as<int>();
  v->cw = s->b_cw.as<double>();
  v->frames = s->b_cframes.as<double>();
  v->bias = s->b_cbias.as<double>();
  v->phi = s->b_cphi.as<double>();
  v->mu = s->b_cmu.as<double>();
  v->gamma_lag = s->b_cgl.as<double>();
  v->gamma = s->b_gamma.as<double>();
  return MPMRB_OK;
}

int mpmrb_sim_set_solve_result(mpmrb_sim* s, const mpmrb_solve_report* r) {
  if (!s || !r) return set_error(MPMRB_E_INVALID, "null sim or report");
  return s->set_solve_result(r->converged, r->iterations, r->ls_evals, r->regularized);
}

int mpmrb_sim_end_step(mpmrb_sim* s, mpmrb_step_stats* st, double* impulses) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  int rc = s->end_step(st, impulses);
  if (rc) return rc;
  if (st->status)
    return set_error(st->status, "advance_step: %s (site %d, index %lld)",
                     st->status == MPMRB_E_DIVERGED ? "SimulationDiverged" : "device error",
                     st->status_detail, (long long)st->status_aux);
  return MPMRB_OK;
}

double mpmrb_sim_staleness(mpmrb_sim* s) { return s ? s->staleness : 0.0; }

int mpmrb_sim_profile_substep(mpmrb_sim* s, float* stage_ms_host, int32_t* sizes_host) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  return s->profile_substep(stage_ms_host, sizes_host);
}

int mpmrb_sim_last_grid(mpmrb_sim* s, int64_t* nb, const int64_t** block_keys,
                        const double** mass, const double** v_star, const double** v_next) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  int hb = 0;
  MPMRB_CUDA_OK(cudaStreamSynchronize(s->ctx->stream));
  MPMRB_CUDA_OK(cudaMemcpy(&hb, s->b_counters.p, 4, cudaMemcpyDeviceToHost));
  *nb = hb;
  *block_keys = (const int64_t*)s->b_bkeys.p;
  *mass = (const double*)s->b_mass.p;
  *v_star = (const double*)s->b_vstar.p;
  *v_next = (const double*)s->b_vnext.p;
  return MPMRB_OK;
}

int mpmrb_sim_last_contacts(mpmrb_sim* s, int64_t* n, const int32_t** particle,
                            const double** gamma_world) {
  if (!s) return set_error(MPMRB_E_INVALID, "null sim");
  int hc[3] = {0, 0, 0};
  MPMRB_CUDA_OK(cudaStreamSynchronize(s->ctx->stream));
  MPMRB_CUDA_OK(cudaMemcpy(hc, s->b_counters.p, sizeof(hc), cudaMemcpyDeviceToHost));
  *n = hc[2];
  // contacts index the sim-internal (sorted) particles: map to the user's ids
  long long cap = s->nc_cap;
  if (hc[2] > 0) {
    int rc = launch_map_ids(*s->ctx, s->b_cpart.as<int>(), s->b_perm.as<int>(),
                            s->b_counters.as<int>() + 2, cap, s->b_cpart_user.as<int>());
    if (rc) return rc;
    MPMRB_CUDA_OK(cudaStreamSynchronize(s->ctx->stream));
  }
  *particle = (const int32_t*)s->b_cpart_user.p;
  *gamma_world = (const double*)s->b_gworld.p;
  return MPMRB_OK;
}

}  // extern "C"
