// Particle-vs-rigid-geometry contact detection on sm_100a.
//
// SDF primitives (geometry.py:16-156), contact frames (geometry.py:172-189),
// detect_contacts (collision.py:88-132) with the first-sight bias cache
// (collision.py:55-85) as per-(geom, particle) stamped slots, and
// contact_velocities (collision.py:135-143).  Contacts are produced in
// (particle, body, geom) order without a sort: each particle scans its geoms in
// (body, geom) order and an exclusive scan of per-particle counts places them.
#include "common.cuh"
#include "contact.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

__global__ void k_sdf_query(const mpmrb_geom* __restrict__ g, const double* __restrict__ pts,
                            long long n, double* __restrict__ phi, double* __restrict__ nrm,
                            double* __restrict__ wit) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  double ph, nn[3], ww[3];
  sdf_local(*g, p, &ph, nn, ww);
  phi[i] = ph;
  for (int d = 0; d < 3; ++d) {
    nrm[3 * i + d] = nn[d];
    wit[3 * i + d] = ww[d];
  }
}

__global__ void k_frames(const double* __restrict__ nrm, long long n, double* __restrict__ fr) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double nn[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
  double F[9];
  contact_frame(nn, F);
  for (int k = 0; k < 9; ++k) fr[9 * i + k] = F[k];
}

__global__ void k_contact_vel(const long long* __restrict__ nodes, const double* __restrict__ w,
                              const double* __restrict__ frames, const double* __restrict__ bias,
                              long long nc, const double* __restrict__ vg,
                              double* __restrict__ vc) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double vp[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 27; ++k) {
    long long nd = nodes[27 * c + k];
    double wk = w[27 * c + k];
    for (int d = 0; d < 3; ++d) vp[d] += wk * vg[3 * nd + d];
  }
  for (int r = 0; r < 3; ++r) {
    const double* R = frames + 9 * c + 3 * r;
    vc[3 * c + r] = (R[0] * vp[0] + R[1] * vp[1] + R[2] * vp[2]) + bias[3 * c + r];
  }
}

// The exact device contact-model functions the solver uses, exposed for parity
// (contact_model.py:62-111).  hess is (n,3,3).
__global__ void k_contact_model(const double* __restrict__ vc, const double* __restrict__ phi,
                                const double* __restrict__ gl, const double* __restrict__ mu,
                                long long n, ContactModel cm, double* __restrict__ energy,
                                double* __restrict__ grad, double* __restrict__ hess) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v[3] = {vc[3 * i], vc[3 * i + 1], vc[3 * i + 2]};
  if (energy) energy[i] = cm_energy(cm, v, phi[i], gl[i], mu[i]);
  if (grad) cm_gradient(cm, v, phi[i], gl[i], mu[i], grad + 3 * i);
  if (hess) {
    double G[4];
    cm_hessian(cm, v, phi[i], gl[i], mu[i], G);
    double* H = hess + 9 * i;
    H[0] = G[0];
    H[1] = G[3];
    H[2] = 0.0;
    H[3] = G[3];
    H[4] = G[1];
    H[5] = 0.0;
    H[6] = 0.0;
    H[7] = 0.0;
    H[8] = G[2];
  }
}

}  // namespace

int launch_contact_model(Ctx& c, const double* vc, const double* phi, const double* gl,
                         const double* mu, long long n, double K, double den, double eps_v,
                         double* energy, double* grad, double* hess) {
  if (n == 0) return MPMRB_OK;
  ContactModel cm{K, den, eps_v};
  k_contact_model<<<grid_for(n, 256), 256, 0, c.stream>>>(vc, phi, gl, mu, n, cm, energy, grad,
                                                           hess);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

// ---------------------------------------------------------------- shared kernels

__global__ void k_contact_count(const double* __restrict__ x, long long n,
                                const mpmrb_geom* __restrict__ geoms, int ngeom, double margin,
                                int* __restrict__ cnt) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  int c = 0;
  for (int g = 0; g < ngeom; ++g) {
    double loc[3], ph, nn[3], ww[3];
    to_local(geoms[g], p, loc);
    sdf_local(geoms[g], loc, &ph, nn, ww);
    c += (ph < margin) ? 1 : 0;
  }
  cnt[i] = c;
}

__global__ void k_contact_emit(const double* __restrict__ x, long long n,
                               const mpmrb_geom* __restrict__ geoms, int ngeom, double margin,
                               const int* __restrict__ cnt, const int* __restrict__ offs,
                               const int* __restrict__ total,
                               long long cap, int* __restrict__ bias_stamp,
                               double* __restrict__ bias_store, const int* __restrict__ epoch_dev,
                               ContactArrays ca, DevStatus* st) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 && *total > cap) raise_status(st, MPMRB_E_CAPACITY, 40, *total);
  if (cnt[i] == 0) return;  // most particles touch no geometry: skip the second SDF pass
  int o = offs[i];
  double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  for (int g = 0; g < ngeom; ++g) {
    const mpmrb_geom& G = geoms[g];
    double loc[3], ph, nl[3], wl[3];
    to_local(G, p, loc);
    sdf_local(G, loc, &ph, nl, wl);
    if (!(ph < margin)) continue;
    int slot = o++;
    if (slot >= cap) continue;
    double nw[3], ww[3];
    to_world_dir(G, nl, nw);
    to_world_dir(G, wl, ww);
    for (int d = 0; d < 3; ++d) ww[d] += G.pos[d];
    double F[9];
    contact_frame(nw, F);
    // rigid-point velocity at the witness in the contact frame (collision.py:112-115)
    double arm[3] = {ww[0] - G.body_pos[0], ww[1] - G.body_pos[1], ww[2] - G.body_pos[2]};
    const double* om = G.body_omega;
    double pv[3] = {G.body_v[0] + (om[1] * arm[2] - om[2] * arm[1]),
                    G.body_v[1] + (om[2] * arm[0] - om[0] * arm[2]),
                    G.body_v[2] + (om[0] * arm[1] - om[1] * arm[0])};
    double b[3];
    for (int r = 0; r < 3; ++r) b[r] = -(F[3 * r] * pv[0] + F[3 * r + 1] * pv[1] + F[3 * r + 2] * pv[2]);
    if (bias_stamp) {
      const int epoch_stamp = *epoch_dev;
      long long key = (long long)g * n + i;
      if (bias_stamp[key] == epoch_stamp) {
        for (int r = 0; r < 3; ++r) b[r] = bias_store[3 * key + r];
      } else {
        bias_stamp[key] = epoch_stamp;
        for (int r = 0; r < 3; ++r) bias_store[3 * key + r] = b[r];
      }
    }
    ca.particle[slot] = (int)i;
    if (ca.particle64) ca.particle64[slot] = i;
    if (ca.body64) ca.body64[slot] = G.body;
    if (ca.geom64) ca.geom64[slot] = G.geom;
    if (ca.body) ca.body[slot] = G.body;
    ca.phi[slot] = ph;
    ca.mu[slot] = G.mu;
    for (int d = 0; d < 3; ++d) {
      ca.normal[3 * slot + d] = nw[d];
      ca.witness[3 * slot + d] = ww[d];
      ca.bias[3 * slot + d] = b[d];
    }
    for (int k = 0; k < 9; ++k) ca.frames[9 * slot + k] = F[k];
  }
}

int launch_sdf_query(Ctx& c, const mpmrb_geom* g_dev, const double* pts, long long n, double* phi,
                     double* normal, double* witness) {
  if (n == 0) return MPMRB_OK;
  k_sdf_query<<<grid_for(n, 256), 256, 0, c.stream>>>(g_dev, pts, n, phi, normal, witness);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_frames(Ctx& c, const double* normals, long long n, double* frames) {
  if (n == 0) return MPMRB_OK;
  k_frames<<<grid_for(n, 256), 256, 0, c.stream>>>(normals, n, frames);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_contact_velocities(Ctx& c, const long long* nodes, const double* w,
                              const double* frames, const double* bias, long long nc,
                              const double* v_grid, double* vc) {
  if (nc == 0) return MPMRB_OK;
  k_contact_vel<<<grid_for(nc, 256), 256, 0, c.stream>>>(nodes, w, frames, bias, nc, v_grid, vc);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_detect(Ctx& c, const double* x, long long n, const mpmrb_geom* geoms_dev, int ngeom,
                  double margin, int* cnt, int* offs, int* total_dev, DevBuf& tiles,
                  long long cap, int* bias_stamp, double* bias_store, const int* epoch_stamp_dev,
                  const ContactArrays& ca) {
  if (n == 0 || ngeom == 0) {
    MPMRB_CUDA_OK(cudaMemsetAsync(total_dev, 0, sizeof(int), c.stream));
    return MPMRB_OK;
  }
  k_contact_count<<<grid_for(n, 128), 128, 0, c.stream>>>(x, n, geoms_dev, ngeom, margin, cnt);
  c.launches++;
  int rc = scan_exclusive_i32(c, cnt, offs, n, nullptr, total_dev, tiles);
  if (rc) return rc;
  k_contact_emit<<<grid_for(n, 128), 128, 0, c.stream>>>(x, n, geoms_dev, ngeom, margin, cnt,
                                                         offs, total_dev, cap, bias_stamp, bias_store,
                                                         epoch_stamp_dev, ca, c.status);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace mpmrb
