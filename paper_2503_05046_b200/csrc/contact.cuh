// Device-side signed distances, frames and the contact model (float64).
#pragma once

#include "common.cuh"
#include "internal.h"

namespace mpmrb {

struct ContactArrays {
  int* particle;          // (cap,) int32 particle id (always written)
  long long* particle64;  // optional int64 copies for the API
  long long* body64;
  long long* geom64;
  int* body;              // optional int32 body id (fused path)
  double* phi;
  double* normal;
  double* witness;
  double* frames;
  double* bias;
  double* mu;
};

// world -> geom-local: local = (x - p_g) @ R_g  (collision.py:101)
__device__ __forceinline__ void to_local(const mpmrb_geom& g, const double* x, double* loc) {
  double r0 = x[0] - g.pos[0], r1 = x[1] - g.pos[1], r2 = x[2] - g.pos[2];
#pragma unroll
  for (int j = 0; j < 3; ++j) loc[j] = r0 * g.rot[j] + r1 * g.rot[3 + j] + r2 * g.rot[6 + j];
}
// local -> world direction: v @ R^T  (collision.py:106-107)
__device__ __forceinline__ void to_world_dir(const mpmrb_geom& g, const double* v, double* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = v[0] * g.rot[3 * i] + v[1] * g.rot[3 * i + 1] + v[2] * g.rot[3 * i + 2];
}

__device__ __forceinline__ double norm3(const double* v) {
  return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
}

// geometry.py:16-156, all in the geom-local frame
__device__ __forceinline__ void sdf_local(const mpmrb_geom& g, const double* p, double* phi,
                                          double* n, double* w) {
  switch (g.kind) {
    case MPMRB_GEOM_HALFSPACE: {
      const double* nn = g.params;
      double ph = (p[0] * nn[0] + p[1] * nn[1] + p[2] * nn[2]) - g.params[3];
      *phi = ph;
      for (int d = 0; d < 3; ++d) {
        n[d] = nn[d];
        w[d] = p[d] - ph * nn[d];
      }
      return;
    }
    case MPMRB_GEOM_SPHERE: {
      double r = g.params[0];
      double d = norm3(p);
      double sd = fmax(d, 1e-30);
      for (int k = 0; k < 3; ++k) n[k] = p[k] / sd;
      if (d < 1e-15) {
        n[0] = 0.0;
        n[1] = 0.0;
        n[2] = 1.0;
      }
      *phi = d - r;
      for (int k = 0; k < 3; ++k) w[k] = r * n[k];
      return;
    }
    case MPMRB_GEOM_BOX: {
      const double* he = g.params;
      double q[3];
      bool outside = false;
      for (int k = 0; k < 3; ++k) {
        q[k] = fabs(p[k]) - he[k];
        outside |= q[k] > 0.0;
        w[k] = fmin(fmax(p[k], -he[k]), he[k]);
      }
      if (outside) {
        double qo[3] = {fmax(q[0], 0.0), fmax(q[1], 0.0), fmax(q[2], 0.0)};
        double d = norm3(qo);
        *phi = d;
        for (int k = 0; k < 3; ++k) n[k] = (p[k] - w[k]) / d;
      } else {
        int ax = 0;
        if (q[1] > q[ax]) ax = 1;
        if (q[2] > q[ax]) ax = 2;  // argmax, first index on ties
        *phi = q[ax];
        double sg = (p[ax] >= 0.0) ? 1.0 : -1.0;
        for (int k = 0; k < 3; ++k) {
          n[k] = 0.0;
          w[k] = p[k];
        }
        n[ax] = sg;
        w[ax] = sg * he[ax];
      }
      return;
    }
    default: {  // capsule along local z
      double r = g.params[0], hl = g.params[1];
      double t = fmin(fmax(p[2], -hl), hl);
      double rel[3] = {p[0], p[1], p[2] - t};
      double d = norm3(rel);
      double sd = fmax(d, 1e-30);
      for (int k = 0; k < 3; ++k) n[k] = rel[k] / sd;
      if (d < 1e-15) {
        n[0] = 1.0;
        n[1] = 0.0;
        n[2] = 0.0;
      }
      *phi = d - r;
      w[0] = r * n[0];
      w[1] = r * n[1];
      w[2] = t + r * n[2];
      return;
    }
  }
}

// rows (t1, t2, n): seed = argmin |n_i| (first on ties), Gram-Schmidt, t2 = n x t1
__device__ __forceinline__ void contact_frame(const double* n, double* F) {
  double a0 = fabs(n[0]), a1 = fabs(n[1]), a2 = fabs(n[2]);
  int s = 0;
  if (a1 < a0) s = 1;
  if (a2 < (s == 0 ? a0 : a1)) s = 2;
  double e[3] = {0.0, 0.0, 0.0};
  e[s] = 1.0;
  double dot = e[0] * n[0] + e[1] * n[1] + e[2] * n[2];
  double t1[3] = {e[0] - dot * n[0], e[1] - dot * n[1], e[2] - dot * n[2]};
  double nn = norm3(t1);
  for (int k = 0; k < 3; ++k) t1[k] /= nn;
  double t2[3] = {n[1] * t1[2] - n[2] * t1[1], n[2] * t1[0] - n[0] * t1[2],
                  n[0] * t1[1] - n[1] * t1[0]};
  for (int k = 0; k < 3; ++k) {
    F[k] = t1[k];
    F[3 + k] = t2[k];
    F[6 + k] = n[k];
  }
}

// ------------------------------------------------------------ contact model
// contact_model.py:62-138 with K = dt(dt+tau_d)k and vhat = -phi/(dt+tau_d)
struct ContactModel {
  double K;        // impulse gain
  double den;      // dt + tau_d
  double eps_v;
};

__device__ __forceinline__ double cm_energy(const ContactModel& cm, const double* vc, double phi,
                                            double gl, double mu) {
  double vhat = -phi / cm.den;
  double gap = fmax(0.0, vhat - vc[2]);
  double s = sqrt(vc[0] * vc[0] + vc[1] * vc[1]);
  double hub = (s <= cm.eps_v) ? s * s / (2.0 * cm.eps_v) : s - 0.5 * cm.eps_v;
  return 0.5 * cm.K * gap * gap + mu * gl * hub;
}

__device__ __forceinline__ void cm_gradient(const ContactModel& cm, const double* vc, double phi,
                                            double gl, double mu, double* g) {
  double vhat = -phi / cm.den;
  g[2] = -(cm.K * fmax(0.0, vhat - vc[2]));
  double s = sqrt(vc[0] * vc[0] + vc[1] * vc[1]);
  double a = mu * gl / fmax(s, cm.eps_v);
  g[0] = a * vc[0];
  g[1] = a * vc[1];
}

// Hessian entries (G00, G11, G22, G01); G02 = G12 = 0.  Normal is active when
// v_n <= vhat (contact_model.py:98-100), same as gap >= 0 in the fused form.
__device__ __forceinline__ void cm_hessian(const ContactModel& cm, const double* vc, double phi,
                                           double gl, double mu, double* G) {
  double vhat = -phi / cm.den;
  G[2] = (vc[2] <= vhat) ? cm.K : 0.0;
  double s = sqrt(vc[0] * vc[0] + vc[1] * vc[1]);
  double a = mu * gl / fmax(s, cm.eps_v);
  double b = (s > cm.eps_v) ? a / fmax(s * s, cm.eps_v * cm.eps_v) : 0.0;
  G[0] = a - b * vc[0] * vc[0];
  G[1] = a - b * vc[1] * vc[1];
  G[3] = -b * vc[0] * vc[1];
}

// Fused gradient + Hessian (+ energy) with the per-solve constants
// vhat = -phi/(dt+tau_d) and mug = mu*gamma_lag precomputed: one sqrt and two
// divisions per evaluation (contact_model.py:114-138).  Same operation order
// as the separate functions above, so results are bitwise identical.
__device__ __forceinline__ double cm_eval(const ContactModel& cm, const double* vc, double vhat,
                                          double mug, double* g, double* G) {
  const double gap = vhat - vc[2];
  g[2] = -(cm.K * fmax(0.0, gap));
  G[2] = (gap >= 0.0) ? cm.K : 0.0;
  const double s = sqrt(vc[0] * vc[0] + vc[1] * vc[1]);
  const double a = mug / fmax(s, cm.eps_v);
  g[0] = a * vc[0];
  g[1] = a * vc[1];
  const double b = (s > cm.eps_v) ? a / fmax(s * s, cm.eps_v * cm.eps_v) : 0.0;
  G[0] = a - b * vc[0] * vc[0];
  G[1] = a - b * vc[1] * vc[1];
  G[3] = -b * vc[0] * vc[1];
  const double gp = fmax(0.0, gap);
  const double hub = (s <= cm.eps_v) ? s * s / (2.0 * cm.eps_v) : s - 0.5 * cm.eps_v;
  return 0.5 * cm.K * gp * gp + mug * hub;  // energy (contact_model.py:62-72)
}

int launch_detect(Ctx& c, const double* x, long long n, const mpmrb_geom* geoms_dev, int ngeom,
                  double margin, int* cnt, int* offs, int* total_dev, DevBuf& tiles,
                  long long cap, int* bias_stamp, double* bias_store,
                  const int* epoch_stamp_dev, const ContactArrays& ca);

}  // namespace mpmrb
