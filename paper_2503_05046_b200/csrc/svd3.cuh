// 3x3 float64 decompositions used per particle:
//  * Higham polar rotation (materials.py:70-83): R <- (R + R^-T)/2, <= 30
//    iterations, stop when max|dR| <= 1e-13.  The reference tests the
//    maximum over the whole batch; per particle the extra iterations a batch
//    would add change R only at roundoff (quadratic convergence).
//  * signed SVD (materials.py:95-106 conventions): one-sided Jacobi on F
//    (no squaring of the condition number), singular values sorted
//    descending like LAPACK, then det-corrected so U, V are rotations and the
//    last singular value carries the sign.
#pragma once

#include "common.cuh"

namespace mpmrb {

__device__ __forceinline__ M3 polar_rotation(const M3& f) {
  M3 r = f;
  for (int it = 0; it < 30; ++it) {
    M3 it_t = m3_inv_transpose(r);
    double delta = 0.0;
    M3 nx;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      nx.a[i] = 0.5 * (r.a[i] + it_t.a[i]);
      delta = fmax(delta, fabs(nx.a[i] - r.a[i]));
    }
    r = nx;
    if (delta <= 1e-13) break;
  }
  return r;
}

// Kirchhoff stress of fixed-corotated elasticity (materials.py:113-122)
__device__ __forceinline__ M3 kirchhoff_fixed_corotated(const M3& f, double mu, double lam) {
  M3 r = polar_rotation(f);
  double j = m3_det(f);
  M3 d;
#pragma unroll
  for (int i = 0; i < 9; ++i) d.a[i] = f.a[i] - r.a[i];
  M3 t = m3_mul_bt(d, f);
  double two_mu = 2.0 * mu;
  double iso = lam * (j - 1.0) * j;
#pragma unroll
  for (int i = 0; i < 9; ++i) t.a[i] = two_mu * t.a[i];
  t(0, 0) += iso;
  t(1, 1) += iso;
  t(2, 2) += iso;
  return t;
}

struct SVD3 {
  M3 u, v;      // F = U diag(s) V^T
  double s[3];
};

__device__ __forceinline__ void jacobi_rotate_cols(M3& a, M3& v, int p, int q, bool& rotated) {
  double alpha = a(0, p) * a(0, p) + a(1, p) * a(1, p) + a(2, p) * a(2, p);
  double beta = a(0, q) * a(0, q) + a(1, q) * a(1, q) + a(2, q) * a(2, q);
  double gamma = a(0, p) * a(0, q) + a(1, p) * a(1, q) + a(2, p) * a(2, q);
  if (gamma == 0.0 || fabs(gamma) <= 1e-15 * sqrt(alpha * beta)) return;
  double zeta = (beta - alpha) / (2.0 * gamma);
  double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = c * t;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double ap = a(i, p), aq = a(i, q);
    a(i, p) = c * ap - s * aq;
    a(i, q) = s * ap + c * aq;
    double vp = v(i, p), vq = v(i, q);
    v(i, p) = c * vp - s * vq;
    v(i, q) = s * vp + c * vq;
  }
  rotated = true;
}

__device__ __forceinline__ void swap_cols(M3& m, int i, int j) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double t = m(r, i);
    m(r, i) = m(r, j);
    m(r, j) = t;
  }
}

__device__ __forceinline__ void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// Signed SVD: U, V proper rotations; s[0] >= s[1] >= |s[2]|, s[2] may be < 0.
__device__ __forceinline__ SVD3 signed_svd(const M3& f) {
  SVD3 out;
  M3 a = f;
  M3 v = m3_identity();
  for (int sweep = 0; sweep < 20; ++sweep) {
    bool rot = false;
    jacobi_rotate_cols(a, v, 0, 1, rot);
    jacobi_rotate_cols(a, v, 0, 2, rot);
    jacobi_rotate_cols(a, v, 1, 2, rot);
    if (!rot) break;
  }
  double s[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) s[j] = sqrt(a(0, j) * a(0, j) + a(1, j) * a(1, j) + a(2, j) * a(2, j));
  // sort descending (columns of a and v follow)
  if (s[0] < s[1]) { double t = s[0]; s[0] = s[1]; s[1] = t; swap_cols(a, 0, 1); swap_cols(v, 0, 1); }
  if (s[0] < s[2]) { double t = s[0]; s[0] = s[2]; s[2] = t; swap_cols(a, 0, 2); swap_cols(v, 0, 2); }
  if (s[1] < s[2]) { double t = s[1]; s[1] = s[2]; s[2] = t; swap_cols(a, 1, 2); swap_cols(v, 1, 2); }
  // U columns = a_j / s_j, completing a basis where s_j vanishes
  M3 u;
  const double tiny = 1e-300;
  double c0[3], c1[3], c2[3];
  if (s[0] > tiny) {
    for (int i = 0; i < 3; ++i) c0[i] = a(i, 0) / s[0];
  } else {
    c0[0] = 1.0; c0[1] = 0.0; c0[2] = 0.0;
  }
  if (s[1] > tiny * fmax(1.0, s[0]) && s[1] > 1e-14 * s[0]) {
    for (int i = 0; i < 3; ++i) c1[i] = a(i, 1) / s[1];
    // re-orthogonalise against c0
    double d = c1[0] * c0[0] + c1[1] * c0[1] + c1[2] * c0[2];
    for (int i = 0; i < 3; ++i) c1[i] -= d * c0[i];
    double nn = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] /= nn;
  } else {
    // any unit vector orthogonal to c0
    int k = (fabs(c0[0]) <= fabs(c0[1]) && fabs(c0[0]) <= fabs(c0[2])) ? 0
            : (fabs(c0[1]) <= fabs(c0[2]) ? 1 : 2);
    double e[3] = {0.0, 0.0, 0.0};
    e[k] = 1.0;
    double d = e[0] * c0[0] + e[1] * c0[1] + e[2] * c0[2];
    for (int i = 0; i < 3; ++i) c1[i] = e[i] - d * c0[i];
    double nn = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] /= nn;
  }
  if (s[2] > 1e-14 * fmax(s[0], tiny)) {
    for (int i = 0; i < 3; ++i) c2[i] = a(i, 2) / s[2];
    double d0 = c2[0] * c0[0] + c2[1] * c0[1] + c2[2] * c0[2];
    double d1 = c2[0] * c1[0] + c2[1] * c1[1] + c2[2] * c1[2];
    for (int i = 0; i < 3; ++i) c2[i] -= d0 * c0[i] + d1 * c1[i];
    double nn = sqrt(c2[0] * c2[0] + c2[1] * c2[1] + c2[2] * c2[2]);
    for (int i = 0; i < 3; ++i) c2[i] /= nn;
  } else {
    cross3(c0, c1, c2);
  }
  for (int i = 0; i < 3; ++i) {
    u(i, 0) = c0[i];
    u(i, 1) = c1[i];
    u(i, 2) = c2[i];
  }
  // det corrections (materials.py:101-106)
  if (m3_det(u) < 0.0) {
    for (int i = 0; i < 3; ++i) u(i, 2) = -u(i, 2);
    s[2] = -s[2];
  }
  if (m3_det(v) < 0.0) {
    for (int i = 0; i < 3; ++i) v(i, 2) = -v(i, 2);
    s[2] = -s[2];
  }
  out.u = u;
  out.v = v;
  out.s[0] = s[0];
  out.s[1] = s[1];
  out.s[2] = s[2];
  return out;
}

// U diag(d) V^T
__device__ __forceinline__ M3 svd_compose(const M3& u, const double* d, const M3& v) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r(i, j) = u(i, 0) * d[0] * v(j, 0) + u(i, 1) * d[1] * v(j, 1) + u(i, 2) * d[2] * v(j, 2);
  return r;
}

// materials.py:86-110 clamp of one inverted / non-finite F (caller tests badness)
__device__ __forceinline__ M3 clamp_singular_values(const M3& f_in) {
  M3 f;
#pragma unroll
  for (int i = 0; i < 9; ++i) f.a[i] = isfinite(f_in.a[i]) ? f_in.a[i] : 0.0;  // nan_to_num
  SVD3 d = signed_svd(f);
  double s[3] = {fmax(d.s[0], kSigmaFloor), fmax(d.s[1], kSigmaFloor), fmax(d.s[2], kSigmaFloor)};
  return svd_compose(d.u, s, d.v);
}

// Hencky St.Venant-Kirchhoff Kirchhoff stress (sand; oracle/plasticity.py)
__device__ __forceinline__ M3 kirchhoff_hencky(const M3& f, double mu, double lam) {
  SVD3 d = signed_svd(f);
  double e[3], tr = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = log(fmax(d.s[i], 1e-12));
    tr += e[i];
  }
  double dd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) dd[i] = 2.0 * mu * e[i] + lam * tr;
  return svd_compose(d.u, dd, d.u);
}

// Drucker-Prager return map on the singular values (oracle/plasticity.py:project)
__device__ __forceinline__ M3 dp_return_map(const M3& f, double mu, double lam, double alpha,
                                            double* dq) {
  SVD3 d = signed_svd(f);
  double e[3], tr = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = log(fmax(d.s[i], 1e-12));
    tr += e[i];
  }
  double eh[3], en2 = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    eh[i] = e[i] - tr / 3.0;
    en2 += eh[i] * eh[i];
  }
  double en = sqrt(en2);
  double dgam = en + (3.0 * lam + 2.0 * mu) / (2.0 * mu) * tr * alpha;
  double out[3];
  if (tr > 0.0) {
    out[0] = out[1] = out[2] = 0.0;  // tip (tension)
  } else if (dgam > 0.0 && en > 0.0) {
    double k = dgam / en;
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] = e[i] - k * eh[i];
  } else {
    *dq = 0.0;
    return f;
  }
  double q2 = 0.0, sig[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    q2 += (e[i] - out[i]) * (e[i] - out[i]);
    sig[i] = exp(out[i]);
  }
  *dq = sqrt(q2);
  return svd_compose(d.u, sig, d.v);
}

// Drucker-Prager return map that also returns the Hencky Kirchhoff stress of
// the projected F (same SVD: U diag(2 mu eps + lam tr eps) U^T), cached for
// the next substep's P2G instead of a second SVD there.
__device__ __forceinline__ M3 dp_return_map_tau(const M3& f, double mu, double lam,
                                                double alpha, double* dq, M3* tau) {
  SVD3 d = signed_svd(f);
  double e[3], tr = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = log(fmax(d.s[i], 1e-12));
    tr += e[i];
  }
  double eh[3], en2 = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    eh[i] = e[i] - tr / 3.0;
    en2 += eh[i] * eh[i];
  }
  double en = sqrt(en2);
  double dgam = en + (3.0 * lam + 2.0 * mu) / (2.0 * mu) * tr * alpha;
  double out[3];
  if (tr > 0.0) {
    out[0] = out[1] = out[2] = 0.0;  // tip (tension)
  } else if (dgam > 0.0 && en > 0.0) {
    double k = dgam / en;
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] = e[i] - k * eh[i];
  } else {
    *dq = 0.0;
    double tr_e = e[0] + e[1] + e[2], dd[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dd[i] = 2.0 * mu * e[i] + lam * tr_e;
    *tau = svd_compose(d.u, dd, d.u);
    return f;
  }
  {
    double tr_o = out[0] + out[1] + out[2], dd[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dd[i] = 2.0 * mu * out[i] + lam * tr_o;
    *tau = svd_compose(d.u, dd, d.u);
  }
  double q2 = 0.0, sig[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    q2 += (e[i] - out[i]) * (e[i] - out[i]);
    sig[i] = exp(out[i]);
  }
  *dq = sqrt(q2);
  return svd_compose(d.u, sig, d.v);
}

}  // namespace mpmrb
