// 3x3 decompositions used per particle, in the particle arithmetic type T
// (double: the reference's float64; float: the fp32 performance mode):
//  * Higham polar rotation (materials.py:70-83): R <- (R + R^-T)/2, <= 30
//    iterations, stop when max|dR| <= 1e-13 (float64).  The reference tests
//    the maximum over the whole batch; per particle the extra iterations a
//    batch would add change R only at roundoff (quadratic convergence).  In
//    float32 the iteration stalls at roundoff near 1e-7, so the per-particle
//    stop is max|dR| <= 1e-6 (Tol<float>).
//  * signed SVD (materials.py:95-106 conventions): one-sided Jacobi on F
//    (no squaring of the condition number), singular values sorted
//    descending like LAPACK, then det-corrected so U, V are rotations and the
//    last singular value carries the sign.
#pragma once

#include "common.cuh"

namespace mpmrb {

// Tolerances per arithmetic type.
template <class T>
struct Tol;
template <>
struct Tol<double> {
  static constexpr double polar = 1e-13;   // materials.py:79
  static constexpr double jacobi = 1e-15;  // off-diagonal / sqrt(alpha beta) to skip a rotation
  static constexpr double rank = 1e-14;    // s_j / s_0 below which U's column j is completed
  static constexpr double tiny = 1e-300;
};
template <>
struct Tol<float> {
  static constexpr float polar = 1e-6f;
  static constexpr float jacobi = 1e-7f;
  static constexpr float rank = 1e-6f;
  static constexpr float tiny = 1e-30f;
};

template <class T>
__device__ __forceinline__ M3T<T> polar_rotation(const M3T<T>& f) {
  M3T<T> r = f;
  for (int it = 0; it < 30; ++it) {
    M3T<T> it_t = m3_inv_transpose(r);
    T delta = T(0);
    M3T<T> nx;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      nx.a[i] = T(0.5) * (r.a[i] + it_t.a[i]);
      delta = fmax(delta, fabs(nx.a[i] - r.a[i]));
    }
    r = nx;
    if (delta <= Tol<T>::polar) break;
  }
  return r;
}

// Kirchhoff stress of fixed-corotated elasticity (materials.py:113-122)
template <class T>
__device__ __forceinline__ M3T<T> kirchhoff_fixed_corotated(const M3T<T>& f, T mu, T lam) {
  M3T<T> r = polar_rotation(f);
  T j = m3_det(f);
  M3T<T> d;
#pragma unroll
  for (int i = 0; i < 9; ++i) d.a[i] = f.a[i] - r.a[i];
  M3T<T> t = m3_mul_bt(d, f);
  T two_mu = T(2) * mu;
  T iso = lam * (j - T(1)) * j;
#pragma unroll
  for (int i = 0; i < 9; ++i) t.a[i] = two_mu * t.a[i];
  t(0, 0) += iso;
  t(1, 1) += iso;
  t(2, 2) += iso;
  return t;
}

template <class T>
struct SVD3T {
  M3T<T> u, v;  // F = U diag(s) V^T
  T s[3];
};
using SVD3 = SVD3T<double>;

template <class T>
__device__ __forceinline__ void jacobi_rotate_cols(M3T<T>& a, M3T<T>& v, int p, int q,
                                                   bool& rotated) {
  T alpha = a(0, p) * a(0, p) + a(1, p) * a(1, p) + a(2, p) * a(2, p);
  T beta = a(0, q) * a(0, q) + a(1, q) * a(1, q) + a(2, q) * a(2, q);
  T gamma = a(0, p) * a(0, q) + a(1, p) * a(1, q) + a(2, p) * a(2, q);
  // skip when |gamma| <= tol sqrt(alpha beta), compared squared (no sqrt)
  if (gamma == T(0) || gamma * gamma <= (Tol<T>::jacobi * Tol<T>::jacobi) * (alpha * beta)) return;
  // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)) with zeta = (beta - alpha) /
  // (2 gamma), rewritten with d = beta - alpha, e = 2 gamma as
  // t = sign(d) e / (|d| + sqrt(d^2 + e^2)): one square root and one division
  // (was two and three), then c = 1 / sqrt(1 + t^2) as one rsqrt
  const T d = beta - alpha, e = T(2) * gamma;
  T t = copysign(T(1), d) * e / (fabs(d) + sqrt(d * d + e * e));
  T c = rsqrt(T(1) + t * t);
  T s = c * t;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T ap = a(i, p), aq = a(i, q);
    a(i, p) = c * ap - s * aq;
    a(i, q) = s * ap + c * aq;
    T vp = v(i, p), vq = v(i, q);
    v(i, p) = c * vp - s * vq;
    v(i, q) = s * vp + c * vq;
  }
  rotated = true;
}

template <class T>
__device__ __forceinline__ void swap_cols(M3T<T>& m, int i, int j) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    T t = m(r, i);
    m(r, i) = m(r, j);
    m(r, j) = t;
  }
}

template <class T>
__device__ __forceinline__ void cross3(const T* a, const T* b, T* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// Signed SVD: U, V proper rotations; s[0] >= s[1] >= |s[2]|, s[2] may be < 0.
template <class T>
__device__ __forceinline__ SVD3T<T> signed_svd(const M3T<T>& f) {
  SVD3T<T> out;
  M3T<T> a = f;
  M3T<T> v = m3_identity<T>();
  for (int sweep = 0; sweep < 20; ++sweep) {
    bool rot = false;
    jacobi_rotate_cols(a, v, 0, 1, rot);
    jacobi_rotate_cols(a, v, 0, 2, rot);
    jacobi_rotate_cols(a, v, 1, 2, rot);
    if (!rot) break;
  }
  T s[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) s[j] = sqrt(a(0, j) * a(0, j) + a(1, j) * a(1, j) + a(2, j) * a(2, j));
  // sort descending (columns of a and v follow)
  if (s[0] < s[1]) { T t = s[0]; s[0] = s[1]; s[1] = t; swap_cols(a, 0, 1); swap_cols(v, 0, 1); }
  if (s[0] < s[2]) { T t = s[0]; s[0] = s[2]; s[2] = t; swap_cols(a, 0, 2); swap_cols(v, 0, 2); }
  if (s[1] < s[2]) { T t = s[1]; s[1] = s[2]; s[2] = t; swap_cols(a, 1, 2); swap_cols(v, 1, 2); }
  // U columns = a_j / s_j, completing a basis where s_j vanishes
  M3T<T> u;
  const T tiny = Tol<T>::tiny;
  T c0[3], c1[3], c2[3];
  if (s[0] > tiny) {
    const T inv = T(1) / s[0];
    for (int i = 0; i < 3; ++i) c0[i] = a(i, 0) * inv;
  } else {
    c0[0] = T(1); c0[1] = T(0); c0[2] = T(0);
  }
  if (s[1] > tiny * fmax(T(1), s[0]) && s[1] > Tol<T>::rank * s[0]) {
    const T inv = T(1) / s[1];
    for (int i = 0; i < 3; ++i) c1[i] = a(i, 1) * inv;
    // re-orthogonalise against c0
    T d = c1[0] * c0[0] + c1[1] * c0[1] + c1[2] * c0[2];
    for (int i = 0; i < 3; ++i) c1[i] -= d * c0[i];
    const T rn = rsqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] *= rn;
  } else {
    // any unit vector orthogonal to c0
    int k = (fabs(c0[0]) <= fabs(c0[1]) && fabs(c0[0]) <= fabs(c0[2])) ? 0
            : (fabs(c0[1]) <= fabs(c0[2]) ? 1 : 2);
    T e[3] = {T(0), T(0), T(0)};
    e[k] = T(1);
    T d = e[0] * c0[0] + e[1] * c0[1] + e[2] * c0[2];
    for (int i = 0; i < 3; ++i) c1[i] = e[i] - d * c0[i];
    const T rn = rsqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] *= rn;
  }
  if (s[2] > Tol<T>::rank * fmax(s[0], tiny)) {
    const T inv = T(1) / s[2];
    for (int i = 0; i < 3; ++i) c2[i] = a(i, 2) * inv;
    T d0 = c2[0] * c0[0] + c2[1] * c0[1] + c2[2] * c0[2];
    T d1 = c2[0] * c1[0] + c2[1] * c1[1] + c2[2] * c1[2];
    for (int i = 0; i < 3; ++i) c2[i] -= d0 * c0[i] + d1 * c1[i];
    const T rn = rsqrt(c2[0] * c2[0] + c2[1] * c2[1] + c2[2] * c2[2]);
    for (int i = 0; i < 3; ++i) c2[i] *= rn;
  } else {
    cross3(c0, c1, c2);
  }
  for (int i = 0; i < 3; ++i) {
    u(i, 0) = c0[i];
    u(i, 1) = c1[i];
    u(i, 2) = c2[i];
  }
  // det corrections (materials.py:101-106)
  if (m3_det(u) < T(0)) {
    for (int i = 0; i < 3; ++i) u(i, 2) = -u(i, 2);
    s[2] = -s[2];
  }
  if (m3_det(v) < T(0)) {
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
template <class T>
__device__ __forceinline__ M3T<T> svd_compose(const M3T<T>& u, const T* d, const M3T<T>& v) {
  M3T<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r(i, j) = u(i, 0) * d[0] * v(j, 0) + u(i, 1) * d[1] * v(j, 1) + u(i, 2) * d[2] * v(j, 2);
  return r;
}

// materials.py:86-110 clamp of one inverted / non-finite F (caller tests badness)
template <class T>
__device__ __forceinline__ M3T<T> clamp_singular_values(const M3T<T>& f_in) {
  M3T<T> f;
#pragma unroll
  for (int i = 0; i < 9; ++i) f.a[i] = isfinite(f_in.a[i]) ? f_in.a[i] : T(0);  // nan_to_num
  SVD3T<T> d = signed_svd(f);
  const T fl = T(kSigmaFloor);
  T s[3] = {fmax(d.s[0], fl), fmax(d.s[1], fl), fmax(d.s[2], fl)};
  return svd_compose(d.u, s, d.v);
}

// Hencky St.Venant-Kirchhoff Kirchhoff stress (sand; oracle/plasticity.py)
template <class T>
__device__ __forceinline__ M3T<T> kirchhoff_hencky(const M3T<T>& f, T mu, T lam) {
  SVD3T<T> d = signed_svd(f);
  T e[3], tr = T(0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = log(fmax(d.s[i], T(1e-12)));
    tr += e[i];
  }
  T dd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) dd[i] = T(2) * mu * e[i] + lam * tr;
  return svd_compose(d.u, dd, d.u);
}

// Drucker-Prager return map on the singular values (oracle/plasticity.py:
// project).  Writes the plastic increment |e - e_proj| to *dq and, when tau
// is given, the Hencky Kirchhoff stress of the projected F (same SVD: U
// diag(2 mu eps + lam tr eps) U^T), cached for the next substep's P2G
// instead of a second SVD there.
template <class T>
__device__ __forceinline__ M3T<T> dp_return_map_tau(const M3T<T>& f, T mu, T lam, T alpha,
                                                    T* dq, M3T<T>* tau) {
  SVD3T<T> d = signed_svd(f);
  T e[3], tr = T(0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = log(fmax(d.s[i], T(1e-12)));
    tr += e[i];
  }
  T eh[3], en2 = T(0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    eh[i] = e[i] - tr / T(3);
    en2 += eh[i] * eh[i];
  }
  T en = sqrt(en2);
  T dgam = en + (T(3) * lam + T(2) * mu) / (T(2) * mu) * tr * alpha;
  T out[3];
  if (tr > T(0)) {
    out[0] = out[1] = out[2] = T(0);  // tip (tension)
  } else if (dgam > T(0) && en > T(0)) {
    T k = dgam / en;
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] = e[i] - k * eh[i];
  } else {
    *dq = T(0);
    if (tau) {
      T tr_e = e[0] + e[1] + e[2], dd[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) dd[i] = T(2) * mu * e[i] + lam * tr_e;
      *tau = svd_compose(d.u, dd, d.u);
    }
    return f;
  }
  if (tau) {
    T tr_o = out[0] + out[1] + out[2], dd[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dd[i] = T(2) * mu * out[i] + lam * tr_o;
    *tau = svd_compose(d.u, dd, d.u);
  }
  T q2 = T(0), sig[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    q2 += (e[i] - out[i]) * (e[i] - out[i]);
    sig[i] = exp(out[i]);
  }
  *dq = sqrt(q2);
  return svd_compose(d.u, sig, d.v);
}

template <class T>
__device__ __forceinline__ M3T<T> dp_return_map(const M3T<T>& f, T mu, T lam, T alpha, T* dq) {
  return dp_return_map_tau<T>(f, mu, lam, alpha, dq, nullptr);
}

}  // namespace mpmrb
