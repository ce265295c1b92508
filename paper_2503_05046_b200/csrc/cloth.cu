// Codimensional cloth on sm_100a (Jiang, Gast, Teran 2017; the paper's cloth
// model).  Parity unpinned: the reference has no cloth; the
// float64 NumPy statement is oracle/cloth.py (forces FD-checked).
//
//  * k_cloth_forces (before P2G): per triangle, F = [d1 d2 d3] diag(Dm^-1, 1)
//    from the vertex particles and the element's transverse direction d3;
//    Gram-Schmidt QR; P = Q C R^-T with C = A R^T - lower(A R^T - R A^T),
//    A = dpsi/dR (in-plane fixed corotated, normal k/3 (1 - r33)^3, shear
//    gamma/2 (r13^2 + r23^2)).  The in-plane columns become forces on the
//    three vertex particles (float64 atomics into fext); the d3 column becomes
//    the element particle's MLS stress tau_e = (P e3) d3^T.
//  * k_cloth_post (after G2P): d3 <- (I + dt C_e) d3, frictional return
//    mapping on R, element particle to the centroid of its vertices.
// Mesh arrays are in the user's particle order; inv_perm maps a user index to
// the sim-internal (sorted) particle index of this step.
#include "common.cuh"
#include "internal.h"

namespace mpmrb {

namespace {

struct QR3 {
  double q[3][3];  // columns q1, q2, q3 (q[c][row])
  double r11, r12, r13, r22, r23, r33;
};

__device__ __forceinline__ QR3 qr_gs(const double* f1, const double* f2, const double* f3) {
  QR3 o;
  o.r11 = sqrt(f1[0] * f1[0] + f1[1] * f1[1] + f1[2] * f1[2]);
#pragma unroll
  for (int d = 0; d < 3; ++d) o.q[0][d] = f1[d] / o.r11;
  o.r12 = o.q[0][0] * f2[0] + o.q[0][1] * f2[1] + o.q[0][2] * f2[2];
  double u2[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) u2[d] = f2[d] - o.r12 * o.q[0][d];
  o.r22 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
#pragma unroll
  for (int d = 0; d < 3; ++d) o.q[1][d] = u2[d] / o.r22;
  o.q[2][0] = o.q[0][1] * o.q[1][2] - o.q[0][2] * o.q[1][1];
  o.q[2][1] = o.q[0][2] * o.q[1][0] - o.q[0][0] * o.q[1][2];
  o.q[2][2] = o.q[0][0] * o.q[1][1] - o.q[0][1] * o.q[1][0];
  o.r13 = o.q[0][0] * f3[0] + o.q[0][1] * f3[1] + o.q[0][2] * f3[2];
  o.r23 = o.q[1][0] * f3[0] + o.q[1][1] * f3[1] + o.q[1][2] * f3[2];
  o.r33 = o.q[2][0] * f3[0] + o.q[2][1] * f3[1] + o.q[2][2] * f3[2];
  return o;
}

__device__ __forceinline__ void element_F(const double* x0, const double* x1, const double* x2,
                                          const double* dmi, const double* d3, double* f1,
                                          double* f2, double* f3) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double a = x1[d] - x0[d], b = x2[d] - x0[d];
    f1[d] = a * dmi[0] + b * dmi[2];  // [d1 d2] Dm^-1, dmi row-major (2,2)
    f2[d] = a * dmi[1] + b * dmi[3];
    f3[d] = d3[d];
  }
}

// P (row-major 3x3) of one element
__device__ __forceinline__ void cloth_piola(const QR3& o, const mpmrb_material& m, double* P) {
  const double a = o.r11, b = o.r12, dd = o.r22;
  const double x = a + dd, y = -b;
  const double nrm = sqrt(x * x + y * y);
  const double cs = x / nrm, sn = y / nrm;
  const double J = a * dd;
  double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  A[0][0] = 2.0 * m.mu * (a - cs) + m.lam * (J - 1.0) * dd;
  A[0][1] = 2.0 * m.mu * (b + sn);
  A[1][1] = 2.0 * m.mu * (dd - cs) + m.lam * (J - 1.0) * a;
  const double comp = fmax(0.0, 1.0 - o.r33);
  A[2][2] = -m.k_normal * comp * comp;
  A[0][2] = m.gamma_shear * o.r13;
  A[1][2] = m.gamma_shear * o.r23;
  const double R[3][3] = {{o.r11, o.r12, o.r13}, {0.0, o.r22, o.r23}, {0.0, 0.0, o.r33}};
  double B[3][3];  // A R^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) B[i][j] = A[i][0] * R[j][0] + A[i][1] * R[j][1] + A[i][2] * R[j][2];
  double Cm[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Cm[i][j] = (i > j) ? B[j][i] : B[i][j];  // B - lower(B - B^T)
  // R^-1 (upper triangular)
  const double i11 = 1.0 / o.r11, i22 = 1.0 / o.r22, i33 = 1.0 / o.r33;
  const double i12 = -o.r12 * i11 * i22;
  const double i23 = -o.r23 * i22 * i33;
  const double i13 = (o.r12 * o.r23 - o.r13 * o.r22) * i11 * i22 * i33;
  const double Ri[3][3] = {{i11, i12, i13}, {0.0, i22, i23}, {0.0, 0.0, i33}};
  double CR[3][3];  // C R^-T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      CR[i][j] = Cm[i][0] * Ri[j][0] + Cm[i][1] * Ri[j][1] + Cm[i][2] * Ri[j][2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      P[3 * i + j] = o.q[0][i] * CR[0][j] + o.q[1][i] * CR[1][j] + o.q[2][i] * CR[2][j];
}

__global__ void k_cloth_forces(long long ne, const int* __restrict__ tri,
                               const int* __restrict__ epart, const double* __restrict__ dm_inv,
                               const double* __restrict__ vol, const double* __restrict__ d3,
                               const int* __restrict__ inv_perm, const double* __restrict__ x,
                               const long long* __restrict__ mid,
                               const mpmrb_material* __restrict__ mats, int nmat,
                               double* __restrict__ fext, double* __restrict__ tau_buf) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x) {
    const int v0 = inv_perm[tri[3 * e]], v1 = inv_perm[tri[3 * e + 1]],
              v2 = inv_perm[tri[3 * e + 2]], pe = inv_perm[epart[e]];
    const long long m_id = mid[pe];
    if (m_id < 0 || m_id >= nmat) continue;
    const mpmrb_material m = mats[m_id];
    double f1[3], f2[3], f3[3];
    element_F(x + 3 * v0, x + 3 * v1, x + 3 * v2, dm_inv + 4 * e, d3 + 3 * e, f1, f2, f3);
    const QR3 o = qr_gs(f1, f2, f3);
    double P[9];
    cloth_piola(o, m, P);
    const double* dmi = dm_inv + 4 * e;
    const double V = vol[e];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      // dpsi/d(d1, d2) = P[:, 0:2] Dm^-T
      const double g1 = P[3 * d] * dmi[0] + P[3 * d + 1] * dmi[1];
      const double g2 = P[3 * d] * dmi[2] + P[3 * d + 1] * dmi[3];
      const double fa = -V * g1, fb = -V * g2;
      atomicAdd(&fext[3 * v1 + d], fa);
      atomicAdd(&fext[3 * v2 + d], fb);
      atomicAdd(&fext[3 * v0 + d], -(fa + fb));
    }
    // element particle: tau_e = (P e3) d3^T (P2G multiplies by the element
    // particle's rest volume, which is the element volume)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) tau_buf[9LL * pe + 3 * i + j] = P[3 * i + 2] * f3[j];
  }
}

// T: the element particles' APIC C (float64, or float32 in the fp32 mode);
// d3, positions and the return map stay float64
template <class T>
__global__ void k_cloth_post(long long ne, const int* __restrict__ tri,
                             const int* __restrict__ epart, const double* __restrict__ dm_inv,
                             double* __restrict__ d3, const int* __restrict__ inv_perm,
                             double* __restrict__ x, const T* __restrict__ c,
                             const long long* __restrict__ mid,
                             const mpmrb_material* __restrict__ mats, int nmat, double dt) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x) {
    const int v0 = inv_perm[tri[3 * e]], v1 = inv_perm[tri[3 * e + 1]],
              v2 = inv_perm[tri[3 * e + 2]], pe = inv_perm[epart[e]];
    const long long m_id = mid[pe];
    if (m_id < 0 || m_id >= nmat) continue;
    const mpmrb_material m = mats[m_id];
    // d3 <- (I + dt C_e) d3
    const T* C = c + 9LL * pe;
    double dn[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      dn[i] = d3[3 * e + i] + dt * ((double)C[3 * i] * d3[3 * e] +
                                    (double)C[3 * i + 1] * d3[3 * e + 1] +
                                    (double)C[3 * i + 2] * d3[3 * e + 2]);
    double f1[3], f2[3], f3[3];
    element_F(x + 3 * v0, x + 3 * v1, x + 3 * v2, dm_inv + 4 * e, dn, f1, f2, f3);
    const QR3 o = qr_gs(f1, f2, f3);
    // return mapping (oracle/cloth.py: return_map)
    double r13 = o.r13, r23 = o.r23, r33 = o.r33;
    if (r33 > 1.0) {
      r33 = 1.0;
      r13 = 0.0;
      r23 = 0.0;
    } else {
      const double s = sqrt(r13 * r13 + r23 * r23);
      const double comp = fmax(0.0, 1.0 - r33);
      const double limit = m.friction * m.k_normal * comp * comp;
      if (m.gamma_shear * s > limit) {
        const double scale = limit / fmax(m.gamma_shear * s, 1e-300);
        r13 *= scale;
        r23 *= scale;
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) d3[3 * e + i] = o.q[0][i] * r13 + o.q[1][i] * r23 + o.q[2][i] * r33;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      x[3LL * pe + d] = (x[3 * v0 + d] + x[3 * v1 + d] + x[3 * v2 + d]) / 3.0;
  }
}

__global__ void k_inverse_perm(const int* __restrict__ perm, long long n, int* __restrict__ inv) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    inv[perm[i]] = (int)i;
}

__global__ void k_gather_i8(const signed char* __restrict__ src, const int* __restrict__ perm,
                            long long n, signed char* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

unsigned cl_grid(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (unsigned)b;
}

}  // namespace

int launch_cloth_forces(Ctx& c, const ClothDev& cl, const ParticlesDev& p,
                        const mpmrb_material* mats_dev, int nmat) {
  if (cl.ne == 0) return MPMRB_OK;
  MPMRB_CUDA_OK(cudaMemsetAsync(p.fext, 0, sizeof(double) * 3 * p.n, c.stream));
  k_cloth_forces<<<cl_grid(cl.ne), 256, 0, c.stream>>>(cl.ne, cl.tri, cl.epart, cl.dm_inv,
                                                       cl.vol, cl.d3, cl.inv_perm, p.x, p.mid,
                                                       mats_dev, nmat, p.fext, p.tau);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

template <class T>
static int cloth_post(Ctx& c, const ClothDev& cl, const ParticlesT<T>& p,
                      const mpmrb_material* mats_dev, int nmat, double dt) {
  if (cl.ne == 0) return MPMRB_OK;
  k_cloth_post<T><<<cl_grid(cl.ne), 256, 0, c.stream>>>(cl.ne, cl.tri, cl.epart, cl.dm_inv, cl.d3,
                                                        cl.inv_perm, p.x, p.c, p.mid, mats_dev,
                                                        nmat, dt);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_cloth_post(Ctx& c, const ClothDev& cl, const ParticlesDev& p,
                      const mpmrb_material* mats_dev, int nmat, double dt) {
  return cloth_post(c, cl, p, mats_dev, nmat, dt);
}

int launch_cloth_post(Ctx& c, const ClothDev& cl, const ParticlesF32& p,
                      const mpmrb_material* mats_dev, int nmat, double dt) {
  return cloth_post(c, cl, p, mats_dev, nmat, dt);
}

int launch_inverse_perm(Ctx& c, const int* perm, long long n, int* inv) {
  if (n == 0) return MPMRB_OK;
  k_inverse_perm<<<cl_grid(n), 256, 0, c.stream>>>(perm, n, inv);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

int launch_gather_i8(Ctx& c, const signed char* src, const int* perm, long long n,
                     signed char* dst) {
  if (n == 0) return MPMRB_OK;
  k_gather_i8<<<cl_grid(n), 256, 0, c.stream>>>(src, perm, n, dst);
  c.launches++;
  MPMRB_CUDA_OK(cudaGetLastError());
  return MPMRB_OK;
}

}  // namespace mpmrb
