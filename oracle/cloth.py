"""Oracle: codimensional cloth (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PARITY UNPINNED.  The reference package has no cloth; the
paper models cloth "following the approach of Jiang et al. 2017: a particle at
each mesh vertex and at the centroid of each triangle face".
This is a float64 NumPy statement of that model (anisotropic elastoplasticity
for cloth, Jiang, Gast, Teran, SIGGRAPH 2017), without bending:

* Triangle e with vertex particles (i0, i1, i2) and an element particle p_e.
  F_e = [d1 d2 d3] diag(Dm^-1, 1), d1 = x_i1 - x_i0, d2 = x_i2 - x_i0 (current
  vertex positions) and d3 the element's transverse direction, advected with
  the grid like an MPM deformation gradient (d3 <- (I + dt C_pe) d3).
* F = Q R (Gram-Schmidt, q3 = q1 x q2).  Energy per rest volume:
    in-plane  fixed corotated on the upper 2x2 block R_hat (mu, lambda),
    normal    k/3 (1 - r33)^3 for r33 <= 1 (resists compression only),
    shear     gamma/2 (r13^2 + r23^2).
* First Piola stress P = Q C R^-T, C = A R^T - lower(A R^T - R A^T), A =
  dpsi/dR (upper part), lower() = strictly lower triangle.
* Forces: in-plane columns act on the vertex particles (f_i1 = -V P_12
  Dm^-T e1, ...), transferred to the grid through the vertices' P2G force
  channel; the d3 column acts through the element particle as the MLS stress
  tau_e = (P e3) d3^T.
* After G2P: return mapping on R (r33 > 1: separated, r33 = 1, r13 = r23 = 0;
  else |gamma (r13, r23)| <= c_f k (1 - r33)^2, friction of cloth-cloth
  contact), d3 = Q (r13, r23, r33); element particles move to the centroid of
  their vertices.

Verified by its own known-answer tests: forces equal minus the finite
-difference gradient of ``energy`` (tests/test_cloth_oracle.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROLE_NONE, ROLE_VERTEX, ROLE_ELEMENT = 0, 1, 2


@dataclass
class ClothParams:
    mu: float
    lam: float
    k_normal: float
    gamma_shear: float
    friction: float


@dataclass
class ClothMesh:
    tri: np.ndarray       # (ne, 3) int64 vertex particle indices
    epart: np.ndarray     # (ne,) int64 element particle index
    dm_inv: np.ndarray    # (ne, 2, 2)
    vol: np.ndarray       # (ne,) rest volume (area x thickness)
    d3: np.ndarray        # (ne, 3) transverse direction (state)
    params: ClothParams

    def roles(self, n: int) -> np.ndarray:
        r = np.zeros(n, dtype=np.int8)
        r[self.tri.ravel()] = ROLE_VERTEX
        r[self.epart] = ROLE_ELEMENT
        return r


def params_from(E: float, nu: float, k_normal: float | None = None,
                gamma_shear: float | None = None, friction: float = 0.3) -> ClothParams:
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return ClothParams(mu=mu, lam=lam, k_normal=E if k_normal is None else k_normal,
                       gamma_shear=0.1 * E if gamma_shear is None else gamma_shear,
                       friction=friction)


def deformation(x: np.ndarray, mesh: ClothMesh, d3: np.ndarray | None = None) -> np.ndarray:
    t = mesh.tri
    d1 = x[t[:, 1]] - x[t[:, 0]]
    d2 = x[t[:, 2]] - x[t[:, 0]]
    F = np.empty((t.shape[0], 3, 3))
    F[:, :, 0:2] = np.stack([d1, d2], axis=-1) @ mesh.dm_inv
    F[:, :, 2] = mesh.d3 if d3 is None else d3
    return F


def qr_gs(F: np.ndarray):
    """Gram-Schmidt QR with q3 = q1 x q2 (r33 = q3 . f3 may be negative)."""
    f1, f2, f3 = F[:, :, 0], F[:, :, 1], F[:, :, 2]
    r11 = np.linalg.norm(f1, axis=1)
    q1 = f1 / r11[:, None]
    r12 = np.einsum("ij,ij->i", q1, f2)
    u2 = f2 - r12[:, None] * q1
    r22 = np.linalg.norm(u2, axis=1)
    q2 = u2 / r22[:, None]
    q3 = np.cross(q1, q2)
    r13 = np.einsum("ij,ij->i", q1, f3)
    r23 = np.einsum("ij,ij->i", q2, f3)
    r33 = np.einsum("ij,ij->i", q3, f3)
    Q = np.stack([q1, q2, q3], axis=-1)
    R = np.zeros_like(F)
    R[:, 0, 0], R[:, 0, 1], R[:, 0, 2] = r11, r12, r13
    R[:, 1, 1], R[:, 1, 2] = r22, r23
    R[:, 2, 2] = r33
    return Q, R


def _polar2(a, b, c, d):
    """Rotation factor of the 2x2 matrix [[a, b], [c, d]] (det > 0 assumed)."""
    x = a + d
    y = c - b
    n = np.sqrt(x * x + y * y)
    cs, sn = x / n, y / n
    return cs, sn


def energy_density(R: np.ndarray, p: ClothParams) -> np.ndarray:
    a, b, d = R[:, 0, 0], R[:, 0, 1], R[:, 1, 1]
    cs, sn = _polar2(a, b, np.zeros_like(a), d)
    # R_hat - Rot, Frobenius squared
    e_fc = (a - cs) ** 2 + (b + sn) ** 2 + (0.0 - sn) ** 2 + (d - cs) ** 2
    J = a * d
    psi = p.mu * e_fc + 0.5 * p.lam * (J - 1.0) ** 2
    r33 = R[:, 2, 2]
    comp = np.maximum(0.0, 1.0 - r33)
    psi = psi + (p.k_normal / 3.0) * comp ** 3
    psi = psi + 0.5 * p.gamma_shear * (R[:, 0, 2] ** 2 + R[:, 1, 2] ** 2)
    return psi


def dpsi_dR(R: np.ndarray, p: ClothParams) -> np.ndarray:
    """A = dpsi/dR, upper-triangular entries only."""
    a, b, d = R[:, 0, 0], R[:, 0, 1], R[:, 1, 1]
    cs, sn = _polar2(a, b, np.zeros_like(a), d)
    J = a * d
    A = np.zeros_like(R)
    # fixed corotated on [[a, b], [0, d]]: 2 mu (F - Rot) + lam (J - 1) J F^-T
    # F^-T = 1/J [[d, 0], [-b, a]]
    A[:, 0, 0] = 2.0 * p.mu * (a - cs) + p.lam * (J - 1.0) * d
    A[:, 0, 1] = 2.0 * p.mu * (b + sn)
    A[:, 1, 1] = 2.0 * p.mu * (d - cs) + p.lam * (J - 1.0) * a
    r33 = R[:, 2, 2]
    A[:, 2, 2] = -p.k_normal * np.maximum(0.0, 1.0 - r33) ** 2
    A[:, 0, 2] = p.gamma_shear * R[:, 0, 2]
    A[:, 1, 2] = p.gamma_shear * R[:, 1, 2]
    return A


def piola(F: np.ndarray, p: ClothParams) -> np.ndarray:
    Q, R = qr_gs(F)
    A = dpsi_dR(R, p)
    B = A @ np.swapaxes(R, 1, 2)
    K = B - np.swapaxes(B, 1, 2)           # B - B^T
    C = B - np.tril(K, k=-1)
    return Q @ C @ np.swapaxes(np.linalg.inv(R), 1, 2)


def energy(x: np.ndarray, mesh: ClothMesh, d3: np.ndarray | None = None) -> float:
    F = deformation(x, mesh, d3)
    _, R = qr_gs(F)
    return float(np.sum(mesh.vol * energy_density(R, mesh.params)))


def forces(x: np.ndarray, mesh: ClothMesh):
    """(vertex forces (n,3), element stresses tau_e (ne,3,3), P (ne,3,3))."""
    F = deformation(x, mesh)
    P = piola(F, mesh.params)
    G = P[:, :, 0:2] @ np.swapaxes(mesh.dm_inv, 1, 2)  # dpsi/d(d1, d2)
    f1 = -mesh.vol[:, None] * G[:, :, 0]
    f2 = -mesh.vol[:, None] * G[:, :, 1]
    f0 = -(f1 + f2)
    fext = np.zeros_like(x)
    t = mesh.tri
    for j, fj in ((0, f0), (1, f1), (2, f2)):
        for d in range(3):
            fext[:, d] += np.bincount(t[:, j], weights=fj[:, d], minlength=x.shape[0])
    tau = P[:, :, 2][:, :, None] * mesh.d3[:, None, :]
    return fext, tau, P


def return_map(F: np.ndarray, p: ClothParams) -> np.ndarray:
    """Cloth-cloth frictional contact plasticity on R; returns the new d3."""
    Q, R = qr_gs(F)
    r13, r23, r33 = R[:, 0, 2].copy(), R[:, 1, 2].copy(), R[:, 2, 2].copy()
    sep = r33 > 1.0
    r33 = np.where(sep, 1.0, r33)
    r13 = np.where(sep, 0.0, r13)
    r23 = np.where(sep, 0.0, r23)
    s = np.sqrt(r13 * r13 + r23 * r23)
    limit = p.friction * p.k_normal * np.maximum(0.0, 1.0 - r33) ** 2
    over = (~sep) & (p.gamma_shear * s > limit)
    scale = np.where(over, limit / np.maximum(p.gamma_shear * s, 1e-300), 1.0)
    r13, r23 = r13 * scale, r23 * scale
    return np.einsum("nij,nj->ni", Q, np.stack([r13, r23, r33], axis=1))


def post_g2p(x: np.ndarray, c: np.ndarray, mesh: ClothMesh, dt: float) -> np.ndarray:
    """d3 advection + return map, element particles to the face centroids.
    Returns the new x (mesh.d3 is updated in place)."""
    ep = mesh.epart
    d3 = np.einsum("nij,nj->ni", np.eye(3)[None] + dt * c[ep], mesh.d3)
    F = deformation(x, mesh, d3)
    mesh.d3 = return_map(F, mesh.params)
    x = x.copy()
    x[ep] = x[mesh.tri].mean(axis=1)
    return x


# ------------------------------------------------------------------ seeding

def sheet(center, size, n_side: int, thickness: float, rho: float, params: ClothParams,
          material_id: int, normal_axis: int = 2):
    """A square sheet: n_side x n_side vertex particles on a regular lattice,
    2 (n_side-1)^2 triangles with an element particle at each centroid; mass
    rho * area * thickness split half to the element particles and half to
    the vertices (a third of each triangle's half per vertex).

    The element particles' rest volume is the element volume (their
    transverse stress acts through it in P2G).

    Returns (x (n,3), mass (n,), vol (n,), material_id (n,), mesh)."""
    center = np.asarray(center, dtype=np.float64)
    lx, ly = size
    u = np.linspace(-0.5 * lx, 0.5 * lx, n_side)
    v = np.linspace(-0.5 * ly, 0.5 * ly, n_side)
    U, V = np.meshgrid(u, v, indexing="ij")
    axes = [a for a in range(3) if a != normal_axis]
    nv = n_side * n_side
    xv = np.tile(center, (nv, 1))
    xv[:, axes[0]] += U.ravel()
    xv[:, axes[1]] += V.ravel()
    tris = []
    for i in range(n_side - 1):
        for j in range(n_side - 1):
            a = i * n_side + j
            b, c_, d = a + n_side, a + 1, a + n_side + 1
            tris.append((a, b, d))
            tris.append((a, d, c_))
    tri = np.asarray(tris, dtype=np.int64)
    ne = tri.shape[0]
    uv = np.stack([U.ravel(), V.ravel()], axis=1)
    dm = np.stack([uv[tri[:, 1]] - uv[tri[:, 0]], uv[tri[:, 2]] - uv[tri[:, 0]]], axis=-1)
    area = 0.5 * np.abs(np.linalg.det(dm))
    dm_inv = np.linalg.inv(dm)
    ex = np.zeros(3)
    ex[normal_axis] = 1.0
    # orientation: q3 = q1 x q2 must equal +normal at rest so r33 = 1
    d1 = xv[tri[:, 1]] - xv[tri[:, 0]]
    d2 = xv[tri[:, 2]] - xv[tri[:, 0]]
    sgn = np.sign(np.cross(d1, d2) @ ex)
    d3 = sgn[:, None] * ex[None, :]
    x = np.concatenate([xv, xv[tri].mean(axis=1)])
    m_tri = rho * area * thickness
    mass = np.zeros(nv + ne)
    for j in range(3):
        mass[:nv] += np.bincount(tri[:, j], weights=m_tri / 6.0, minlength=nv)
    mass[nv:] = 0.5 * m_tri
    vol = mass / rho
    vol[nv:] = area * thickness  # element particles carry the element volume
    mid = np.full(nv + ne, material_id, dtype=np.int64)
    mesh = ClothMesh(tri=tri, epart=np.arange(nv, nv + ne, dtype=np.int64), dm_inv=dm_inv,
                     vol=area * thickness, d3=d3, params=params)
    return x, mass, vol, mid, mesh
