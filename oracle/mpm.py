"""Oracle: fixed-corotated stress, MLS/APIC P2G, grid update, G2P and the
singular-value clamp.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  Lamé parameters         /root/reference/pkg/src/mpmrb/materials.py:40-46
  det / inverse-transpose materials.py:49-67
  Higham polar rotation   materials.py:70-83 (batch-wide max|dR| <= 1e-13, <= 30 iters)
  signed-SVD clamp        materials.py:86-110 (sigma floor 0.05)
  Kirchhoff stress        materials.py:113-122, per-material grouping mpm.py:56-63
  P2G channels            mpm.py:66-99
  grid update             mpm.py:102-115 (active = mass > 1e-12, grid.py:19)
  G2P                     mpm.py:118-138
"""

from __future__ import annotations

import numpy as np

from .grid import MASS_EPS, Stencil, scatter_in_order

SIGMA_FLOOR = 0.05


def lame(E: float, nu: float) -> tuple[float, float]:
    """(mu, lambda) of Young's modulus / Poisson ratio (materials.py:40-46)."""
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def det33(m: np.ndarray) -> np.ndarray:
    """Column-triple-product determinant (materials.py:49-54)."""
    c0, c1, c2 = m[..., :, 0], m[..., :, 1], m[..., :, 2]
    return np.einsum("...i,...i->...", c0, np.cross(c1, c2))


def inv_transpose33(m: np.ndarray) -> np.ndarray:
    """Adjugate inverse-transpose (materials.py:57-67)."""
    c0, c1, c2 = m[..., :, 0], m[..., :, 1], m[..., :, 2]
    k0, k1, k2 = np.cross(c1, c2), np.cross(c2, c0), np.cross(c0, c1)
    d = np.einsum("...i,...i->...", c0, k0)
    return np.stack([k0, k1, k2], axis=-1) / d[..., None, None]


def polar_R(f: np.ndarray, iters: int = 30, tol: float = 1e-13) -> np.ndarray:
    """Rotation of F = R S by R <- (R + R^-T)/2 until the batch max change <= tol."""
    r = np.array(f, dtype=np.float64, copy=True)
    for _ in range(iters):
        nxt = 0.5 * (r + inv_transpose33(r))
        change = np.max(np.abs(nxt - r)) if r.size else 0.0
        r = nxt
        if change <= tol:
            break
    return r


def kirchhoff(f: np.ndarray, mu: float, lam: float) -> np.ndarray:
    """tau = 2 mu (F - R) F^T + lam (J - 1) J I for one material (materials.py:113-122)."""
    r = polar_R(f)
    j = det33(f)
    tau = 2.0 * mu * ((f - r) @ np.swapaxes(f, -1, -2))
    iso = lam * (j - 1.0) * j
    for d in range(3):
        tau[..., d, d] += iso
    return tau


def stresses(f: np.ndarray, material_id: np.ndarray, materials) -> np.ndarray:
    """Per-material-group Kirchhoff stress (mpm.py:56-63).

    ``materials`` is a list of (E, nu) pairs or objects with youngs_modulus /
    poisson_ratio.  The reference is elastic-only; materials whose ``model`` is
    "sand" use the (parity-unpinned) Hencky stress of oracle.plasticity.
    """
    from .plasticity import KIND_SAND, hencky_stress, material_kind
    tau = np.zeros_like(f)
    for mid in np.unique(material_id):
        m = materials[int(mid)]
        E, nu = (m if isinstance(m, tuple) else (m.youngs_modulus, m.poisson_ratio))[:2]
        mu, lam = lame(E, nu)
        sel = material_id == mid
        if not isinstance(m, tuple) and getattr(m, "model", "elastic") == "cloth":
            continue  # cloth: stresses come from the mesh (oracle/cloth.py)
        if not isinstance(m, tuple) and material_kind(m) == KIND_SAND:
            tau[sel] = hencky_stress(f[sel], mu, lam)
        else:
            tau[sel] = kirchhoff(f[sel], mu, lam)
    return tau


def p2g(x, v, f, c, mass, vol0, material_id, materials, st: Stencil, dt: float,
        n_nodes: int, extra_tau=None, fext=None):
    """Scatter mass, APIC momentum and the MLS force impulse (mpm.py:66-99).

    ``extra_tau`` (n,3,3) adds per-particle stresses (cloth element particles)
    and ``fext`` (n,3) per-particle forces applied as dt f w in the force
    channel (cloth vertex particles) — both NEW, oracle/cloth.py.

    Returns (mass (N,), mom_apic (N,3), mom_force (N,3)).
    """
    n = x.shape[0]
    if n == 0:
        return np.zeros(n_nodes), np.zeros((n_nodes, 3)), np.zeros((n_nodes, 3))
    tau = stresses(f, material_id, materials)
    if extra_tau is not None:
        tau = tau + extra_tau
    w = st.weights
    dinv = 4.0 / (st.h * st.h)
    mv = mass[:, None] * v
    mc = mass[:, None, None] * c
    s = (-dt * dinv) * vol0[:, None, None] * tau
    contrib = np.empty((n, 27, 7))
    contrib[:, :, 0] = w * mass[:, None]
    contrib[:, :, 1:4] = w[:, :, None] * (mv[:, None, :] + st.dpos @ mc.transpose(0, 2, 1))
    contrib[:, :, 4:7] = w[:, :, None] * (st.dpos @ s.transpose(0, 2, 1))
    if fext is not None:
        contrib[:, :, 4:7] += w[:, :, None] * (dt * fext)[:, None, :]
    out = scatter_in_order(st.nodes, contrib, n_nodes)
    return out[:, 0].copy(), out[:, 1:4].copy(), out[:, 4:7].copy()


def grid_update(mass, mom_apic, mom_force, gravity, dt: float):
    """(active, v_k, v_star) from the scattered channels (mpm.py:102-115)."""
    active = mass > MASS_EPS
    inv_m = np.zeros_like(mass)
    np.divide(1.0, mass, out=inv_m, where=active)
    v_k = mom_apic * inv_m[:, None]
    v_star = (mom_apic + mom_force) * inv_m[:, None] + dt * np.asarray(gravity, dtype=np.float64)
    v_k[~active] = 0.0
    v_star[~active] = 0.0
    return active, v_k, v_star


def clamp_inverted(f: np.ndarray) -> tuple[np.ndarray, int]:
    """Repair det<=0 / non-finite F via signed SVD, sigma >= 0.05 (materials.py:86-110)."""
    f = np.asarray(f, dtype=np.float64)
    bad = ~(det33(f) > 0.0) | ~np.isfinite(f).all(axis=(-2, -1))
    k = int(bad.sum())
    if k == 0:
        return f, 0
    out = f.copy()
    fb = np.nan_to_num(f[bad], nan=0.0, posinf=0.0, neginf=0.0)
    u, s, vt = np.linalg.svd(fb)
    flip_u = np.linalg.det(u) < 0
    u[flip_u, :, 2] = -u[flip_u, :, 2]
    s[flip_u, 2] = -s[flip_u, 2]
    flip_v = np.linalg.det(vt) < 0
    vt[flip_v, 2, :] = -vt[flip_v, 2, :]
    s[flip_v, 2] = -s[flip_v, 2]
    s = np.maximum(s, SIGMA_FLOOR)
    out[bad] = u @ (s[..., None] * vt)
    return out, k


def g2p(x, f, st: Stencil, v_next: np.ndarray, dt: float, keep_f=None):
    """Gather v, C; advect x; F <- (I + dt C) F; clamp (mpm.py:118-138).
    ``keep_f`` (n,) bool: particles whose F is left unchanged (cloth).

    Returns (x_new, v_new, c_new, f_new, n_clamped).
    """
    if x.shape[0] == 0:
        return x, np.zeros((0, 3)), np.zeros((0, 3, 3)), f, 0
    wv = st.weights[:, :, None] * v_next[st.nodes]
    v_new = wv.sum(axis=1)
    dinv = 4.0 / (st.h * st.h)
    c_new = dinv * (wv.transpose(0, 2, 1) @ st.dpos)
    x_new = x + dt * v_new
    f_new = (np.eye(3)[None] + dt * c_new) @ f
    if keep_f is not None:
        f_new[keep_f] = f[keep_f]
    f_new, k = clamp_inverted(f_new)
    return x_new, v_new, c_new, f_new, k
