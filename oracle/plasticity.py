"""Oracle: Drucker–Prager sand (Hencky St.Venant–Kirchhoff + return map).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PARITY UNPINNED: the reference declares plasticity out of scope
(materials.py:1-8 is elastic-only).  This is
a fresh float64 restatement of the published model the paper builds on
(Klár et al. 2016, "Drucker–Prager elastoplasticity for sand animation", the
sand model cited at /root/reference/PAPER.md:28), hooked where the reference's
material code sits: the stress in ``compute_stresses`` (mpm.py:56-63) and the
post-update F in ``grid_to_particle`` (mpm.py:135-137).  It is pinned only by
its own analytic known-answer tests (tests/test_plasticity_oracle.py).

Model (d = 3, F = U diag(sigma) V^T with det-corrected U, V):
  eps   = log(sigma)
  tau   = U diag(2 mu eps + lam tr(eps)) U^T                      (Kirchhoff)
  alpha = sqrt(2/3) * 2 sin(phi_f) / (3 - sin(phi_f))
  ehat  = eps - tr(eps)/3
  case II  tr(eps) > 0 (tension)                                  : sigma = 1
  case I   dgamma = |ehat| + (3 lam + 2 mu)/(2 mu) tr(eps) alpha <= 0
           (this includes |ehat| == 0 under compression)            : keep
  case III eps <- eps - dgamma ehat/|ehat|,  sigma = exp(eps)
  plastic state q += |eps_before - eps_after| (accumulated plastic strain)
"""

from __future__ import annotations

import numpy as np

KIND_ELASTIC = 0
KIND_SAND = 1


def material_kind(m) -> int:
    return KIND_SAND if getattr(m, "model", "elastic") == "sand" else KIND_ELASTIC


def dp_alpha(friction_angle_deg: float) -> float:
    s = np.sin(np.deg2rad(friction_angle_deg))
    return np.sqrt(2.0 / 3.0) * 2.0 * s / (3.0 - s)


def signed_svd(f: np.ndarray):
    """SVD with proper-rotation U, V; the last singular value carries the sign."""
    u, s, vt = np.linalg.svd(f)
    fu = np.linalg.det(u) < 0
    u[fu, :, 2] = -u[fu, :, 2]
    s[fu, 2] = -s[fu, 2]
    fv = np.linalg.det(vt) < 0
    vt[fv, 2, :] = -vt[fv, 2, :]
    s[fv, 2] = -s[fv, 2]
    return u, s, vt


def hencky_stress(f: np.ndarray, mu: float, lam: float) -> np.ndarray:
    """Kirchhoff stress of the Hencky St.Venant–Kirchhoff model."""
    u, s, _ = signed_svd(f)
    eps = np.log(np.maximum(s, 1e-12))
    tr = eps.sum(axis=1)
    d = 2.0 * mu * eps + lam * tr[:, None]
    return np.einsum("pik,pk,pjk->pij", u, d, u)


def project(s: np.ndarray, mu: float, lam: float, alpha: float):
    """Return-map singular values (n,3). Returns (sigma_new, dq)."""
    eps = np.log(np.maximum(s, 1e-12))
    tr = eps.sum(axis=1)
    ehat = eps - tr[:, None] / 3.0
    en = np.sqrt(np.sum(ehat * ehat, axis=1))
    dgam = en + (3.0 * lam + 2.0 * mu) / (2.0 * mu) * tr * alpha
    out = eps.copy()
    tip = tr > 0.0
    cone = (~tip) & (dgam > 0.0) & (en > 0.0)
    out[tip] = 0.0
    safe = np.where(en > 0.0, en, 1.0)
    out[cone] = eps[cone] - (dgam[cone] / safe[cone])[:, None] * ehat[cone]
    dq = np.sqrt(np.sum((eps - out) ** 2, axis=1))
    # case I: unchanged (including tip test false and dgam <= 0)
    keep = ~(tip | cone)
    sig = np.exp(out)
    sig[keep] = s[keep]
    dq[keep] = 0.0
    return sig, dq


def return_map(f: np.ndarray, plastic: np.ndarray, material_id: np.ndarray, materials):
    """Apply the DP projection to every sand particle. Returns (F, plastic)."""
    kinds = np.array([material_kind(m) for m in materials], dtype=np.int64)
    if not (kinds == KIND_SAND).any() or f.shape[0] == 0:
        return f, plastic
    f = f.copy()
    plastic = plastic.copy()
    from .mpm import lame
    for mid in np.unique(material_id):
        m = materials[int(mid)]
        if material_kind(m) != KIND_SAND:
            continue
        sel = np.flatnonzero(material_id == mid)
        mu, lam = lame(m.youngs_modulus, m.poisson_ratio)
        u, s, vt = signed_svd(f[sel])
        sig, dq = project(s, mu, lam, dp_alpha(m.friction_angle))
        f[sel] = np.einsum("pik,pk,pkj->pij", u, sig, vt)
        plastic[sel] += dq
    return f, plastic
