"""Constitutive models.

* elastic: fixed-corotated hyperelasticity, tau = 2 mu (F - R) F^T +
  lam (J - 1) J I (reference materials.py:1-122) — the stress is evaluated
  inside the fused P2G kernel (csrc/svd3.cuh: kirchhoff_fixed_corotated).
* sand (NEW, parity unpinned — the reference declares plasticity out of scope,
  SPEC.md:8,98,111): Hencky St.Venant–Kirchhoff stress plus a Drucker–Prager
  return map applied in the G2P kernel (Klár et al. 2016; oracle/plasticity.py
  restates it in NumPy).
* cloth (NEW, parity unpinned): codimensional cloth of Jiang et al. 2017 as the
  paper uses it — in-plane fixed corotated (mu, lambda),
  transverse compression k_normal, transverse shear gamma_shear and cloth-cloth
  friction (csrc/cloth.cu; oracle/cloth.py).  Defaults: k_normal = E,
  gamma_shear = 0.1 E, friction 0.3 (proposed; the paper gives only E, nu, rho).
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

log = logging.getLogger(__name__)

SIGMA_MIN = 0.05  # materials.py:21


@dataclass(frozen=True)
class Material:
    youngs_modulus: float
    poisson_ratio: float
    density: float
    model: str = "elastic"          # "elastic" | "sand" | "cloth"
    friction_angle: float = 30.0    # degrees, sand only
    cloth_normal_stiffness: float | None = None  # cloth: default E
    cloth_shear_stiffness: float | None = None   # cloth: default 0.1 E
    cloth_friction: float = 0.3                  # cloth-cloth friction

    def __post_init__(self):
        if not (self.youngs_modulus > 0.0):
            raise ValueError(f"youngs_modulus must be > 0, got {self.youngs_modulus}")
        if not (0.0 <= self.poisson_ratio < 0.5):
            raise ValueError(f"poisson_ratio must be in [0, 0.5), got {self.poisson_ratio}")
        if not (self.density > 0.0):
            raise ValueError(f"density must be > 0, got {self.density}")
        if self.model not in ("elastic", "sand", "cloth"):
            raise ValueError(f"unknown material model {self.model!r}")
        if self.model == "sand" and not (0.0 < self.friction_angle < 90.0):
            raise ValueError("friction_angle must be in (0, 90) degrees")

    @property
    def lame(self) -> tuple[float, float]:
        """(mu, lambda) from (E, nu) (materials.py:40-46)."""
        e, nu = self.youngs_modulus, self.poisson_ratio
        return e / (2.0 * (1.0 + nu)), e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))

    @property
    def dp_alpha(self) -> float:
        s = np.sin(np.deg2rad(self.friction_angle))
        return float(np.sqrt(2.0 / 3.0) * 2.0 * s / (3.0 - s))

    @property
    def cloth_params(self) -> tuple[float, float, float]:
        """(k_normal, gamma_shear, friction) of the cloth model."""
        E = self.youngs_modulus
        k = E if self.cloth_normal_stiffness is None else self.cloth_normal_stiffness
        g = 0.1 * E if self.cloth_shear_stiffness is None else self.cloth_shear_stiffness
        return float(k), float(g), float(self.cloth_friction)

    def to_struct(self) -> _lib.Material:
        m = _lib.Material()
        m.kind = {"sand": _lib.MAT_SAND, "cloth": _lib.MAT_CLOTH}.get(self.model, _lib.MAT_ELASTIC)
        m.mu, m.lam = self.lame
        m.dp_alpha = self.dp_alpha if self.model == "sand" else 0.0
        if self.model == "cloth":
            m.k_normal, m.gamma_shear, m.friction = self.cloth_params
        return m


def material_table(materials) -> tuple:
    arr = (_lib.Material * max(1, len(materials)))()
    for i, m in enumerate(materials):
        arr[i] = m.to_struct()
    return arr, len(materials)


def det3(m) -> torch.Tensor:
    """Column triple-product determinant of (...,3,3) (materials.py:49-54)."""
    m = _lib.as_dev(m)
    return torch.einsum("...i,...i->...", m[..., :, 0],
                        torch.linalg.cross(m[..., :, 1], m[..., :, 2], dim=-1))


def _stack_op(fn, m) -> torch.Tensor:
    m = _lib.as_dev(m)
    shape = m.shape
    flat = m.reshape(-1, 3, 3).contiguous()
    out = torch.empty_like(flat)
    _lib.check(fn(_lib.ctx(), _lib.ptr(flat), flat.shape[0], _lib.ptr(out)))
    return out.reshape(shape)


def inverse_transpose3(m) -> torch.Tensor:
    """Batched inverse-transpose via the adjugate (materials.py:57-67)."""
    return _stack_op(_lib.lib().mpmrb_inverse_transpose3, m)


def polar_rotation(f) -> torch.Tensor:
    """Rotation factor of the polar decomposition (materials.py:70-83), Higham
    iteration on the device (per-matrix stop at max|dR| <= 1e-13)."""
    return _stack_op(_lib.lib().mpmrb_polar_rotation, f)


def energy_density(f, material: Material) -> float:
    """psi(F) = mu sum (s_i - 1)^2 + lam/2 (J - 1)^2 with signed singular
    values (materials.py:138-149); the reference uses it only in
    verification oracles (not the runtime force path), as here."""
    fd = _lib.as_dev(f)
    if fd.shape != (3, 3):
        raise ValueError(f"expected a (3, 3) deformation gradient, got {tuple(fd.shape)}")
    if not bool(torch.isfinite(fd).all()):
        raise ValueError("deformation gradient has non-finite entries")
    mu, lam = material.lame
    u, s, vt = torch.linalg.svd(fd)
    if float(torch.linalg.det(u) * torch.linalg.det(vt)) < 0:
        s = s.clone()
        s[2] = -s[2]
    j = float(det3(fd))
    return float(mu * torch.sum((s - 1.0) ** 2)) + 0.5 * lam * (j - 1.0) ** 2


def kirchhoff_stress_batch(f, mu: float, lam: float) -> torch.Tensor:
    """tau(F) for a (n,3,3) stack of one elastic material (materials.py:113-122)."""
    f = _lib.as_dev(f)
    shape = f.shape
    f = f.reshape(-1, 3, 3).contiguous()
    mat = _lib.Material()
    mat.kind, mat.mu, mat.lam = _lib.MAT_ELASTIC, float(mu), float(lam)
    tab = (_lib.Material * 1)(mat)
    mid = torch.zeros(f.shape[0], dtype=torch.int64, device=f.device)
    tau = torch.empty_like(f)
    _lib.check(_lib.lib().mpmrb_compute_stresses(_lib.ctx(), _lib.ptr(f), _lib.ptr(mid),
                                                 f.shape[0], tab, 1, _lib.ptr(tau)))
    return tau.reshape(shape)


def compute_stress(f, material: Material) -> torch.Tensor:
    """Kirchhoff stress of one deformation gradient (materials.py:125-136)."""
    fn = np.asarray(_lib.to_numpy(f), dtype=np.float64)
    if fn.shape != (3, 3):
        raise ValueError(f"expected a (3, 3) deformation gradient, got {fn.shape}")
    if not np.isfinite(fn).all():
        raise ValueError("deformation gradient has non-finite entries")
    if not np.linalg.det(fn) > 0.0:
        raise ValueError("deformation gradient must have positive determinant")
    tab, n = material_table([material])
    fd = _lib.as_dev(fn).reshape(1, 3, 3).contiguous()
    mid = torch.zeros(1, dtype=torch.int64, device=fd.device)
    tau = torch.empty_like(fd)
    _lib.check(_lib.lib().mpmrb_compute_stresses(_lib.ctx(), _lib.ptr(fd), _lib.ptr(mid), 1, tab,
                                                 n, _lib.ptr(tau)))
    return tau[0]


def clamp_degenerate(f) -> tuple[torch.Tensor, int]:
    """Clamp singular values at SIGMA_MIN where det(F) <= 0 or non-finite
    (materials.py:86-110).  Returns (repaired stack, number repaired)."""
    fd = _lib.as_dev(f).reshape(-1, 3, 3).contiguous()
    out = torch.empty_like(fd)
    nbad = C.c_int64()
    _lib.check(_lib.lib().mpmrb_clamp_degenerate(_lib.ctx(), _lib.ptr(fd), fd.shape[0],
                                                 _lib.ptr(out), C.byref(nbad)))
    if nbad.value:
        log.warning("clamped %d inverted deformation gradients (singular value floor %.2f)",
                    int(nbad.value), SIGMA_MIN)
    return out, int(nbad.value)
