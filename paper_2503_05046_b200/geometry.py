"""Collision primitives and their signed-distance queries.

Shapes are small host descriptions (reference geometry.py:16-156: same names,
validation and mass properties).  Queries run on the GPU through the same
device SDF code the fused contact-detection kernel uses
(csrc/contact.cuh: sdf_local, contact_frame).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class HalfSpace:
    """Solid half-space below the plane n . p = offset (geometry.py:16-37)."""

    normal: tuple = (0.0, 0.0, 1.0)
    offset: float = 0.0

    def __post_init__(self):
        if abs(float(np.linalg.norm(self.normal)) - 1.0) > 1e-9:
            raise ValueError("half-space normal must be unit length")

    kind = _lib.GEOM_HALFSPACE

    def params(self):
        return (*(float(a) for a in self.normal), float(self.offset))

    @property
    def volume(self) -> float:
        raise ValueError("half-spaces have no finite volume (kinematic only)")

    def query(self, p):
        return query_signed_distance(self, p)


@dataclass(frozen=True)
class Sphere:
    radius: float

    def __post_init__(self):
        if not self.radius > 0:
            raise ValueError("sphere radius must be positive")

    kind = _lib.GEOM_SPHERE

    def params(self):
        return (float(self.radius), 0.0, 0.0, 0.0)

    @property
    def volume(self) -> float:
        return 4.0 / 3.0 * np.pi * self.radius ** 3

    def unit_inertia(self) -> np.ndarray:
        return np.eye(3) * (0.4 * self.radius ** 2)

    def query(self, p):
        return query_signed_distance(self, p)


@dataclass(frozen=True)
class Box:
    half_extents: tuple

    def __post_init__(self):
        if not all(e > 0 for e in self.half_extents):
            raise ValueError("box half_extents must be positive")

    kind = _lib.GEOM_BOX

    def params(self):
        return (*(float(a) for a in self.half_extents), 0.0)

    @property
    def volume(self) -> float:
        a, b, c = self.half_extents
        return 8.0 * a * b * c

    def unit_inertia(self) -> np.ndarray:
        sx, sy, sz = (2.0 * np.asarray(self.half_extents, dtype=np.float64)) ** 2
        return np.diag([(sy + sz) / 12.0, (sx + sz) / 12.0, (sx + sy) / 12.0])

    def query(self, p):
        return query_signed_distance(self, p)


@dataclass(frozen=True)
class Capsule:
    """Capsule along the local z axis."""

    radius: float
    half_length: float

    def __post_init__(self):
        if not (self.radius > 0 and self.half_length > 0):
            raise ValueError("capsule radius and half_length must be positive")

    kind = _lib.GEOM_CAPSULE

    def params(self):
        return (float(self.radius), float(self.half_length), 0.0, 0.0)

    @property
    def volume(self) -> float:
        r, hl = self.radius, self.half_length
        return np.pi * r * r * 2.0 * hl + 4.0 / 3.0 * np.pi * r ** 3

    def unit_inertia(self) -> np.ndarray:
        # cylinder + two hemispherical caps, unit total mass
        r, hl = self.radius, self.half_length
        length = 2.0 * hl
        vc, vs = np.pi * r * r * length, 4.0 / 3.0 * np.pi * r ** 3
        mc, ms = vc / (vc + vs), vs / (vc + vs)
        izz = 0.5 * mc * r * r + 0.4 * ms * r * r
        ixx = mc * (length * length / 12.0 + 0.25 * r * r) + ms * (
            0.4 * r * r + hl * hl + 0.375 * r * length)
        return np.diag([ixx, ixx, izz])

    def query(self, p):
        return query_signed_distance(self, p)


Shape = HalfSpace | Sphere | Box | Capsule


def geom_struct(shape, rot=np.eye(3), pos=(0.0, 0.0, 0.0), mu=0.0, body=0, geom=0,
                body_pos=(0.0, 0.0, 0.0), body_v=(0.0, 0.0, 0.0),
                body_omega=(0.0, 0.0, 0.0)) -> _lib.Geom:
    g = _lib.Geom()
    g.kind = shape.kind
    g.body = body
    g.geom = geom
    g.rot[:] = [float(a) for a in np.asarray(rot, dtype=np.float64).ravel()]
    g.pos[:] = [float(a) for a in pos]
    g.params[:] = shape.params()
    g.mu = float(mu)
    g.body_pos[:] = [float(a) for a in body_pos]
    g.body_v[:] = [float(a) for a in body_v]
    g.body_omega[:] = [float(a) for a in body_omega]
    return g


def query_signed_distance(shape, points):
    """phi, outward normal, closest surface point for (n,3) LOCAL points
    (geometry.py:162-169).  Returns CUDA tensors."""
    if isinstance(points, torch.Tensor):
        bad = points.dim() != 2 or points.shape[-1] != 3
    else:
        points = np.asarray(points, dtype=np.float64)
        bad = points.ndim != 2 or points.shape[1] != 3
    if bad:
        raise ValueError("points must have shape (n, 3)")
    pts = _lib.as_dev(points)
    if pts.numel() and not bool(torch.isfinite(pts).all()):
        raise ValueError("query points must be finite")
    n = pts.shape[0]
    phi = _lib.empty((n,))
    nrm = _lib.empty((n, 3))
    wit = _lib.empty((n, 3))
    g = geom_struct(shape)
    _lib.check(_lib.lib().mpmrb_sdf_query(_lib.ctx(), C.byref(g), _lib.ptr(pts), n,
                                          _lib.ptr(phi), _lib.ptr(nrm), _lib.ptr(wit)))
    return phi, nrm, wit


def contact_frames(normals):
    """World-to-contact rotations, rows (t1, t2, n) (geometry.py:186-189)."""
    nrm = _lib.as_dev(normals)
    n = nrm.shape[0]
    out = _lib.empty((n, 3, 3))
    _lib.check(_lib.lib().mpmrb_contact_frames(_lib.ctx(), _lib.ptr(nrm), n, _lib.ptr(out)))
    return out


def tangent_basis(normals):
    fr = contact_frames(normals)
    return fr[:, 0, :], fr[:, 1, :]
