"""Oracle: analytic signed-distance primitives and contact frames.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Each query maps geom-local points (n,3) to (phi, outward normal, witness).
Restates:
  half-space   /root/reference/pkg/src/mpmrb/geometry.py:16-37
  sphere       geometry.py:40-64   (normal (0,0,1) when |p| < 1e-15)
  box          geometry.py:67-112  (interior: nearest face, argmax ties x<y<z)
  capsule      geometry.py:115-156 (z-axis core, normal (1,0,0) when degenerate)
  frames       geometry.py:172-189 (seed = argmin|n| first on ties; rows t1,t2,n)

Shapes are described by plain tuples so the oracle does not depend on the
product's classes: ("halfspace", normal(3), offset), ("sphere", r),
("box", half_extents(3)), ("capsule", r, half_length).
"""

from __future__ import annotations

import numpy as np


def shape_tuple(shape) -> tuple:
    """Normalise a shape object (product or reference class) to a tuple."""
    if isinstance(shape, tuple):
        return shape
    name = type(shape).__name__.lower()
    if name == "halfspace":
        return ("halfspace", tuple(float(a) for a in shape.normal), float(shape.offset))
    if name == "sphere":
        return ("sphere", float(shape.radius))
    if name == "box":
        return ("box", tuple(float(a) for a in shape.half_extents))
    if name == "capsule":
        return ("capsule", float(shape.radius), float(shape.half_length))
    raise TypeError(f"unknown shape {shape!r}")


def _halfspace(p, nrm, off):
    nrm = np.asarray(nrm, dtype=np.float64)
    phi = p @ nrm - off
    normal = np.tile(nrm, (p.shape[0], 1))
    return phi, normal, p - phi[:, None] * normal


def _sphere(p, r):
    d = np.sqrt(np.sum(p * p, axis=1))
    normal = p / np.maximum(d, 1e-30)[:, None]
    normal[d < 1e-15] = (0.0, 0.0, 1.0)
    return d - r, normal, r * normal


def _box(p, he):
    he = np.asarray(he, dtype=np.float64)
    q = np.abs(p) - he
    out_mask = (q > 0.0).any(axis=1)
    n = p.shape[0]
    phi = np.empty(n)
    normal = np.zeros((n, 3))
    witness = np.clip(p, -he, he)
    if out_mask.any():
        qo = np.maximum(q[out_mask], 0.0)
        d = np.sqrt(np.sum(qo * qo, axis=1))
        phi[out_mask] = d
        normal[out_mask] = (p[out_mask] - witness[out_mask]) / d[:, None]
    ins = np.flatnonzero(~out_mask)
    if ins.size:
        qi = q[ins]
        ax = np.argmax(qi, axis=1)          # first max wins -> x < y < z ties
        r = np.arange(ins.size)
        phi[ins] = qi[r, ax]
        sgn = np.where(p[ins, ax] >= 0.0, 1.0, -1.0)
        nn = np.zeros((ins.size, 3))
        nn[r, ax] = sgn
        normal[ins] = nn
        w = p[ins].copy()
        w[r, ax] = sgn * he[ax]
        witness[ins] = w
    return phi, normal, witness


def _capsule(p, r, hl):
    core = np.zeros_like(p)
    core[:, 2] = np.clip(p[:, 2], -hl, hl)
    rel = p - core
    d = np.sqrt(np.sum(rel * rel, axis=1))
    normal = rel / np.maximum(d, 1e-30)[:, None]
    normal[d < 1e-15] = (1.0, 0.0, 0.0)
    return d - r, normal, core + r * normal


def query(shape, p: np.ndarray):
    s = shape_tuple(shape)
    p = np.asarray(p, dtype=np.float64)
    if s[0] == "halfspace":
        return _halfspace(p, s[1], s[2])
    if s[0] == "sphere":
        return _sphere(p, s[1])
    if s[0] == "box":
        return _box(p, s[1])
    if s[0] == "capsule":
        return _capsule(p, s[1], s[2])
    raise ValueError(s[0])


def frames(normals: np.ndarray) -> np.ndarray:
    """World->contact rotations with rows (t1, t2, n) (geometry.py:172-189)."""
    n = np.asarray(normals, dtype=np.float64)
    k = n.shape[0]
    seed = np.argmin(np.abs(n), axis=1)
    e = np.zeros_like(n)
    e[np.arange(k), seed] = 1.0
    t1 = e - np.sum(e * n, axis=1)[:, None] * n
    t1 = t1 / np.sqrt(np.sum(t1 * t1, axis=1))[:, None]
    t2 = np.cross(n, t1)
    return np.stack([t1, t2, n], axis=1)
