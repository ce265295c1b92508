"""Codimensional cloth meshes (NEW; parity unpinned — the reference has no
cloth).

The paper simulates cloth "with a particle at each mesh vertex and at the
centroid of each triangle face, following Jiang et al. 2017".
A ``ClothMesh`` holds that mesh on the device in the user's particle order:
triangles of vertex-particle indices, the element particle of each triangle,
the rest inverse Dm^-1, rest volume and the transverse direction d3 (state,
advanced by the fused substep, csrc/cloth.cu), plus the per-particle roles.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

ROLE_NONE, ROLE_VERTEX, ROLE_ELEMENT = _lib.CLOTH_NONE, _lib.CLOTH_VERTEX, _lib.CLOTH_ELEMENT


@dataclass
class ClothMesh:
    tri: torch.Tensor     # (ne, 3) int32 vertex particle indices
    epart: torch.Tensor   # (ne,) int32 element particle index
    dm_inv: torch.Tensor  # (ne, 2, 2) float64
    vol: torch.Tensor     # (ne,) float64 rest volume (area x thickness)
    d3: torch.Tensor      # (ne, 3) float64 transverse direction (state)
    role: torch.Tensor    # (n,) int8 per-particle role

    @property
    def n_elements(self) -> int:
        return int(self.tri.shape[0])

    @classmethod
    def from_arrays(cls, tri, epart, dm_inv, vol, d3, role) -> "ClothMesh":
        return cls(tri=_lib.as_dev(tri, torch.int32), epart=_lib.as_dev(epart, torch.int32),
                   dm_inv=_lib.as_dev(dm_inv), vol=_lib.as_dev(vol), d3=_lib.as_dev(d3),
                   role=_lib.as_dev(role, torch.int8))

    def offset(self, first_particle: int, n_total: int) -> "ClothMesh":
        """The same mesh with its particle indices shifted (concatenated sets)."""
        role = torch.zeros(n_total, dtype=torch.int8, device=self.role.device)
        role[first_particle:first_particle + self.role.shape[0]] = self.role
        return ClothMesh(self.tri + first_particle, self.epart + first_particle, self.dm_inv,
                         self.vol, self.d3, role)


def sheet_arrays(center, size, n_side: int, thickness: float, rho: float,
                 normal_axis: int = 2) -> dict:
    """Host arrays of a square sheet: n_side^2 vertex particles on a lattice,
    2 (n_side-1)^2 triangles, one element particle per triangle centroid.
    Mass rho * area * thickness per triangle, half on the element particle and
    a sixth on each vertex; the element particle's rest volume is the element
    volume (its transverse stress acts through it), d3 = the sheet normal."""
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
    i, j = np.meshgrid(np.arange(n_side - 1), np.arange(n_side - 1), indexing="ij")
    a = (i * n_side + j).ravel()
    b, c, d = a + n_side, a + 1, a + n_side + 1
    tri = np.stack([np.stack([a, b, d], 1), np.stack([a, d, c], 1)], 1).reshape(-1, 3)
    ne = tri.shape[0]
    uv = np.stack([U.ravel(), V.ravel()], axis=1)
    dm = np.stack([uv[tri[:, 1]] - uv[tri[:, 0]], uv[tri[:, 2]] - uv[tri[:, 0]]], axis=-1)
    area = 0.5 * np.abs(np.linalg.det(dm))
    nrm = np.zeros(3)
    nrm[normal_axis] = 1.0
    d1 = xv[tri[:, 1]] - xv[tri[:, 0]]
    d2 = xv[tri[:, 2]] - xv[tri[:, 0]]
    d3 = np.sign(np.cross(d1, d2) @ nrm)[:, None] * nrm[None, :]
    m_tri = rho * area * thickness
    mass = np.zeros(nv + ne)
    for k in range(3):
        mass[:nv] += np.bincount(tri[:, k], weights=m_tri / 6.0, minlength=nv)
    mass[nv:] = 0.5 * m_tri
    vol = mass / rho
    vol[nv:] = area * thickness
    role = np.concatenate([np.full(nv, ROLE_VERTEX, np.int8), np.full(ne, ROLE_ELEMENT, np.int8)])
    return dict(x=np.concatenate([xv, xv[tri].mean(axis=1)]), mass=mass, vol=vol, tri=tri,
                epart=np.arange(nv, nv + ne), dm_inv=np.linalg.inv(dm), vol_e=area * thickness,
                d3=d3, role=role)
