"""MLS/APIC transfers on quadratic B-splines, on the GPU.

Same entry points as the reference mpm.py:25-138.  The kernels never
materialise the (n,27) stencil: weights, node ids and offsets are recomputed in
registers from x (csrc/common.cuh make_stencil1 / resolve_blocks).
``build_stencil`` exists for API parity and tests and does materialise them.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from itertools import product

import numpy as np
import torch

from . import _lib
from .grid import SparseGrid
from .materials import Material, material_table
from .particles import ParticleSet
from .transfer import PlanEpochError, ScatterStats, SortPlan

# canonical stencil slot order: x-major offsets (mpm.py:25)
OFFSETS = np.array(list(product(range(3), repeat=3)), dtype=np.int64)


@dataclass
class Stencil:
    base: torch.Tensor     # (n,3) int64
    weights: torch.Tensor  # (n,27)
    nodes: torch.Tensor    # (n,27) int64
    dpos: torch.Tensor     # (n,27,3)
    h: float


def build_stencil(positions, grid: SparseGrid) -> Stencil:
    """mpm.py:39-53; AllocationError when a node falls outside the grid."""
    from .grid import base_cells
    x = _lib.as_dev(positions)
    n = x.shape[0]
    w = _lib.empty((n, 27))
    nodes = torch.empty((n, 27), dtype=torch.int64, device=x.device)
    dpos = _lib.empty((n, 27, 3))
    g = grid.view()
    _lib.check(_lib.lib().mpmrb_build_stencil(_lib.ctx(), C.byref(g), _lib.ptr(x), n,
                                              _lib.ptr(w), _lib.ptr(nodes), _lib.ptr(dpos)))
    return Stencil(base=base_cells(x, grid.h), weights=w, nodes=nodes, dpos=dpos, h=grid.h)


def compute_stresses(particles: ParticleSet, materials: list[Material]) -> torch.Tensor:
    """Kirchhoff stress per particle (mpm.py:56-63)."""
    tab, nm = material_table(materials)
    tau = torch.empty_like(particles.f)
    _lib.check(_lib.lib().mpmrb_compute_stresses(_lib.ctx(), _lib.ptr(particles.f),
                                                 _lib.ptr(particles.material_id), particles.n,
                                                 tab, nm, _lib.ptr(tau)))
    return tau


def particle_to_grid(particles: ParticleSet, grid: SparseGrid, stencil: Stencil | None,
                     materials: list[Material], dt: float, plan: SortPlan, epoch: int,
                     mode: str = "deterministic", workers: int | None = None,
                     stats: ScatterStats | None = None) -> None:
    """Fill grid.mass, grid.mom_apic, grid.mom_force (mpm.py:66-99).
    ``mode="deterministic"`` (the reference's default) materialises the
    (n, 27, 7) contributions and sums every node channel in particle-id /
    slot order (ordered scatter: bitwise reproducible, plan-independent);
    ``mode="fast"`` is the fused path's kernel: stress, then warp-private
    shared-memory node tiles flushed with one float64 atomic per (node,
    channel), within the reference's fast-vs-deterministic bound.
    ``stencil`` is accepted for API compatibility; the kernels recompute it
    from particles.x."""
    if epoch != plan.epoch:
        raise PlanEpochError(f"plan epoch {plan.epoch} used in step {epoch}")
    if mode not in ("deterministic", "fast"):
        raise ValueError(f"unknown scatter mode {mode!r}")
    tab, nm = material_table(materials)
    g = grid.view()
    pv = particles.view()
    fn = _lib.lib().mpmrb_p2g_ordered if mode == "deterministic" else _lib.lib().mpmrb_p2g
    _lib.check(fn(_lib.ctx(), C.byref(g), C.byref(pv), tab, nm, float(dt), _lib.ptr(grid.mass),
                  _lib.ptr(grid.mom_apic), _lib.ptr(grid.mom_force)))
    if stats is not None:
        stats.rows = particles.n
        stats.chunks = 1


def grid_update(grid: SparseGrid, gravity, dt: float) -> None:
    """v_k, v* and the active mask (mpm.py:102-115)."""
    g = (C.c_double * 3)(*[float(a) for a in np.asarray(_lib.to_numpy(gravity)).ravel()])
    _lib.check(_lib.lib().mpmrb_grid_update(_lib.ctx(), grid.n_nodes, _lib.ptr(grid.mass),
                                            _lib.ptr(grid.mom_apic), _lib.ptr(grid.mom_force), g,
                                            float(dt), _lib.ptr(grid.active), _lib.ptr(grid.v_k),
                                            _lib.ptr(grid.v_star)))


def grid_to_particle(particles: ParticleSet, grid: SparseGrid, stencil: Stencil | None,
                     dt: float, materials: list[Material] | None = None) -> int:
    """Gather v_next, update v, C, x, F in place (mpm.py:118-138); clamps
    inverted F (materials.py:86-110); applies the sand return map when
    ``materials`` is given.  Returns the number of clamped F."""
    tab, nm = material_table(materials or [])
    if materials is None:
        # elastic-only semantics of the reference: every id maps to an elastic entry
        nmax = int(particles.material_id.max()) + 1 if particles.n else 1
        tab, nm = material_table([Material(1.0, 0.0, 1.0)] * nmax)
    v_next = grid.v_next.contiguous()
    g = grid.view()
    pv = particles.view()
    ncl = C.c_int64()
    _lib.check(_lib.lib().mpmrb_g2p(_lib.ctx(), C.byref(g), C.byref(pv), tab, nm,
                                    _lib.ptr(v_next), float(dt), C.byref(ncl)))
    return int(ncl.value)
