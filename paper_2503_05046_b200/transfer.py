"""Partial-sort binning and the scatter contract.

* ``build_sort_plan`` (transfer.py:85-102): one-pass stable 10-bit Morton
  counting sort on the GPU (csrc/binning.cu); keys, perm, inv_perm, bins are
  bit-identical to the reference's stable argsort.
* ``scatter_reduce`` (transfer.py:148-248): float64 REDG atomics.  The
  reference's "deterministic" mode sums in particle-id order; atomics cannot
  reproduce that order bitwise, so both modes here agree with the reference to
  floating-point reassociation (the reference's own fast-mode bound,
  <= 1e-12 * max, test_transfer.py:85-93).  The plan/epoch/mode contract and
  errors are kept exactly.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

MORTON_BITS = 10
CELL_BIAS = 1 << 20
_WORKER_ENV = "MPMRB_WORKERS"


class PlanEpochError(RuntimeError):
    """A SortPlan from a different coupling step was used."""


def morton_keys(cells) -> torch.Tensor:
    """Low 10 bits of the biased Morton interleave of (n,3) cells (transfer.py:55-61)."""
    c = _lib.as_dev(cells, torch.int64) + CELL_BIAS
    if c.numel() and (int(c.min()) < 0 or int(c.max()) >= (1 << 21)):
        raise ValueError("cell coordinate outside Morton range (|coord| < 2^20)")
    k = torch.zeros(c.shape[0], dtype=torch.int64, device=c.device)
    for i in range(4):
        for a in range(3):
            bit = 3 * i + a
            if bit < MORTON_BITS:
                k |= ((c[:, a] >> i) & 1) << bit
    return k.to(torch.int32).to(torch.uint16) if hasattr(torch, "uint16") else k


@dataclass
class SortPlan:
    """Bin assignment of one particle set, valid for a single coupling step."""

    epoch: int
    keys: torch.Tensor        # (n,) uint16
    perm: torch.Tensor        # (n,) int64
    inv_perm: torch.Tensor    # (n,) int64
    bin_keys: torch.Tensor    # (nb,) uint16
    bin_starts: torch.Tensor  # (nb+1,) int64
    bin_of: torch.Tensor      # (n,) int64

    @property
    def n_particles(self) -> int:
        return int(self.keys.shape[0])

    @property
    def n_bins(self) -> int:
        return int(self.bin_keys.shape[0])


def build_sort_plan(positions, h: float, epoch: int) -> SortPlan:
    x = _lib.as_dev(positions)
    n = x.shape[0]
    dev = x.device
    keys = torch.empty(n, dtype=torch.uint16, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    inv = torch.empty(n, dtype=torch.int64, device=dev)
    bkeys = torch.empty(1024, dtype=torch.uint16, device=dev)
    bstarts = torch.empty(1025, dtype=torch.int64, device=dev)
    bin_of = torch.empty(n, dtype=torch.int64, device=dev)
    nb = C.c_int64()
    _lib.check(_lib.lib().mpmrb_sort_plan(_lib.ctx(), _lib.ptr(x), n, float(h), _lib.ptr(keys),
                                          _lib.ptr(perm), _lib.ptr(inv), _lib.ptr(bkeys),
                                          _lib.ptr(bstarts), _lib.ptr(bin_of), C.byref(nb)))
    k = int(nb.value)
    return SortPlan(epoch=int(epoch), keys=keys, perm=perm, inv_perm=inv,
                    bin_keys=bkeys[:k].clone(), bin_starts=bstarts[: k + 1].clone(),
                    bin_of=bin_of)


def plan_staleness(plan: SortPlan, positions, h: float) -> float:
    """Fraction of particles whose key changed since the plan (transfer.py:105-113)."""
    x = _lib.as_dev(positions)
    if x.shape[0] != plan.n_particles:
        raise ValueError("plan was built for a different particle count")
    if plan.n_particles == 0:
        return 0.0
    out = C.c_double()
    _lib.check(_lib.lib().mpmrb_plan_staleness(_lib.ctx(), _lib.ptr(plan.keys), _lib.ptr(x),
                                               x.shape[0], float(h), C.byref(out)))
    return float(out.value)


def resolve_workers(workers: int | None) -> int:
    """Kept for API compatibility (transfer.py:116-122); the GPU ignores it."""
    if workers is None:
        workers = min(4, os.cpu_count() or 1)
    cap = os.environ.get(_WORKER_ENV)
    if cap:
        workers = min(workers, max(1, int(cap)))
    return max(1, int(workers))


@dataclass
class ScatterStats:
    merges_performed: int = 0
    nodes_touched: int = 0
    chunks: int = 0
    rows: int = 0


def scatter_reduce(node_ids, values, n_out: int, plan: SortPlan, epoch: int,
                   mode: str = "deterministic", workers: int | None = None, particle_ids=None,
                   stats: ScatterStats | None = None) -> torch.Tensor:
    """Sum (rows, k[, C]) stencil contributions into (n_out[, C]) node channels."""
    if epoch != plan.epoch:
        raise PlanEpochError(f"plan epoch {plan.epoch} used in step {epoch}")
    if mode not in ("deterministic", "fast"):
        raise ValueError(f"unknown scatter mode {mode!r}")
    vals = _lib.as_dev(values)
    ids = _lib.as_dev(node_ids, torch.int64)
    squeeze = vals.dim() == 2
    if squeeze:
        vals = vals[..., None].contiguous()
    rows, k, nch = vals.shape
    if tuple(ids.shape) != (rows, k):
        raise ValueError("node_ids and values disagree on rows/slots")
    if particle_ids is None and rows != plan.n_particles:
        raise ValueError("row count does not match the plan's particle count")
    out = torch.empty((n_out, nch), dtype=torch.float64, device=vals.device)
    # Both modes run the ordered segmented fold: bitwise the reference's
    # bincount order (transfer.py:135-145).  The reference's fast mode only
    # promises a result within 1e-12 of deterministic that repeats for a given
    # worker count (test_transfer.py:77-102); the ordered fold meets that
    # exactly.  The unordered float64-atomic scatter is scatter_naive.
    fn = _lib.lib().mpmrb_scatter_reduce_ordered
    _lib.check(fn(_lib.ctx(), _lib.ptr(ids), _lib.ptr(vals), rows, k, nch, n_out, _lib.ptr(out)))
    if stats is not None:
        touched = int(torch.unique(ids).numel()) if rows else 0
        stats.rows = rows
        stats.chunks = 1
        stats.merges_performed = touched
        stats.nodes_touched = touched
    return out[:, 0] if squeeze else out


def scatter_naive(node_ids, values, n_out: int) -> torch.Tensor:
    """transfer.py:251-260's per-contribution baseline: on the GPU, one float64
    atomic per contribution (summation order unspecified)."""
    vals = _lib.as_dev(values)
    ids = _lib.as_dev(node_ids, torch.int64)
    squeeze = vals.dim() == 2
    if squeeze:
        vals = vals[..., None].contiguous()
    rows, k, nch = vals.shape
    out = torch.empty((n_out, nch), dtype=torch.float64, device=vals.device)
    _lib.check(_lib.lib().mpmrb_scatter_reduce(_lib.ctx(), _lib.ptr(ids), _lib.ptr(vals), rows, k,
                                               nch, n_out, _lib.ptr(out)))
    return out[:, 0] if squeeze else out
