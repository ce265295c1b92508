"""Block-sparse background grid on the GPU.

4x4x4-node blocks keyed by packed block coordinates (reference grid.py:16-132).
``SparseGrid.allocate`` runs the hash-table build kernels (csrc/binning.cu):
candidate blocks are inserted into an open-addressing table, deduplicated,
bitonic-sorted, and each slot stores its block's SORTED index, so block order
(and therefore every node id) is bit-identical to the reference's
``np.unique`` order.  Node lookup is a hash probe, not a binary search.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

BLOCK = 4
BLOCK_NODES = BLOCK ** 3
COORD_BIAS = 1 << 20
MASS_EPS = 1e-12


class AllocationError(RuntimeError):
    """A grid node outside the allocated block set was addressed."""


def _next_pow2(v: int) -> int:
    p = 1
    while p < v:
        p <<= 1
    return p


def pack_block_keys(bcoords) -> torch.Tensor:
    """(n,3) block coords -> sortable int64 keys (grid.py:26-31)."""
    b = _lib.as_dev(bcoords, torch.int64) + COORD_BIAS
    if b.numel() and (int(b.min()) < 0 or int(b.max()) >= (1 << 21)):
        raise AllocationError("block coordinate outside packable range (|coord| < 2^20)")
    return (b[:, 0] << 42) | (b[:, 1] << 21) | b[:, 2]


def base_cells(positions, h: float) -> torch.Tensor:
    """floor(x/h - 0.5) (grid.py:34-36), computed by the device kernel."""
    x = _lib.as_dev(positions)
    out = torch.empty(x.shape, dtype=torch.int64, device=x.device)
    _lib.check(_lib.lib().mpmrb_base_cells(_lib.ctx(), _lib.ptr(x), x.shape[0], float(h),
                                           _lib.ptr(out)))
    return out


class SparseGrid:
    """Node channels live in HBM: mass (N,), mom_apic/mom_force/v_star/v_k/
    v_next (N,3) float64 and active (N,) bool with N = 64 * n_blocks."""

    def __init__(self, h: float, block_keys: torch.Tensor, hash_keys: torch.Tensor,
                 hash_vals: torch.Tensor):
        self.h = float(h)
        self.block_keys = block_keys
        self._hash_keys = hash_keys
        self._hash_vals = hash_vals
        n = self.n_nodes
        self.mass = _lib.zeros((n,))
        self.mom_apic = _lib.zeros((n, 3))
        self.mom_force = _lib.zeros((n, 3))
        self.v_star = _lib.zeros((n, 3))
        self.v_k = _lib.zeros((n, 3))
        self.v_next = _lib.zeros((n, 3))
        self.active = torch.zeros(n, dtype=torch.bool, device=block_keys.device)

    @property
    def n_blocks(self) -> int:
        return int(self.block_keys.shape[0])

    @property
    def n_nodes(self) -> int:
        return self.n_blocks * BLOCK_NODES

    @property
    def block_coords(self) -> torch.Tensor:
        k = self.block_keys
        m = (1 << 21) - 1
        return torch.stack([(k >> 42) - COORD_BIAS, ((k >> 21) & m) - COORD_BIAS,
                            (k & m) - COORD_BIAS], dim=1)

    def view(self) -> _lib.GridView:
        g = _lib.GridView()
        g.block_keys = _lib.ptr(self.block_keys)
        g.hash_keys = _lib.ptr(self._hash_keys)
        g.hash_vals = _lib.ptr(self._hash_vals)
        g.n_blocks = self.n_blocks
        g.hash_cap = int(self._hash_keys.shape[0])
        g.h = self.h
        return g

    @classmethod
    def allocate(cls, positions, h: float) -> "SparseGrid":
        """Blocks covering every 3-wide stencil (grid.py:71-103)."""
        if not (h > 0.0):
            raise ValueError("grid spacing h must be positive")
        x = _lib.as_dev(positions)
        n = x.shape[0]
        cap = max(64, 2 * ((n + 63) // 64) + 64)
        L = _lib.lib()
        for _ in range(4):
            hcap = _next_pow2(max(1024, 4 * cap))
            keys = torch.empty(cap, dtype=torch.int64, device=x.device)
            hk = torch.empty(hcap, dtype=torch.int64, device=x.device)
            hv = torch.empty(hcap, dtype=torch.int32, device=x.device)
            nb = C.c_int64()
            rc = L.mpmrb_grid_allocate(_lib.ctx(), _lib.ptr(x), n, float(h), _lib.ptr(keys), cap,
                                       _lib.ptr(hk), _lib.ptr(hv), hcap, C.byref(nb))
            if rc == _lib.E_CAPACITY:
                cap = int(nb.value) + 64
                continue
            _lib.check(rc)
            return cls(h, keys[: int(nb.value)].clone(), hk, hv)
        raise AllocationError("grid allocation did not converge")

    def node_ids(self, node_coords) -> torch.Tensor:
        """Linear ids of (..., 3) integer node coordinates (grid.py:105-122)."""
        c = _lib.as_dev(node_coords, torch.int64)
        shape = c.shape[:-1]
        flat = c.reshape(-1, 3).contiguous()
        out = torch.empty(flat.shape[0], dtype=torch.int64, device=flat.device)
        g = self.view()
        _lib.check(_lib.lib().mpmrb_node_ids(_lib.ctx(), C.byref(g), _lib.ptr(flat),
                                             flat.shape[0], _lib.ptr(out)))
        return out.reshape(shape)

    def node_coords(self, node_ids) -> torch.Tensor:
        ids = _lib.as_dev(node_ids, torch.int64)
        blk = ids // BLOCK_NODES
        r = ids % BLOCK_NODES
        loc = torch.stack([r // (BLOCK * BLOCK), (r // BLOCK) % BLOCK, r % BLOCK], dim=-1)
        return self.block_coords[blk] * BLOCK + loc

    def node_positions(self, node_ids) -> torch.Tensor:
        return self.node_coords(node_ids).to(torch.float64) * self.h
