"""Oracle: particle binning, block-sparse grid and quadratic B-spline stencils.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  base cells            /root/reference/pkg/src/mpmrb/grid.py:34-36
  block-key packing      grid.py:16-19, 26-31
  grid allocation        grid.py:71-103
  node-id lookup         grid.py:105-122, node coords grid.py:124-132
  truncated Morton key   transfer.py:34-35, 44-61
  sort plan              transfer.py:64-102, staleness transfer.py:105-113
  deterministic scatter  transfer.py:135-187 (id-ordered np.bincount)
  stencil                mpm.py:25, 28-53
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BLOCK_EDGE = 4
NODES_PER_BLOCK = 64
BIAS21 = 1 << 20
MASK21 = (1 << 21) - 1
MASS_EPS = 1e-12
MORTON_KEEP_BITS = 10

# x-major offset table (mpm.py:25): slot k = 9*ox + 3*oy + oz
STENCIL_OFFSETS = np.array([[a, b, c] for a in range(3) for b in range(3) for c in range(3)],
                           dtype=np.int64)


class OracleAllocationError(RuntimeError):
    pass


def base_cells(x: np.ndarray, h: float) -> np.ndarray:
    """floor(x/h - 0.5) with IEEE division then subtraction (grid.py:34-36)."""
    q = np.asarray(x, dtype=np.float64) / h
    return np.floor(q - 0.5).astype(np.int64)


def pack_blocks(b: np.ndarray) -> np.ndarray:
    """(m,3) block coords -> int64 keys, 21 biased bits per axis (grid.py:26-31)."""
    biased = np.asarray(b, dtype=np.int64) + BIAS21
    if biased.size and ((biased < 0).any() or (biased > MASK21).any()):
        raise OracleAllocationError("block coordinate outside packable range")
    return (biased[:, 0] << 42) | (biased[:, 1] << 21) | biased[:, 2]


def unpack_blocks(keys: np.ndarray) -> np.ndarray:
    k = np.asarray(keys, dtype=np.int64)
    return np.stack([(k >> 42) - BIAS21, ((k >> 21) & MASK21) - BIAS21,
                     (k & MASK21) - BIAS21], axis=1)


def allocate_blocks(x: np.ndarray, h: float) -> np.ndarray:
    """Sorted unique keys of every block touched by a 3-wide stencil (grid.py:71-103).

    Each axis contributes block base>>2 and (base+2)>>2 (grid.py:82-96).
    """
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] == 0:
        return np.zeros(0, dtype=np.int64)
    if not np.isfinite(x).all():
        raise OracleAllocationError("non-finite particle positions")
    base = base_cells(x, h)
    lo = base >> 2
    hi = (base + 2) >> 2
    corners = []
    for sx in (lo[:, 0], hi[:, 0]):
        for sy in (lo[:, 1], hi[:, 1]):
            for sz in (lo[:, 2], hi[:, 2]):
                corners.append(np.stack([sx, sy, sz], axis=1))
    return np.unique(pack_blocks(np.concatenate(corners)))


def lookup_nodes(block_keys: np.ndarray, coords: np.ndarray) -> np.ndarray:
    """Linear node ids of integer node coordinates (..., 3) (grid.py:105-122)."""
    flat = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    keys = pack_blocks(flat >> 2)
    pos = np.searchsorted(block_keys, keys)
    nb = block_keys.shape[0]
    ok = pos < nb
    pos_c = np.where(ok, pos, 0)
    ok &= (block_keys[pos_c] == keys) if nb else np.zeros_like(ok)
    if not ok.all():
        raise OracleAllocationError(f"{int((~ok).sum())} stencil nodes outside allocated blocks")
    loc = flat & 3
    lin = pos_c * NODES_PER_BLOCK + loc[:, 0] * 16 + loc[:, 1] * 4 + loc[:, 2]
    return lin.reshape(np.asarray(coords).shape[:-1])


def node_coords(block_keys: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Integer coordinates of linear node ids (grid.py:124-129)."""
    ids = np.asarray(ids, dtype=np.int64)
    blk = unpack_blocks(block_keys)[ids // NODES_PER_BLOCK]
    r = ids % NODES_PER_BLOCK
    return blk * BLOCK_EDGE + np.stack([r // 16, (r // 4) % 4, r % 4], axis=-1)


# ---------------------------------------------------------------- Morton / plan

def _spread3(v: np.ndarray) -> np.ndarray:
    """Insert two zero bits between each of the low 21 bits (transfer.py:44-52).

    Implemented bit by bit (the reference uses the magic-mask cascade); the
    result is identical for every 21-bit input.
    """
    v = np.asarray(v, dtype=np.int64) & MASK21
    out = np.zeros_like(v)
    for i in range(21):
        out |= ((v >> i) & 1) << (3 * i)
    return out


def morton10(cells: np.ndarray) -> np.ndarray:
    """Low 10 bits of the biased Morton interleave, uint16 (transfer.py:55-61)."""
    c = np.asarray(cells, dtype=np.int64) + BIAS21
    if (c < 0).any() or (c > MASK21).any():
        raise ValueError("cell coordinate outside Morton range (|coord| < 2^20)")
    full = _spread3(c[:, 0]) | (_spread3(c[:, 1]) << 1) | (_spread3(c[:, 2]) << 2)
    return (full & ((1 << MORTON_KEEP_BITS) - 1)).astype(np.uint16)


@dataclass
class Plan:
    epoch: int
    keys: np.ndarray
    perm: np.ndarray
    inv_perm: np.ndarray
    bin_keys: np.ndarray
    bin_starts: np.ndarray
    bin_of: np.ndarray


def sort_plan(x: np.ndarray, h: float, epoch: int) -> Plan:
    """Stable key sort and bin run-lengths (transfer.py:85-102)."""
    keys = morton10(base_cells(x, h))
    n = keys.shape[0]
    perm = np.argsort(keys, kind="stable").astype(np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n, dtype=np.int64)
    sk = keys[perm]
    if n:
        heads = np.concatenate(([True], sk[1:] != sk[:-1]))
        starts = np.append(np.flatnonzero(heads), n).astype(np.int64)
        bkeys = sk[heads]
    else:
        starts = np.zeros(1, dtype=np.int64)
        bkeys = np.zeros(0, dtype=np.uint16)
    bin_of = np.searchsorted(bkeys, keys).astype(np.int64)
    return Plan(epoch, keys, perm, inv, bkeys, starts, bin_of)


def staleness(plan: Plan, x: np.ndarray, h: float) -> float:
    """Fraction of particles whose key moved since the plan (transfer.py:105-113)."""
    if plan.keys.shape[0] == 0:
        return 0.0
    return float(np.mean(morton10(base_cells(x, h)) != plan.keys))


def scatter_in_order(node_ids: np.ndarray, values: np.ndarray, n_out: int) -> np.ndarray:
    """Sum (rows, k[, C]) contributions in row-major order (transfer.py:135-187).

    One bincount per channel accumulates entries in input order, which is the
    reference's deterministic (particle-id) summation order.
    """
    squeeze = values.ndim == 2
    vals = values[..., None] if squeeze else values
    idx = np.asarray(node_ids, dtype=np.int64).ravel()
    out = np.empty((n_out, vals.shape[-1]))
    for ch in range(vals.shape[-1]):
        out[:, ch] = np.bincount(idx, weights=vals[..., ch].ravel(), minlength=n_out)
    return out[:, 0] if squeeze else out


# ---------------------------------------------------------------- stencil

@dataclass
class Stencil:
    base: np.ndarray     # (n,3)
    weights: np.ndarray  # (n,27)
    nodes: np.ndarray    # (n,27)
    dpos: np.ndarray     # (n,27,3)
    h: float


def bspline_1d(fx: np.ndarray) -> np.ndarray:
    """Quadratic B-spline weights of offsets 0,1,2 for fx in [0.5,1.5) (mpm.py:42-46)."""
    return np.stack([0.5 * (1.5 - fx) ** 2, 0.75 - (fx - 1.0) ** 2, 0.5 * (fx - 0.5) ** 2],
                    axis=1)


def make_stencil(x: np.ndarray, block_keys: np.ndarray, h: float) -> Stencil:
    """Weights, node ids and node-minus-particle offsets (mpm.py:39-53)."""
    x = np.asarray(x, dtype=np.float64)
    base = base_cells(x, h)
    fx = x / h - base
    w1 = bspline_1d(fx)                                     # (n, 3 offsets, 3 axes)
    o = STENCIL_OFFSETS
    weights = w1[:, o[:, 0], 0] * w1[:, o[:, 1], 1] * w1[:, o[:, 2], 2]
    nodes = lookup_nodes(block_keys, base[:, None, :] + o[None, :, :])
    dpos = (o[None, :, :] - fx[:, None, :]) * h
    return Stencil(base=base, weights=weights, nodes=nodes, dpos=dpos, h=h)
