"""Slab domain decomposition of ONE scene over ranks (second
bullet): the north-star's "slab domain decomposition of large scenes with P2G
halo exchange".  No reference counterpart: the reference is single-process.

Layout.  Rank r owns the particles whose x (``axis``) lies in the slab
[X_r, X_{r+1}); the interior bounds are equal-count quantiles of the initial
positions snapped to grid-block boundaries (multiples of 4h).  Particles
migrate once per rigid step, at its start (the reference builds its sort plan
once per step too, ``coupling.py:168-219``).  Each substep (``coupling.py:
115-150``) then runs the same fine-grained device operators as
``coupling.advance_step_ops`` on the rank's particles, with three exchanges:

1. **P2G halo reduce.**  After P2G, every rank sends the 7 node channels of its
   blocks within two blocks of a slab boundary (particles drift at most that
   far within a step; checked) and adds the channels of every block it shares
   with a neighbour.  A block is shared by at most two ranks and IEEE addition
   commutes, so both copies of a shared node hold bitwise-identical sums and
   the grid update agrees on both sides.
2. **Contact solve**, one of two modes (``SlabState.solve``).
   ``"gather0"`` (default): the contact solve is latency-bound (DESIGN.md
   §3), so the contact problem -- contacts with their stencils keyed by global
   node coordinates, the contact nodes' (m, v*, v_k), and three scalars per
   rank summarising its contact-free active nodes -- is gathered to rank 0
   once per substep and solved by the fused solver
   (``quasi_newton_solve_ext``).  Contact-free nodes enter every reduction in
   closed form (g = m (v - v*), H = m I), so the global problem is exactly
   the single-scene one.
   ``"allreduce"``: the solve runs on every rank (``_solve_allreduce``).
   Contacts stay where they were detected, the contact-node state is
   replicated, one vector all-reduce per iteration sums J^T dl/dv_c and the
   Hessian blocks, and every line-search evaluation all-reduces the two
   scalars phi'(alpha), phi''(alpha) (solver.py:301-325).
3. **Solution scatter** (gather0 mode).  Rank 0 broadcasts the contact-node velocities,
   P = prod(1 - alpha) (free nodes finish at v* + P (v_k - v*)), the impulses
   and the solve report.  Reactions accumulate per rank; the step wrench is
   all-reduced, so every rank advances the (replicated) rigid bodies alike.

Node ownership (each active node counted once in the free-node sums and the
statistics): a node of a block shared with a neighbour belongs to the rank
whose slab contains the node's coordinate; a node of an unshared block belongs
to the only rank that has it.

The P2G halos and the particle migration are point-to-point exchanges with the
two adjacent ranks only (``Comm.neighbours``, batch_isend_irecv); the contact
problem is gathered to rank 0 (``Comm.gather0``).  The communication layer
works on CPU tensors under gloo (tests, and several ranks sharing one GPU) and
on device tensors under NCCL.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import coupling as _coupling
from .collision import BiasCache, contact_velocities, detect_contacts
from .contact_model import normal_impulse
from .coupling import ImpulseAccumulator, SimState, StepSummary, _rigid_update
from .grid import BLOCK_NODES, COORD_BIAS, SparseGrid
from .mpm import build_stencil, grid_to_particle, grid_update, particle_to_grid
from .particles import ParticleSet
from .solver import ContactProblem, SolveReport, quasi_newton_solve_ext
from .transfer import build_sort_plan, plan_staleness

BLOCK_EDGE = 4
HALO_BLOCKS = 2       # blocks on each side of a slab bound that may be shared
MIN_SLAB_BLOCKS = 2 * HALO_BLOCKS  # halo bands of adjacent bounds never overlap
PARTICLE_FIELDS = ("x", "v", "f", "c", "mass", "volume0", "material_id", "plastic")


# ------------------------------------------------------------------ pure logic

def slab_bounds(x_axis: np.ndarray, world: int, h: float) -> np.ndarray:
    """Interior slab bounds: equal-count quantiles of the positions snapped to
    block boundaries; returns [-inf, X_1, ..., X_{W-1}, +inf]."""
    if world == 1:
        return np.array([-np.inf, np.inf])
    width = BLOCK_EDGE * h
    qs = np.quantile(np.asarray(x_axis, float), np.arange(1, world) / world)
    blocks = np.round(qs / width).astype(np.int64)
    for k in range(1, len(blocks)):
        blocks[k] = max(blocks[k], blocks[k - 1] + MIN_SLAB_BLOCKS)
    bounds = np.concatenate([[-np.inf], blocks * width, [np.inf]])
    counts = np.bincount(np.searchsorted(bounds[1:-1], x_axis, side="right"), minlength=world)
    if counts.min() == 0:
        raise ValueError(f"scene too narrow for {world} slabs of >= {MIN_SLAB_BLOCKS} blocks")
    return bounds


def slab_of(x_axis: torch.Tensor, bounds: np.ndarray) -> torch.Tensor:
    """Owning rank of each position (slab [X_r, X_{r+1}))."""
    inner = torch.as_tensor(bounds[1:-1], dtype=x_axis.dtype, device=x_axis.device)
    return torch.searchsorted(inner, x_axis.contiguous(), right=True)


def pack_coords(c: torch.Tensor) -> torch.Tensor:
    """(k,3) int64 node coordinates -> global 63-bit keys (grid.py:26-31 packing)."""
    c = c.to(torch.int64) + COORD_BIAS
    return (c[:, 0] << 42) | (c[:, 1] << 21) | c[:, 2]


def node_coords(block_coords: torch.Tensor, node_ids: torch.Tensor) -> torch.Tensor:
    """Global coordinates of local node ids (node = block * 64 + (lx*4+ly)*4+lz)."""
    b = node_ids // BLOCK_NODES
    lid = node_ids % BLOCK_NODES
    off = torch.stack([lid >> 4, (lid >> 2) & 3, lid & 3], dim=1)
    return block_coords[b] * BLOCK_EDGE + off


def halo_band(block_axis: torch.Tensor, bounds: np.ndarray, rank: int, h: float,
              side: str = "both") -> torch.Tensor:
    """Blocks within HALO_BLOCKS of this rank's interior slab bounds: its left
    bound (shared with rank - 1), its right bound (rank + 1), or both."""
    band = torch.zeros_like(block_axis, dtype=torch.bool)
    width = BLOCK_EDGE * h
    ks = {"left": (rank,), "right": (rank + 1,), "both": (rank, rank + 1)}[side]
    for k in ks:
        if 0 < k < len(bounds) - 1:
            bX = int(round(bounds[k] / width))
            band |= (block_axis >= bX - HALO_BLOCKS) & (block_axis < bX + HALO_BLOCKS)
    return band


def match_keys(mine_sorted: torch.Tensor, theirs: torch.Tensor):
    """Positions of ``theirs`` in the sorted ``mine_sorted`` (or -1)."""
    if mine_sorted.numel() == 0 or theirs.numel() == 0:
        return torch.full_like(theirs, -1)
    pos = torch.searchsorted(mine_sorted, theirs).clamp(max=mine_sorted.numel() - 1)
    return torch.where(mine_sorted[pos] == theirs, pos, torch.full_like(pos, -1))


def node_owned(coords_axis: torch.Tensor, block_shared: torch.Tensor, bounds: np.ndarray,
               rank: int, h: float) -> torch.Tensor:
    """Ownership of active nodes: by coordinate in shared blocks, else mine."""
    slab = slab_of(coords_axis.to(torch.float64) * h, bounds)
    return (~block_shared) | (slab == rank)


def free_sums(m, v_star, v0) -> torch.Tensor:
    """(S0, Q0, Q1) of contact-free nodes (solver.cu closed form)."""
    e = v0 - v_star
    return torch.stack([(m[:, None] * e * e).sum(), (m[:, None] * v_star * v_star).sum(),
                        (m[:, None] * v_star * e).sum()])


# ------------------------------------------------------------------ communication

class Comm:
    """torch.distributed wrapper: variable-size all-gathers / broadcasts on the
    backend's device (CPU under gloo, the rank's GPU under NCCL)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self.dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def allgather(self, t: torch.Tensor) -> list[torch.Tensor]:
        """All ranks' tensors (same trailing shape and dtype; any row count)."""
        if self.world == 1:
            return [t]
        src = t.to(self.dev).contiguous()
        n = torch.tensor([src.shape[0]], dtype=torch.int64, device=self.dev)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(k.item()) for k in ns]
        cap = max(max(ns), 1)
        pad = torch.zeros((cap,) + tuple(src.shape[1:]), dtype=src.dtype, device=self.dev)
        pad[: src.shape[0]] = src
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return [o[:k].to(t.device) for o, k in zip(outs, ns)]

    def neighbours(self, to_left: torch.Tensor | None, to_right: torch.Tensor | None):
        """Exchange with the adjacent ranks only: send ``to_left`` to rank - 1
        and ``to_right`` to rank + 1 (same trailing shape and dtype, any row
        count); returns (from_left, from_right), None at the ends of the
        chain.  Point-to-point (batch_isend_irecv): two neighbours per rank
        whatever the world size, instead of an all-gather to every rank."""
        if self.world == 1:
            return None, None
        have = [(self.rank - 1, to_left), (self.rank + 1, to_right)]
        have = [(q, t) for q, t in have if 0 <= q < self.world]
        proto = next(t for _, t in have if t is not None)
        tail, dtype = tuple(proto.shape[1:]), proto.dtype
        # 1. row counts
        sends, recvs, ops = {}, {}, []
        for q, t in have:
            sends[q] = torch.tensor([t.shape[0]], dtype=torch.int64, device=self.dev)
            recvs[q] = torch.zeros(1, dtype=torch.int64, device=self.dev)
            ops.append(dist.P2POp(dist.isend, sends[q], q, group=self.group))
            ops.append(dist.P2POp(dist.irecv, recvs[q], q, group=self.group))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        # 2. payloads
        ops, bufs = [], {}
        for q, t in have:
            k = int(recvs[q].item())
            bufs[q] = torch.empty((k,) + tail, dtype=dtype, device=self.dev)
            if t.shape[0]:
                ops.append(dist.P2POp(dist.isend, t.to(self.dev).contiguous(), q, group=self.group))
            if k:
                ops.append(dist.P2POp(dist.irecv, bufs[q], q, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        dev = proto.device
        left = bufs[self.rank - 1].to(dev) if (self.rank - 1) in bufs else None
        right = bufs[self.rank + 1].to(dev) if (self.rank + 1) in bufs else None
        return left, right

    def gather0(self, t: torch.Tensor) -> list[torch.Tensor] | None:
        """Every rank's tensor on rank 0 (None elsewhere); any row count."""
        if self.world == 1:
            return [t]
        src = t.to(self.dev).contiguous()
        n = torch.tensor([src.shape[0]], dtype=torch.int64, device=self.dev)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(k.item()) for k in ns]
        cap = max(max(ns), 1)
        pad = torch.zeros((cap,) + tuple(src.shape[1:]), dtype=src.dtype, device=self.dev)
        pad[: src.shape[0]] = src
        outs = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(pad, outs, dst=0, group=self.group)
        if self.rank != 0:
            return None
        return [o[:k].to(t.device) for o, k in zip(outs, ns)]

    def sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        x = t.to(self.dev).clone()
        dist.all_reduce(x, group=self.group)
        return x.to(t.device)

    def bcast(self, t: torch.Tensor | None, shape_dtype=None, src: int = 0) -> torch.Tensor:
        """Broadcast from ``src``; other ranks pass None and receive any shape."""
        if self.world == 1:
            return t
        if self.rank == src:
            x = t.to(self.dev).contiguous()
            meta = torch.tensor([x.dim()] + list(x.shape) + [0] * (4 - x.dim()),
                                dtype=torch.int64, device=self.dev)
        else:
            meta = torch.zeros(5, dtype=torch.int64, device=self.dev)
        dist.broadcast(meta, src, group=self.group)
        shape = tuple(int(s) for s in meta[1: 1 + int(meta[0])].tolist())
        dtype = shape_dtype if shape_dtype is not None else (t.dtype if t is not None else torch.float64)
        if self.rank != src:
            x = torch.empty(shape, dtype=dtype, device=self.dev)
        dist.broadcast(x, src, group=self.group)
        return x


# ------------------------------------------------------------------ state

@dataclass
class SlabState:
    """A rank's share of one scene: the replicated scene constants and bodies
    (``state``, whose particle set is this rank's) plus the global ids."""

    state: SimState
    gid: torch.Tensor          # (n_local,) global particle ids
    bounds: np.ndarray
    axis: int
    comm: Comm
    solve: str = "gather0"     # contact solve: "gather0" (rank 0) or "allreduce" (all ranks)

    @staticmethod
    def from_state(state: SimState, comm: Comm | None = None, axis: int = 0,
                   solve: str = "gather0") -> "SlabState":
        """Split a fully built (replicated) scene: every rank calls this with the
        same ``state`` and keeps its slab's particles.  ``solve`` picks the
        distributed contact solve (module docstring, item 2)."""
        if solve not in ("gather0", "allreduce"):
            raise ValueError(f"unknown slab solve mode {solve!r}")
        if state.cloth is not None and state.cloth.n_elements > 0:
            # mesh elements index particles that migration renumbers per rank
            raise ValueError("cloth is not supported under slab decomposition")
        comm = comm or Comm()
        p = state.particles
        x_axis = p.x[:, axis]
        bounds = slab_bounds(x_axis.detach().cpu().numpy(), comm.world, state.h)
        mine = slab_of(x_axis, bounds) == comm.rank
        idx = torch.nonzero(mine, as_tuple=False).reshape(-1)
        local = ParticleSet(*(getattr(p, k)[idx].clone() for k in PARTICLE_FIELDS),
                            validate=False)
        st = SimState(particles=local, materials=state.materials, bodies=state.bodies,
                      h=state.h, step=state.step, contact_params=state.contact_params,
                      solver_params=state.solver_params, mode=state.mode, workers=state.workers)
        st.time, st.step_index = state.time, state.step_index
        return SlabState(st, idx.clone(), bounds, axis, comm, solve)

    # -------------------------------------------------------------- migration
    def migrate(self) -> None:
        """Send particles that left the slab to their new owner (once per step)."""
        c, p = self.comm, self.state.particles
        dest = slab_of(p.x[:, self.axis], self.bounds)
        if c.world > 1:
            moving = dest != c.rank
            skip = int((dest - c.rank).abs().max()) > 1 if dest.numel() else False
            tot = c.sum(torch.tensor([int(moving.sum()), int(skip)], dtype=torch.int64))
            if int(tot[1]):  # every rank raises (no rank is left in a collective)
                raise RuntimeError("slab decomposition: a particle skipped a slab within one "
                                   "step (reduce dt or widen the slabs)")
            if int(tot[0]) == 0:
                return
            keep = torch.nonzero(~moving, as_tuple=False).reshape(-1)
            # grouped point-to-point: left movers to rank - 1, right movers to rank + 1
            lo_idx = torch.nonzero(dest < c.rank, as_tuple=False).reshape(-1)
            hi_idx = torch.nonzero(dest > c.rank, as_tuple=False).reshape(-1)
            from_l, from_r = c.neighbours(_pack_particles(p, self.gid, lo_idx, dest[lo_idx]),
                                          _pack_particles(p, self.gid, hi_idx, dest[hi_idx]))
            got = torch.cat([t for t in (from_l, from_r) if t is not None] or
                            [_pack_particles(p, self.gid, lo_idx[:0], dest[:0])])
            arrays = {k: getattr(p, k)[keep] for k in PARTICLE_FIELDS}
            gid = self.gid[keep]
            if got.shape[0]:
                g_gid, g_arr = _unpack_particles(got, p.x.device)
                for k in PARTICLE_FIELDS:
                    arrays[k] = torch.cat([arrays[k], g_arr[k]])
                gid = torch.cat([gid, g_gid])
            order = torch.argsort(gid)  # canonical local order: ascending global id
            self.state.particles = ParticleSet(*(arrays[k][order].contiguous()
                                                 for k in PARTICLE_FIELDS), validate=False)
            self.gid = gid[order].contiguous()

    def drift_check(self) -> None:
        """Particles must stay within the halo band of their slab during a step."""
        lo, hi = self.bounds[self.comm.rank], self.bounds[self.comm.rank + 1]
        x = self.state.particles.x[:, self.axis]
        slack = (HALO_BLOCKS - 1) * BLOCK_EDGE * self.state.h
        if not x.numel():
            return
        xmin, xmax = torch.stack([x.min(), x.max()]).tolist()   # one host sync
        if xmin < lo - slack or xmax >= hi + slack:
            raise RuntimeError("slab decomposition: particles drifted beyond the halo band "
                               "within one step (reduce dt or widen HALO_BLOCKS)")


def _pack_particles(p: ParticleSet, gid, idx, dest) -> torch.Tensor:
    cols = [dest.to(torch.float64)[:, None], gid[idx].to(torch.float64)[:, None],
            p.x[idx], p.v[idx], p.f[idx].reshape(-1, 9), p.c[idx].reshape(-1, 9),
            p.mass[idx][:, None], p.volume0[idx][:, None],
            p.material_id[idx].to(torch.float64)[:, None], p.plastic[idx][:, None]]
    return torch.cat(cols, dim=1)


def _unpack_particles(t: torch.Tensor, device):
    t = t.to(device)
    gid = t[:, 1].to(torch.int64)
    arr = dict(x=t[:, 2:5].contiguous(), v=t[:, 5:8].contiguous(),
               f=t[:, 8:17].reshape(-1, 3, 3).contiguous(),
               c=t[:, 17:26].reshape(-1, 3, 3).contiguous(), mass=t[:, 26].contiguous(),
               volume0=t[:, 27].contiguous(), material_id=t[:, 28].to(torch.int64),
               plastic=t[:, 29].contiguous())
    return gid, arr


# ------------------------------------------------------------------ substep

def _halo_reduce(ss: SlabState, grid: SparseGrid) -> torch.Tensor:
    """Sum the node channels of blocks shared with neighbours; returns the
    per-block "shared" mask."""
    return _halo_sum(ss, grid.block_keys, grid.mass, grid.mom_apic, grid.mom_force)


def _halo_sum(ss: SlabState, block_keys, mass, mom_apic, mom_force) -> torch.Tensor:
    """_halo_reduce on raw channel arrays ((nb*64,), (nb*64, 3), (nb*64, 3),
    updated in place): the operator pipeline's grid or the fused simulator's."""
    c = ss.comm
    nb = int(block_keys.shape[0])
    shared = torch.zeros(nb, dtype=torch.bool, device=block_keys.device)
    if c.world == 1 or nb == 0:
        return shared
    k = block_keys
    msk = (1 << 21) - 1
    bc = torch.stack([(k >> 42) - COORD_BIAS, ((k >> 21) & msk) - COORD_BIAS,
                      (k & msk) - COORD_BIAS], dim=1)
    ch = torch.cat([mass.view(-1, BLOCK_NODES, 1), mom_apic.reshape(-1, BLOCK_NODES, 3),
                    mom_force.reshape(-1, BLOCK_NODES, 3)], dim=2)  # (nb, 64, 7)

    def band_payload(side):
        idx = torch.nonzero(halo_band(bc[:, ss.axis], ss.bounds, c.rank, ss.state.h, side),
                            as_tuple=False).reshape(-1)
        # one row per block: packed key (as float64 bits) + 64 x 7 channels
        key = block_keys[idx].view(torch.float64)[:, None]
        return torch.cat([key, ch[idx].reshape(-1, BLOCK_NODES * 7)], dim=1)

    # each band goes to the one neighbour that can share it (point-to-point)
    from_l, from_r = c.neighbours(band_payload("left"), band_payload("right"))
    add = torch.zeros_like(ch)
    for got in (from_l, from_r):
        if got is None or got.numel() == 0:
            continue
        got = got.to(ch.device)
        pos = match_keys(block_keys, got[:, 0].contiguous().view(torch.int64))
        hit = pos >= 0
        if bool(hit.any()):
            add[pos[hit]] += got[hit, 1:].reshape(-1, BLOCK_NODES, 7)
            shared[pos[hit]] = True
    ch = ch + add
    mass.copy_(ch[:, :, 0].reshape(-1))
    mom_apic.copy_(ch[:, :, 1:4].reshape(-1, 3))
    mom_force.copy_(ch[:, :, 4:7].reshape(-1, 3))
    return shared


def _contact_problem(ss: SlabState, act, coords, owned, loc, w, m_a, vs_a, vk_a) -> dict:
    """The part of the distributed contact problem both solve modes share:
    this rank's contacts' stencils keyed by global node coordinates (``loc``:
    (nc, 27) active-node index or -1 for a dead slot, ``w`` zero there), the
    global contact-node set C (sorted keys, identical on every rank) and the
    all-reduced (S0, Q0, Q1) of the contact-free owned nodes.  ``m_a``,
    ``vs_a``, ``vk_a``: m, v*, v_k of the active nodes."""
    c = ss.comm
    keys_act = pack_coords(coords)
    n_act = int(act.shape[0])
    dead = loc < 0
    skeys = torch.where(dead, torch.full_like(loc, -1), keys_act[loc.clamp(min=0)])
    # the contact nodes: flags with a trash slot for dead slots (one nonzero
    # instead of a sort-based unique)
    flag = torch.zeros(n_act + 1, dtype=torch.bool, device=act.device)
    flag[torch.where(dead, torch.full_like(loc, n_act), loc).reshape(-1)] = True
    cn = torch.nonzero(flag[:n_act], as_tuple=False).reshape(-1)
    all_cn = c.allgather(keys_act[cn])
    C = torch.cat([k.to(act.device) for k in all_cn])
    # sorted; shared nodes appear once per rank that has contacts on them
    C = torch.unique(C) if c.world > 1 else torch.sort(C).values
    posC = match_keys(C, keys_act)                     # active node -> C, or -1
    fm = (owned & (posC < 0)).to(m_a.dtype)            # contact-free owned nodes
    ext = c.sum(free_sums(m_a * fm, vs_a, vk_a))
    nrec = torch.cat([m_a[cn][:, None], vs_a[cn], vk_a[cn]], dim=1)
    return dict(act=act, keys_act=keys_act, owned=owned, skeys=skeys, w=w, cn=cn,
                all_cn=all_cn, C=C, posC=posC, ext=ext, nrec=nrec)


def _local_contact_problem(ss: SlabState, grid, stencil, contacts, dt_s, block_shared):
    """_contact_problem from the operator pipeline's grid, stencil and contacts
    (also sets the contacts' lagged normal impulse, contact_model.py:50-55)."""
    st = ss.state
    dev = grid.mass.device
    act = torch.nonzero(grid.active, as_tuple=False).reshape(-1)
    coords = node_coords(grid.block_coords, act)
    owned = node_owned(coords[:, ss.axis], block_shared[act // BLOCK_NODES], ss.bounds,
                       ss.comm.rank, st.h)
    remap = torch.full((grid.n_nodes,), -1, dtype=torch.int64, device=dev)
    remap[act] = torch.arange(act.shape[0], device=dev)
    if contacts.n:
        vcs = contact_velocities(contacts, stencil, grid.v_k)
        contacts.gamma_lag = normal_impulse(vcs[:, 2], contacts.phi, st.contact_params, dt_s)
        loc = remap[stencil.nodes[contacts.particle]]          # (nc,27) active index or -1
        w = stencil.weights[contacts.particle].clone()
        w[loc < 0] = 0.0
    else:
        loc = torch.zeros((0, 27), dtype=torch.int64, device=dev)
        w = _lib.zeros((0, 27))
    return _contact_problem(ss, act, coords, owned, loc, w, grid.mass[act], grid.v_star[act],
                            grid.v_k[act])


def _active_v_next(vs_a, vk_a, lp, v_C, P):
    """v_next of the active nodes: contact nodes from the solution over C,
    every other one at v* + P (v_k - v*)."""
    va = vs_a + P * (vk_a - vs_a)
    pos = lp["posC"]
    if v_C.shape[0] == 0:
        return va
    return torch.where((pos >= 0)[:, None], v_C[pos.clamp(min=0)], va)


def _local_v_next(grid, lp, v_C, P):
    act = lp["act"]
    v_next = _lib.zeros((grid.n_nodes, 3))
    v_next[act] = _active_v_next(grid.v_star[act], grid.v_k[act], lp, v_C, P)
    return v_next


def _contact_records(cts, w) -> torch.Tensor:
    if not cts.n:
        return _lib.zeros((0, 9 + 3 + 3 + 27))
    return torch.cat([cts.frames.reshape(-1, 9), cts.bias, cts.phi[:, None],
                      cts.mu[:, None], cts.gamma_lag[:, None], w], dim=1)


def _solve_gather0(ss: SlabState, lp: dict, cts, dt_s):
    """solve="gather0": gather the contact problem to rank 0, solve it there
    with the fused solver (free nodes in closed form), broadcast the solution.
    ``cts``: this rank's contacts (n, frames, bias, phi, mu, gamma_lag).
    Returns (v over C, P, gamma (local contacts, contact frame), report)."""
    st, c = ss.state, ss.comm
    dev = lp["act"].device
    C, skeys = lp["C"], lp["skeys"]
    crec = _contact_records(cts, lp["w"])
    # the contact records go to rank 0 only; every rank needs the counts
    g_ck = c.gather0(skeys)
    g_cr = c.gather0(crec)
    g_nk = lp["all_cn"]
    g_nr = c.gather0(lp["nrec"])
    counts = [int(k) for k in c.allgather(torch.tensor([[skeys.shape[0]]], dtype=torch.int64))]
    if c.rank == 0:
        ck = torch.cat([k.to(dev) for k in g_ck])
        cr = torch.cat([r.to(dev) for r in g_cr])
        nk = torch.cat([k.to(dev) for k in g_nk])
        nr = torch.cat([r.to(dev) for r in g_nr])
        m, vs, v0 = _node_state(C, nk, nr)
        nodes = match_keys(C, ck.reshape(-1)).reshape(-1, 27).clamp(min=0)
        prob = ContactProblem(m=m, v_star=vs, v_init=v0, nodes=nodes, w=cr[:, 15:42].contiguous(),
                              frames=cr[:, 0:9].reshape(-1, 3, 3).contiguous(),
                              bias=cr[:, 9:12].contiguous(), phi=cr[:, 12].contiguous(),
                              mu=cr[:, 13].contiguous(), gamma_lag=cr[:, 14].contiguous(),
                              contact_params=st.contact_params, dt=dt_s)
        v_sol, gamma_all, report, P = quasi_newton_solve_ext(prob, st.solver_params,
                                                             lp["ext"].tolist())
        meta = torch.tensor([P, float(report.converged), float(report.iterations),
                             float(report.ls_evals), float(report.regularized)],
                            dtype=torch.float64, device=dev)
    else:
        v_sol = gamma_all = meta = None
    meta = c.bcast(meta)
    v_sol = c.bcast(v_sol).to(dev)
    gamma_all = c.bcast(gamma_all).to(dev)
    mt = meta.tolist()                                   # one read-back
    P = float(mt[0])
    start = sum(counts[: c.rank])
    gamma = gamma_all[start: start + cts.n]
    report = SolveReport(converged=mt[1] > 0.5, iterations=int(mt[2]),
                         n_contacts=int(sum(counts)), n_dofs=3 * int(C.shape[0]),
                         ls_evals=int(mt[3]), regularized=int(mt[4]))
    return v_sol, P, gamma, report


def _node_state(C, keys, recs):
    """(m, v*, v0) over the sorted contact-node set C from (key, record) rows;
    copies of a shared node are bitwise identical (P2G halo reduce)."""
    dev = C.device
    first = match_keys(C, keys)                                  # every record maps into C
    m = torch.empty(C.shape[0], dtype=torch.float64, device=dev)
    vs = torch.empty((C.shape[0], 3), dtype=torch.float64, device=dev)
    v0 = torch.empty((C.shape[0], 3), dtype=torch.float64, device=dev)
    m[first] = recs[:, 0]
    vs[first] = recs[:, 1:4]
    v0[first] = recs[:, 4:7]
    return m, vs, v0


def _ordered_scatter(nodes, vals, n_out: int) -> torch.Tensor:
    """(nc, 27, k) per-slot values summed onto n_out nodes in contact order
    (mpmrb_scatter_reduce_ordered)."""
    out = torch.empty((n_out, vals.shape[2]), dtype=torch.float64, device=vals.device)
    if n_out == 0:
        return out
    _lib.check(_lib.lib().mpmrb_scatter_reduce_ordered(
        _lib.ctx(), _lib.ptr(nodes.contiguous()), _lib.ptr(vals.contiguous()), nodes.shape[0],
        27, vals.shape[2], n_out, _lib.ptr(out)))
    return out


def _solve_allreduce(ss: SlabState, lp: dict, cts, dt_s):
    """solve="allreduce": the quasi-Newton solve of solver.py:328-382 spread
    over the ranks.  Contacts stay on the rank that detected them; the state
    of the global contact-node set C (m, v*, v) is replicated on every rank;
    the contact-free nodes enter in closed form through (S0, Q0, Q1) and
    P = prod(1 - alpha), as in the fused kernel (solver.cu free-node terms).
    Per iteration one vector all-reduce sums the ranks' J^T dl/dv_c and
    Hessian blocks over C (solver.py:127-167); every rank then forms the same
    gradient, residual (solver.py:188-194) and block-Cholesky direction
    (solver.py:224-256) redundantly.  Each exact line-search evaluation
    (solver.py:266-325) all-reduces two scalars (the contact part of phi',
    phi''), so every rank takes the same branch and alpha.
    Returns (v over C, P, gamma (local contacts, contact frame), report)."""
    from .contact_model import contact_grad_hess, contact_impulses
    from .collision import _contact_velocities_raw
    from .solver import line_search, solve_search_direction
    st, c = ss.state, ss.comm
    sp, cp = st.solver_params, st.contact_params
    dev = lp["act"].device
    C = lp["C"]
    nC, nc = int(C.shape[0]), cts.n
    g_nr = c.allgather(lp["nrec"])
    m, vs, v = _node_state(C, torch.cat([k.to(dev) for k in lp["all_cn"]]),
                           torch.cat([r.to(dev) for r in g_nr]))
    n_glob = int(c.sum(torch.tensor([nc], dtype=torch.int64)).item())
    nodes = match_keys(C, lp["skeys"].reshape(-1)).reshape(-1, 27).clamp(min=0)
    w = lp["w"]
    if nc:
        frames, bias = cts.frames, cts.bias
        phi, gl, mu = cts.phi, cts.gamma_lag, cts.mu
    S0, Q0, Q1 = (float(x) for x in lp["ext"].tolist())

    def contact_terms(v):
        """vc of the local contacts and their (J^T g_c | H_c) over C, (nC, 12)."""
        if not nc:
            return None, torch.zeros((nC, 12), dtype=torch.float64, device=dev)
        vc = _contact_velocities_raw(nodes, w, frames, bias, v)
        g_c, big_g = contact_grad_hess(vc, phi, gl, mu, cp, dt_s)
        gw = torch.einsum("ci,cij->cj", g_c, frames)                      # R^T g_c
        rgr = frames.transpose(1, 2) @ big_g @ frames
        vals = torch.cat([w[:, :, None] * gw[:, None, :],
                          (w * w)[:, :, None] * rgr.reshape(-1, 1, 9)], dim=2)
        return vc, _ordered_scatter(nodes, vals, nC)

    P, it, evals, converged = 1.0, 0, 0, False
    while True:
        vc, loc = contact_terms(v)
        tot = c.sum(loc)                                 # the per-iteration vector all-reduce
        jt, hc = tot[:, :3], tot[:, 3:]
        e = v - vs
        g = m[:, None] * e + jt
        p2s = P * P * S0
        s = torch.stack([(g * g / m[:, None]).sum(), (m[:, None] * v * v).sum(),
                         (jt * jt / m[:, None]).sum()]).tolist() if nC else [0.0, 0.0, 0.0]
        residual = float(np.sqrt(s[0] + p2s))
        threshold = sp.eps_a + sp.eps_r * max(np.sqrt(s[1] + Q0 + 2.0 * P * Q1 + p2s),
                                              np.sqrt(s[2]))
        if it >= sp.max_iters:
            converged = residual < threshold
            break
        if residual < (threshold if it > 0 else sp.eps_a):   # test-last, solver.py:339-345
            converged = True
            break
        h = torch.diag_embed(m[:, None].expand(-1, 3).contiguous()) + hc.reshape(-1, 3, 3)
        d = solve_search_direction(h, g) if nC else torch.zeros_like(v)
        md = m[:, None] * d
        a1 = float((e * md).sum()) - p2s                 # free nodes: d = -P e0
        a2 = float((d * md).sum()) + p2s
        dvc = (torch.einsum("cij,cj->ci", frames, torch.einsum("ck,ckd->cd", w, d[nodes]))
               if nc else None)

        def local_part(alpha: float) -> torch.Tensor:
            if not nc:
                return torch.zeros(2, dtype=torch.float64, device=dev)
            g_a, big_a = contact_grad_hess(vc + alpha * dvc, phi, gl, mu, cp, dt_s)
            return torch.stack([(g_a * dvc).sum(),
                                (dvc * torch.einsum("cij,cj->ci", big_a, dvc)).sum()])

        # the search always evaluates alpha = 0 and then alpha = 1
        # (solver.py:269-276): both travel in one all-reduce
        first = c.sum(torch.cat([local_part(0.0), local_part(1.0)])).tolist()
        known = {0.0: first[0:2], 1.0: first[2:4]}

        def deriv(alpha: float):
            tot2 = known.pop(alpha, None)
            if tot2 is None:
                tot2 = c.sum(local_part(alpha)).tolist()  # the line search's scalar all-reduce
            return a1 + a2 * alpha + tot2[0], a2 + tot2[1]

        ls = line_search(deriv, max_iters=sp.ls_max_iters, tol=sp.ls_tol)
        v = v + ls.alpha * d
        P *= 1.0 - ls.alpha
        it += 1
        evals += ls.evals
    if not bool(torch.isfinite(v).all()):
        raise FloatingPointError("contact solve produced non-finite velocities")
    gamma = contact_impulses(vc, phi, gl, mu, cp, dt_s) if nc else _lib.zeros((0, 3))
    report = SolveReport(converged=converged, iterations=it, n_contacts=n_glob, n_dofs=3 * nC,
                         ls_evals=evals)
    return v, P, gamma, report


_SOLVES = {"gather0": _solve_gather0, "allreduce": _solve_allreduce}


def slab_substep(ss: SlabState, dt_s: float, plan, epoch: int) -> dict:
    """coupling.py:115-150 on this rank's slab (the three exchanges above)."""
    st, c = ss.state, ss.comm
    p = st.particles
    grid = SparseGrid.allocate(p.x, st.h)
    stencil = build_stencil(p.x, grid)
    particle_to_grid(p, grid, stencil, st.materials, dt_s, plan, epoch, mode=st.mode,
                     workers=st.workers)
    shared = _halo_reduce(ss, grid)
    grid_update(grid, st.step.gravity, dt_s)
    contacts = detect_contacts(p, st.bodies, st.margin, st._bias_cache)
    n_glob = int(c.sum(torch.tensor([contacts.n], dtype=torch.int64)).item())
    if n_glob == 0:
        grid.v_next = grid.v_star
        act = torch.nonzero(grid.active, as_tuple=False).reshape(-1)
        coords = node_coords(grid.block_coords, act)
        owned = node_owned(coords[:, ss.axis], shared[act // BLOCK_NODES], ss.bounds, c.rank,
                           st.h)
        report = SolveReport(converged=True, n_contacts=0)
    else:
        lp = _local_contact_problem(ss, grid, stencil, contacts, dt_s, shared)
        v_C, P, gamma, report = _SOLVES[ss.solve](ss, lp, contacts, dt_s)
        grid.v_next, owned = _local_v_next(grid, lp, v_C, P), lp["owned"]
        if contacts.n:
            gamma_world = torch.einsum("ci,cij->cj", gamma, contacts.frames)
            bpos = torch.as_tensor(np.stack([np.asarray(b.position) for b in st.bodies]),
                                   dtype=torch.float64, device=gamma.device)
            st._accum.add_reactions(contacts.body, gamma_world, contacts.witness - bpos[contacts.body])
    clamped = grid_to_particle(p, grid, stencil, dt_s, st.materials)
    # per-rank statistics stay local; slab_advance_step reduces them once per step
    return dict(n_contacts=n_glob, report=report, clamped=clamped, n_active=owned.sum())


def slab_advance_step(ss: SlabState) -> StepSummary:
    """advance_step (coupling.py:168-219) of the whole scene; every rank returns
    the same summary."""
    st, c = ss.state, ss.comm
    ss.migrate()
    p = st.particles
    epoch = st.step_index
    plan = build_sort_plan(p.x, st.h, epoch)
    st._bias_cache = BiasCache()
    st._accum = ImpulseAccumulator(len(st.bodies))
    n = st.step.substeps
    dt_s = st.step.dt / n
    ncs, its, acts, clamped, conv = [], [], [], 0, True
    for _ in range(n):
        info = slab_substep(ss, dt_s, plan, epoch)
        ss.drift_check()
        ncs.append(info["n_contacts"])
        its.append(info["report"].iterations)
        acts.append(info["n_active"])
        conv &= info["report"].converged
        clamped += info["clamped"]
    dt = st.step.dt
    # one all-reduce of the step's per-rank statistics (active nodes per
    # substep, clamped gradients) instead of one per substep
    stats = torch.cat([torch.stack(acts).to(torch.float64).cpu(),
                       torch.tensor([float(clamped)], dtype=torch.float64)])
    stats = c.sum(stats)
    acts = [int(a) for a in stats[:-1].tolist()]
    clamped = int(stats[-1].item())
    acc = torch.as_tensor(np.concatenate([st._accum.linear, st._accum.angular], axis=1))
    acc = c.sum(acc).numpy()
    nb = len(st.bodies)
    st._accum.linear[:] = acc[:, :3]
    st._accum.angular[:] = acc[:, 3:]
    wrench = acc / dt
    new_time = st.time + dt
    _rigid_update(st, new_time)
    stale = torch.tensor([plan_staleness(plan, p.x, st.h) * p.n, float(p.n)], dtype=torch.float64)
    stale = c.sum(stale)
    n_tot = int(stale[1].item())
    summary = StepSummary(step_index=st.step_index, time=new_time, n_particles=n_tot,
                          n_active_nodes=float(np.mean(acts)),
                          n_contacts_mean=float(np.mean(ncs)), n_contacts_max=int(np.max(ncs)),
                          iterations_mean=float(np.mean(its)), iterations_max=int(np.max(its)),
                          all_converged=conv,
                          staleness=float(stale[0].item()) / max(n_tot, 1),
                          clamped_gradients=clamped, wrench=wrench[:nb])
    st.time = new_time
    st.step_index += 1
    return summary


# ------------------------------------------------------------------ fused mode

_TYPESTR = {torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4"}


class _DevArray:
    """A device pointer of the simulator as a zero-copy torch view."""

    def __init__(self, ptr, shape, dtype):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=_TYPESTR[dtype],
                                             data=(int(ptr or 0), False), version=2,
                                             strides=None)


def _dev(ptr, shape, dtype=torch.float64) -> torch.Tensor:
    if int(np.prod(shape)) == 0:
        return torch.empty(shape, dtype=dtype, device=_lib.device())
    return torch.as_tensor(_DevArray(ptr, shape, dtype), device=_lib.device())


def _views(sim) -> _lib.SimViews:
    v = _lib.SimViews()
    _lib.check(_lib.lib().mpmrb_sim_get_views(sim, C.byref(v)))
    return v


def _block_coords(keys: torch.Tensor) -> torch.Tensor:
    msk = (1 << 21) - 1
    return torch.stack([(keys >> 42) - COORD_BIAS, ((keys >> 21) & msk) - COORD_BIAS,
                        (keys & msk) - COORD_BIAS], dim=1)


def _fused_substep(ss: SlabState, sim, dt_s: float) -> dict:
    """One substep of the fused simulator on this rank's slab (coupling.py:
    115-150): part 0 (grid + P2G kernels), the P2G halo reduce on the
    simulator's own node channels, part 1 (grid update, active compaction,
    contacts), the distributed contact solve writing v_next and the impulses
    into the simulator's arrays, part 3 (reactions, G2P kernels)."""
    st, c = ss.state, ss.comm
    L = _lib.lib()
    _lib.check(L.mpmrb_sim_substep_part(sim, 0))
    shared = None
    if c.world > 1:   # the halo reduce needs the block count before part 1
        with torch.cuda.nvtx.range("slab halo reduce"):
            V = _views(sim)
            nb = int(V.n_blocks)
            N = nb * BLOCK_NODES
            shared = _halo_sum(ss, _dev(V.block_keys, (nb,), torch.int64), _dev(V.mass, (N,)),
                               _dev(V.mom_apic, (N, 3)), _dev(V.mom_force, (N, 3)))
    _lib.check(L.mpmrb_sim_substep_part(sim, 1))
    V = _views(sim)
    nb = int(V.n_blocks)
    N = nb * BLOCK_NODES
    keys = _dev(V.block_keys, (nb,), torch.int64)
    if shared is None:
        shared = torch.zeros(nb, dtype=torch.bool, device=keys.device)
    na, nc = int(V.n_active), int(V.n_contacts)
    act = _dev(V.act, (na,), torch.int32).to(torch.int64)
    coords = node_coords(_block_coords(keys), act)
    owned = node_owned(coords[:, ss.axis], shared[act // BLOCK_NODES], ss.bounds, c.rank, st.h)
    n_glob = int(c.sum(torch.tensor([nc], dtype=torch.int64)).item())
    if n_glob == 0:
        _lib.check(L.mpmrb_sim_substep_part(sim, 2))   # no contacts anywhere: v_next = v*
        report = SolveReport(converged=True, n_contacts=0)
    else:
        m_a, vs_a, vk_a = _dev(V.m_act, (na,)), _dev(V.v_star_act, (na, 3)), _dev(V.v_k_act,
                                                                                    (na, 3))
        cap = int(V.nc_cap)
        loc = _dev(V.cnodes, (27, cap), torch.int32)[:, :nc].t().to(torch.int64)
        w = _dev(V.cw, (27, cap))[:, :nc].t().contiguous()
        cts = SimpleNamespace(n=nc, frames=_dev(V.frames, (nc, 3, 3)), bias=_dev(V.bias, (nc, 3)),
                              phi=_dev(V.phi, (nc,)), mu=_dev(V.mu, (nc,)),
                              gamma_lag=_dev(V.gamma_lag, (nc,)))
        with torch.cuda.nvtx.range(f"slab contact solve ({ss.solve})"):
            lp = _contact_problem(ss, act, coords, owned, loc, w, m_a, vs_a, vk_a)
            v_C, P, gamma, report = _SOLVES[ss.solve](ss, lp, cts, dt_s)
        _dev(V.v_next, (N, 3))[act] = _active_v_next(vs_a, vk_a, lp, v_C, P)
        if nc:
            _dev(V.gamma, (nc, 3)).copy_(gamma)
        rep = _lib.SolveReportC()
        rep.converged, rep.iterations = int(report.converged), int(report.iterations)
        rep.ls_evals, rep.regularized = int(report.ls_evals), int(report.regularized)
        _lib.check(L.mpmrb_sim_set_solve_result(sim, C.byref(rep)))
    _lib.check(L.mpmrb_sim_substep_part(sim, 3))
    return dict(n_contacts=n_glob, report=report, n_active=owned.sum())


def slab_advance_step_fused(ss: SlabState) -> StepSummary:
    """slab_advance_step on the fused simulator's kernels (the substep's
    device pipeline of coupling.advance_step: stress-fused tiled P2G, hash
    grid, contact detection and preparation, G2P with the return map), with
    the slab exchanges between its parts (``_fused_substep``).  Particles
    migrate at the step start; the drift guard runs on the step's final
    positions.  Every rank returns the same summary."""
    st, c = ss.state, ss.comm
    L = _lib.lib()
    ss.migrate()
    p = st.particles
    sim = _coupling._ensure_sim(st)
    stream = _coupling._stream_of(st)
    stream.wait_stream(torch.cuda.current_stream())
    n = st.step.substeps
    dt = st.step.dt
    dt_s = dt / n
    nb = len(st.bodies)
    stats = _lib.StepStats()
    imp = (C.c_double * (6 * max(nb, 1)))()
    ncs, its, acts, conv = [], [], [], True
    with torch.cuda.stream(stream):
        _lib.bind_stream(st._ctx, stream)
        _coupling._configure_sim(st, sim, dt_s)
        rc = L.mpmrb_sim_begin_step(sim, st.step_index, n)
        if rc == _lib.E_DIVERGED:
            raise _coupling.SimulationDiverged(
                f"non-finite or out-of-range particle state after step {st.step_index}")
        _lib.check(rc)
        for _ in range(n):
            info = _fused_substep(ss, sim, dt_s)
            ncs.append(info["n_contacts"])
            its.append(info["report"].iterations)
            acts.append(info["n_active"])
            conv &= info["report"].converged
        rc = L.mpmrb_sim_end_step(sim, C.byref(stats), imp)
    if rc == _lib.E_DIVERGED:
        raise _coupling.SimulationDiverged(f"non-finite particle state after step {st.step_index}")
    _lib.check(rc)
    torch.cuda.current_stream().wait_stream(stream)
    ss.drift_check()
    acc = np.frombuffer(imp, dtype=np.float64)[: 6 * nb].reshape(nb, 6).copy()
    acc = c.sum(torch.as_tensor(acc)).numpy()
    st._accum.linear[:] = acc[:, 0:3]
    st._accum.angular[:] = acc[:, 3:6]
    loc = torch.cat([torch.stack(acts).to(torch.float64).cpu(),
                     torch.tensor([float(stats.clamped), _coupling._last_staleness(st) * p.n,
                                   float(p.n)], dtype=torch.float64)])
    tot = c.sum(loc)
    acts = [int(a) for a in tot[:n].tolist()]
    clamped, stale, n_tot = int(tot[n]), float(tot[n + 1]), int(tot[n + 2])
    new_time = st.time + dt
    wrench = np.concatenate([st._accum.linear / dt, st._accum.angular / dt], axis=1)
    _rigid_update(st, new_time)
    summary = StepSummary(step_index=st.step_index, time=new_time, n_particles=n_tot,
                          n_active_nodes=float(np.mean(acts)),
                          n_contacts_mean=float(np.mean(ncs)), n_contacts_max=int(np.max(ncs)),
                          iterations_mean=float(np.mean(its)), iterations_max=int(np.max(its)),
                          all_converged=conv, staleness=stale / max(n_tot, 1),
                          clamped_gradients=clamped, wrench=wrench)
    st.time = new_time
    st.step_index += 1
    return summary


def gather_particles(ss: SlabState) -> dict:
    """The whole scene's particle arrays in global-id order (on every rank)."""
    p = ss.state.particles
    pay = _pack_particles(p, ss.gid, torch.arange(p.n, device=p.x.device),
                          torch.zeros(p.n, dtype=torch.int64, device=p.x.device))
    allp = torch.cat([t.to(p.x.device) for t in ss.comm.allgather(pay)])
    gid, arr = _unpack_particles(allp, p.x.device)
    order = torch.argsort(gid)
    return {k: v[order] for k, v in arr.items()}
