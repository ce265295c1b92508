"""Slab domain decomposition (paper_2503_05046_b200/slab.py), host logic on CPU:
slab bounds, ownership, halo bands, key packing, the particle migration
payload, the distributed solve's problem assembly, and the gloo communication
layer at world_size 2 and 3.  The device path
(2 ranks sharing cuda:0 vs the single-scene run) is tests/test_gpu_parity.py::
test_slab_decomposition_matches_single_scene."""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_05046_b200 import slab as S  # noqa: E402

H = 0.01


def test_slab_bounds_equal_count_and_block_aligned():
    rng = np.random.default_rng(0)
    x = rng.uniform(-0.8, 0.8, 20000)
    for world in (2, 4, 8):
        b = S.slab_bounds(x, world, H)
        assert b[0] == -np.inf and b[-1] == np.inf and len(b) == world + 1
        inner = b[1:-1]
        np.testing.assert_allclose(inner / (4 * H), np.round(inner / (4 * H)), atol=1e-9)
        assert np.all(np.diff(inner) >= S.MIN_SLAB_BLOCKS * 4 * H - 1e-12)
        counts = np.bincount(S.slab_of(torch.as_tensor(x), b).numpy(), minlength=world)
        assert counts.sum() == x.size
        assert counts.min() > 0.8 * x.size / world  # equal-count up to block snapping
    assert S.slab_bounds(x, 1, H).tolist() == [-np.inf, np.inf]
    with pytest.raises(ValueError):
        S.slab_bounds(rng.uniform(-0.05, 0.05, 1000), 4, H)


def test_slab_of_is_half_open():
    b = np.array([-np.inf, 0.0, 0.2, np.inf])
    x = torch.tensor([-1e-9, 0.0, 0.1999999, 0.2, 5.0], dtype=torch.float64)
    assert S.slab_of(x, b).tolist() == [0, 1, 1, 2, 2]


def test_node_keys_match_global_grid_packing():
    """Node coordinates from (block coords, local id) follow grid.py:121 and the
    keys pack like grid.py:26-31; distinct nodes get distinct keys."""
    bc = torch.tensor([[0, 0, 0], [-1, 2, 3], [5, -7, 1]], dtype=torch.int64)
    ids = torch.arange(3 * 64, dtype=torch.int64)
    c = S.node_coords(bc, ids)
    lid = ids % 64
    np.testing.assert_array_equal(c[:, 0] % 4, (lid >> 4).numpy())
    np.testing.assert_array_equal(c[:, 1] % 4, ((lid >> 2) & 3).numpy())
    np.testing.assert_array_equal(c[:, 2] % 4, (lid & 3).numpy())
    np.testing.assert_array_equal((c // 4).numpy(), bc[ids // 64].numpy())
    k = S.pack_coords(c)
    assert torch.unique(k).numel() == k.numel()
    bias = 1 << 20
    np.testing.assert_array_equal(((k >> 42) - bias).numpy(), c[:, 0].numpy())
    np.testing.assert_array_equal((((k >> 21) & ((1 << 21) - 1)) - bias).numpy(), c[:, 1].numpy())


def test_halo_band_covers_every_block_two_ranks_can_share():
    """A particle of rank r within the drift slack of the bound X touches blocks
    [(base)>>2, (base+2)>>2]; the band must contain every block that particles
    of BOTH sides can touch."""
    b = np.array([-np.inf, 0.4, np.inf])
    slack = (S.HALO_BLOCKS - 1) * 4 * H
    xs_left = np.linspace(0.4 - 1.0, 0.4 + slack - 1e-9, 4001)
    xs_right = np.linspace(0.4 - slack, 0.4 + 1.0, 4001)

    def blocks(xs):
        base = np.floor(xs / H - 0.5).astype(np.int64)
        return set((base >> 2).tolist()) | set(((base + 2) >> 2).tolist())

    both = blocks(xs_left) & blocks(xs_right)
    cand = torch.tensor(sorted(both), dtype=torch.int64)
    for rank in (0, 1):
        assert bool(S.halo_band(cand, b, rank, H).all()), rank


def test_match_keys():
    mine = torch.tensor([3, 7, 9, 20], dtype=torch.int64)
    theirs = torch.tensor([7, 8, 20, 1, 3], dtype=torch.int64)
    assert S.match_keys(mine, theirs).tolist() == [1, -1, 3, -1, 0]
    assert S.match_keys(mine[:0], theirs).tolist() == [-1] * 5


def test_node_ownership_counts_each_node_once():
    """Two ranks holding copies of shared blocks: ownership by coordinate in
    shared blocks, by possession otherwise -> every node owned exactly once."""
    b = np.array([-np.inf, 0.4, np.inf])
    # node x coordinates (in cells) held by each rank; 36..43 shared
    left = torch.arange(20, 44)
    right = torch.arange(36, 60)
    shared_l = (left >= 36)
    shared_r = (right < 44)
    own_l = S.node_owned(left, shared_l, b, 0, H)
    own_r = S.node_owned(right, shared_r, b, 1, H)
    owners = {}
    for xs, own in ((left, own_l), (right, own_r)):
        for x, o in zip(xs.tolist(), own.tolist()):
            owners[x] = owners.get(x, 0) + int(o)
    assert set(owners) == set(range(20, 60))
    assert all(v == 1 for v in owners.values())


def test_free_sums_closed_form():
    rng = np.random.default_rng(1)
    m = torch.as_tensor(rng.uniform(0.1, 1, 50))
    vs = torch.as_tensor(rng.normal(size=(50, 3)))
    v0 = torch.as_tensor(rng.normal(size=(50, 3)))
    S0, Q0, Q1 = S.free_sums(m, vs, v0).tolist()
    e = (v0 - vs).numpy()
    mm = m.numpy()[:, None]
    assert S0 == pytest.approx(float((mm * e * e).sum()))
    assert Q0 == pytest.approx(float((mm * vs.numpy() ** 2).sum()))
    assert Q1 == pytest.approx(float((mm * vs.numpy() * e).sum()))
    # the free nodes' |M^1/2 v|^2 at v = v* + P e equals Q0 + 2 P Q1 + P^2 S0
    P = 0.37
    v = vs.numpy() + P * e
    assert float((mm * v * v).sum()) == pytest.approx(Q0 + 2 * P * Q1 + P * P * S0)


class _P:  # particle-set stand-in with CPU tensors
    def __init__(self, n, seed):
        g = torch.Generator().manual_seed(seed)
        self.x = torch.rand(n, 3, generator=g, dtype=torch.float64)
        self.v = torch.rand(n, 3, generator=g, dtype=torch.float64)
        self.f = torch.rand(n, 3, 3, generator=g, dtype=torch.float64)
        self.c = torch.rand(n, 3, 3, generator=g, dtype=torch.float64)
        self.mass = torch.rand(n, generator=g, dtype=torch.float64)
        self.volume0 = torch.rand(n, generator=g, dtype=torch.float64)
        self.material_id = torch.randint(0, 3, (n,), generator=g)
        self.plastic = torch.rand(n, generator=g, dtype=torch.float64)


def test_migration_payload_roundtrip():
    p = _P(40, 3)
    gid = torch.arange(100, 140)
    idx = torch.tensor([3, 17, 39])
    dest = torch.tensor([1, 0, 2])
    pay = S._pack_particles(p, gid, idx, dest)
    assert pay[:, 0].tolist() == [1.0, 0.0, 2.0]
    g, arr = S._unpack_particles(pay, torch.device("cpu"))
    assert g.tolist() == [103, 117, 139]
    for k in S.PARTICLE_FIELDS:
        assert torch.equal(arr[k], getattr(p, k)[idx]), k


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _comm_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = S.Comm()
    assert (c.rank, c.world) == (rank, world)
    mine = torch.arange(rank * 3 + 1, dtype=torch.float64).reshape(-1, 1) + 10 * rank
    got = c.allgather(mine)
    empty = c.allgather(torch.zeros((0, 4), dtype=torch.int64) if rank == 0
                        else torch.ones((2, 4), dtype=torch.int64))
    s = c.sum(torch.tensor([rank + 1.0, 2.0 * rank], dtype=torch.float64))
    b = c.bcast(torch.arange(6, dtype=torch.float64).reshape(2, 3) if rank == 0 else None)
    torch.save(dict(got=got, empty=empty, s=s, b=b), os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_comm_world2_gloo(tmp_path):
    world = 2
    mp.spawn(_comm_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for rank in range(world):
        r = torch.load(tmp_path / f"r{rank}.pt")
        assert [t.flatten().tolist() for t in r["got"]] == [[0.0], [10.0, 11.0, 12.0, 13.0]]
        assert r["empty"][0].shape == (0, 4) and r["empty"][1].shape == (2, 4)
        assert r["s"].tolist() == [3.0, 2.0]
        assert r["b"].tolist() == [[0.0, 1.0, 2.0], [3.0, 4.0, 5.0]]


def _neighbour_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = S.Comm()
    # rank r sends r+1 rows of value 100 r + 1 to the left and 2 (r+1) rows of
    # 100 r + 2 to the right; rank 1 sends nothing to the left (empty payload)
    to_l = torch.full((0 if rank == 1 else rank + 1, 2), 100.0 * rank + 1)
    to_r = torch.full((2 * (rank + 1), 2), 100.0 * rank + 2)
    fl, fr = c.neighbours(to_l, to_r)
    g = c.gather0(torch.full((rank, 3), float(rank), dtype=torch.float64))
    torch.save(dict(fl=fl, fr=fr, g=g), os.path.join(out, f"n{rank}.pt"))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_exchange_and_gather0_gloo(tmp_path, world):
    """Comm.neighbours (the P2G halo and migration exchange) reaches exactly
    the adjacent ranks, with variable and empty payloads; gather0 collects
    every rank's rows on rank 0 only."""
    mp.spawn(_neighbour_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
             join=True)
    for rank in range(world):
        r = torch.load(tmp_path / f"n{rank}.pt")
        if rank == 0:
            assert r["fl"] is None
            assert [t.shape[0] for t in r["g"]] == list(range(world))
            assert all(bool((t == q).all()) for q, t in enumerate(r["g"]))
        else:
            left = rank - 1  # its right payload: 2 (left + 1) rows of 100 left + 2
            assert r["fl"].shape == (2 * (left + 1), 2) and bool((r["fl"] == 100 * left + 2).all())
            assert r["g"] is None
        if rank == world - 1:
            assert r["fr"] is None
        else:
            right = rank + 1  # its left payload (empty from rank 1)
            n = 0 if right == 1 else right + 1
            assert r["fr"].shape == (n, 2) and bool((r["fr"] == 100 * right + 1).all())


def test_contact_problem_assembly_host_logic():
    """_contact_problem (the distributed solve's shared prologue) at one rank
    on CPU tensors: the contact-node set, the stencil keys, the free-node sums
    over owned contact-free nodes and the node records agree with a direct
    restatement; _active_v_next puts the solution on contact nodes and
    v* + P (v_k - v*) everywhere else."""
    from types import SimpleNamespace
    rng = np.random.default_rng(3)
    na, nc = 60, 7
    coords = torch.as_tensor(rng.integers(-50, 50, size=(na, 3)))
    act = torch.arange(na)
    owned = torch.as_tensor(rng.random(na) < 0.8)
    loc = torch.as_tensor(rng.integers(0, na, size=(nc, 27)))
    loc[torch.as_tensor(rng.random((nc, 27)) < 0.2)] = -1
    w = torch.as_tensor(rng.random((nc, 27)))
    w[loc < 0] = 0.0
    m = torch.as_tensor(rng.uniform(0.1, 1.0, na))
    vs = torch.as_tensor(rng.normal(size=(na, 3)))
    vk = torch.as_tensor(rng.normal(size=(na, 3)))
    ss = SimpleNamespace(comm=S.Comm())
    lp = S._contact_problem(ss, act, coords, owned, loc, w, m, vs, vk)
    keys = S.pack_coords(coords)
    cn_ref = np.unique(loc[loc >= 0].numpy())
    assert lp["cn"].tolist() == cn_ref.tolist()
    assert lp["C"].tolist() == sorted(keys[cn_ref].tolist())
    sk = lp["skeys"].numpy()
    assert (sk[loc.numpy() < 0] == -1).all()
    assert (sk[loc.numpy() >= 0] == keys.numpy()[loc.numpy()[loc.numpy() >= 0]]).all()
    free = owned.numpy() & ~np.isin(np.arange(na), cn_ref)
    ref = S.free_sums(m[free], vs[free], vk[free])
    assert torch.allclose(lp["ext"], ref, rtol=1e-13, atol=1e-13)
    assert torch.equal(lp["nrec"][:, 0], m[cn_ref])
    # v_next: solution on C, closed form elsewhere
    v_C = torch.as_tensor(rng.normal(size=(lp["C"].shape[0], 3)))
    P = 0.3
    va = S._active_v_next(vs, vk, lp, v_C, P)
    pos = {k: i for i, k in enumerate(lp["C"].tolist())}
    for i in range(na):
        k = int(keys[i])
        exp = v_C[pos[k]] if k in pos else vs[i] + P * (vk[i] - vs[i])
        assert torch.equal(va[i], exp)


def test_slab_rejects_unknown_solve_and_cloth():
    """from_state validates before touching any device state."""
    from types import SimpleNamespace
    st = SimpleNamespace(cloth=None)
    with pytest.raises(ValueError):
        S.SlabState.from_state(st, solve="bogus")
    st = SimpleNamespace(cloth=SimpleNamespace(n_elements=3))
    with pytest.raises(ValueError):
        S.SlabState.from_state(st)
