"""The warp tiles of k_p2g / k_g2p (mpm.cu warp_segment) must be invisible in
the results, whatever the particle order: a warp whose particles do not fit one
node tile is cut into segments of consecutive lanes, down to one particle per
segment.  Orders tried: the sort plan's Morton order, random, reversed, and an
adversarial interleaving of three far-apart clusters (every lane of a warp in
a different place, so every warp is 32 segments).

* P2G ("fast", warp tiles + float64 atomics) agrees with the reference-order
  deterministic P2G within the reference's fast-vs-deterministic bound
  (test_transfer.py:85-93, 1e-12 of the channel's max) for every order, and
  conserves mass and momentum (test_mpm.py:115-124).
* G2P is a per-particle gather in a fixed slot order, so its outputs are
  bitwise identical for every order once permuted back."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.fixture(scope="module")
def mp():
    import paper_2503_05046_b200 as m
    return m


H = 0.02


def _scene(seed=3):
    rng = np.random.default_rng(seed)
    centers = np.array([[0.1, 0.1, 0.1], [0.9, 0.2, 0.5], [0.3, 0.8, 0.9]])
    x = np.concatenate([c + rng.uniform(-0.06, 0.06, size=(1400, 3)) for c in centers])
    n = x.shape[0]
    v = rng.normal(size=(n, 3))
    f = np.eye(3)[None] + 0.05 * rng.normal(size=(n, 3, 3))
    c = 0.2 * rng.normal(size=(n, 3, 3))
    vol = np.full(n, 2e-6)
    return x, v, f, c, 1200.0 * vol, vol


def _orders(mp, x):
    n = x.shape[0]
    rng = np.random.default_rng(11)
    plan = mp.build_sort_plan(x, H, 0)
    perm = np_(plan.perm).astype(np.int64)  # Morton-binned order (transfer.py:85-102)
    inter = np.stack([np.arange(0, 1400), np.arange(1400, 2800), np.arange(2800, 4200)], 1).ravel()
    return {"sorted": perm, "random": rng.permutation(n), "reversed": np.arange(n)[::-1].copy(),
            "interleaved": inter}


def _particles(mp, arrs, order):
    x, v, f, c, m, vol = arrs
    return mp.ParticleSet(x[order], v[order], f[order], c[order], m[order], vol[order])


def test_p2g_tiles_any_order_match_deterministic(mp):
    arrs = _scene()
    mats = [mp.Material(2e5, 0.3, 1200.0)]
    dt = 1e-4
    ref = None
    for name, order in _orders(mp, arrs[0]).items():
        p = _particles(mp, arrs, order)
        plan = mp.build_sort_plan(p.x, H, 0)
        out = {}
        for mode in ("deterministic", "fast"):
            grid = mp.SparseGrid.allocate(p.x, H)
            mp.particle_to_grid(p, grid, None, mats, dt, plan, 0, mode=mode)
            out[mode] = [np_(grid.mass), np_(grid.mom_apic), np_(grid.mom_force)]
        for a, b in zip(out["fast"], out["deterministic"]):
            assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max(), name
        if ref is None:
            ref = out["deterministic"]
        else:  # the node layout does not depend on the particle order
            for a, b in zip(out["fast"], ref):
                assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max(), name
        gm, ga = out["fast"][0], out["fast"][1]
        assert gm.sum() == pytest.approx(float(arrs[4].sum()), rel=1e-13)
        ptot = (arrs[4][:, None] * arrs[1]).sum(0)
        np.testing.assert_allclose(ga.sum(0), ptot, rtol=1e-12, atol=1e-15)


def test_g2p_tiles_any_order_bitwise(mp):
    arrs = _scene(5)
    x = arrs[0]
    dt = 1e-4
    res = {}
    for name, order in _orders(mp, x).items():
        p = _particles(mp, arrs, order)
        grid = mp.SparseGrid.allocate(p.x, H)
        pos = np_(grid.node_positions(torch.arange(grid.n_nodes, device="cuda")))
        vn = 0.3 + np.sin(7.0 * pos) * np.array([1.0, -0.5, 0.25])  # smooth, order-free field
        grid.v_next = mp._lib.as_dev(vn)
        mp.grid_to_particle(p, grid, None, dt)
        inv = np.empty_like(order)
        inv[order] = np.arange(order.size)
        res[name] = [np_(a)[inv] for a in (p.x, p.v, p.c, p.f)]
    base = res["sorted"]
    for name, got in res.items():
        for a, b in zip(got, base):
            assert np.array_equal(a, b), name
