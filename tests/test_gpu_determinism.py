"""Deterministic-mode contract of the reference's scatter (transfer.py:9-14,
135-187) on the GPU: ``mode="deterministic"`` sums every (node, channel) in
particle-id / slot order -- the np.bincount order -- so it is bitwise equal to
the reference's own deterministic scatter and independent of the sort plan;
``mode="fast"`` runs the same ordered fold; the float64-atomic
``scatter_naive`` agrees within the reference's own fast-vs-deterministic
bound (test_transfer.py:85-93).  Mirrors
test_deterministic_matches_serial_oracle / test_deterministic_is_plan_independent /
test_fast_matches_deterministic_within_tolerance."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import grid as og  # noqa: E402


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.fixture(scope="module")
def mp():
    import paper_2503_05046_b200 as m
    return m


@pytest.mark.parametrize("nch", [0, 1, 3, 4, 7, 9])
def test_deterministic_scatter_is_bitwise_the_reference_order(mp, nch):
    rng = np.random.default_rng(10 + nch)
    rows, k, n_out = 2000, 27, 900
    ids = rng.integers(0, n_out - 50, size=(rows, k))  # the last 50 nodes stay empty
    shape = (rows, k) if nch == 0 else (rows, k, nch)
    vals = rng.normal(size=shape) * np.exp(rng.normal(0, 4, size=shape))  # wide magnitudes
    vals.ravel()[::97] = -0.0
    plan = mp.build_sort_plan(rng.uniform(size=(rows, 3)), 0.05, 3)
    out = np_(mp.scatter_reduce(ids, vals, n_out, plan, 3))
    ref = og.scatter_in_order(ids, vals, n_out)  # np.bincount, row-major order
    np.testing.assert_array_equal(out, ref)
    assert np.array_equal(np.signbit(out), np.signbit(ref))
    # the reference's fused channel-offset bincount (transfer.py:140-145) is the same order
    if nch > 1:
        off = (np.arange(nch)[:, None] * n_out + ids.ravel()[None, :]).ravel()
        fused = np.bincount(off, weights=vals.reshape(-1, nch).T.ravel(),
                            minlength=nch * n_out).reshape(nch, n_out).T
        np.testing.assert_array_equal(out, fused)
    # fast mode runs the same ordered fold (the reference's fast-mode contract,
    # test_transfer.py:77-102, is met exactly); the float64-atomic scatter is
    # scatter_naive, within the reference's fast-vs-deterministic bound
    fast = np_(mp.scatter_reduce(ids, vals, n_out, plan, 3, mode="fast"))
    np.testing.assert_array_equal(fast, ref)
    from paper_2503_05046_b200.transfer import scatter_naive
    naive = np_(scatter_naive(ids, vals, n_out))
    assert np.abs(naive - ref).max() <= 1e-12 * np.abs(ref).max()


def test_deterministic_scatter_is_plan_independent_and_reproducible(mp):
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 0.3, size=(500, 3))
    ids = rng.integers(0, 300, size=(500, 27))
    vals = rng.normal(size=(500, 27, 7))
    p1 = mp.build_sort_plan(x, 0.05, 0)
    p2 = mp.build_sort_plan(x[::-1].copy(), 0.013, 0)  # a different plan
    a = np_(mp.scatter_reduce(ids, vals, 300, p1, 0))
    b = np_(mp.scatter_reduce(ids, vals, 300, p2, 0))
    c = np_(mp.scatter_reduce(ids, vals, 300, p1, 0))
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)


def test_deterministic_scatter_subset_and_edges(mp):
    rng = np.random.default_rng(5)
    plan = mp.build_sort_plan(rng.uniform(size=(40, 3)), 0.05, 0)
    pids = np.array([3, 7, 11, 30])
    ids = rng.integers(0, 20, size=(4, 27))
    vals = rng.normal(size=(4, 27, 3))
    out = np_(mp.scatter_reduce(ids, vals, 20, plan, 0, particle_ids=pids))
    np.testing.assert_array_equal(out, og.scatter_in_order(ids, vals, 20))
    empty = np_(mp.scatter_reduce(np.zeros((0, 27), np.int64), np.zeros((0, 27, 3)), 5, plan, 0,
                                  particle_ids=np.zeros(0, np.int64)))
    np.testing.assert_array_equal(empty, np.zeros((5, 3)))
    with pytest.raises(ValueError):  # node id out of range (transfer.py:161-170 ValueError)
        mp.scatter_reduce(np.full((4, 27), 25), vals, 20, plan, 0, particle_ids=pids)


@pytest.mark.parametrize("tag", ["a", "b"])
def test_deterministic_p2g_is_reproducible_and_matches_reference(mp, golden, tag):
    g = golden("p2g_g2p")
    mats = [mp.Material(E, nu, r) for E, nu, r in zip(g["mat_E"], g["mat_nu"], g["mat_rho"])]
    h, dt = float(g[f"{tag}_h"]), float(g[f"{tag}_dt"])
    p = mp.ParticleSet(g[f"{tag}_x"], g[f"{tag}_v"], g[f"{tag}_f"], g[f"{tag}_c"],
                       g[f"{tag}_mass"], g[f"{tag}_vol"], g[f"{tag}_mid"])
    plan = mp.build_sort_plan(p.x, h, 0)
    out = []
    for mode in ("deterministic", "deterministic", "fast"):
        grid = mp.SparseGrid.allocate(p.x, h)
        mp.particle_to_grid(p, grid, None, mats, dt, plan, 0, mode=mode)
        out.append([np_(grid.mass), np_(grid.mom_apic), np_(grid.mom_force)])
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)  # bitwise reproducible
    # vs the reference's deterministic grid: the scatter order is the
    # reference's; the per-entry values differ in the last bits (stress)
    assert np.abs(out[0][0] - g[f"{tag}_gmass"]).max() <= 1e-13 * g[f"{tag}_mass"].max()
    for got, key in zip(out[0][1:], ("mom_apic", "mom_force")):
        ref = g[f"{tag}_{key}"]
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), key
    for a, b in zip(out[0], out[2]):
        assert np.abs(a - b).max() <= 1e-12 * max(np.abs(a).max(), 1e-300)
