"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and against the reference tests' known answers.
CPU only."""

import numpy as np
import pytest

from oracle import contact as ocm
from oracle import grid as og
from oracle import mpm as om
from oracle import sdf as osdf
from oracle import solver as osv
from oracle import step as ostep
from scenes import load_scene_json, oracle_state

from types import SimpleNamespace


@pytest.mark.parametrize("tag", ["uniform", "negative", "dense"])
def test_binning_matches_reference(golden, tag):
    g = golden("binning")
    x, h = g[f"{tag}_x"], float(g[f"{tag}_h"])
    assert np.array_equal(og.base_cells(x, h), g[f"{tag}_cells"])
    assert np.array_equal(og.morton10(og.base_cells(x, h)), g[f"{tag}_keys"])
    plan = og.sort_plan(x, h, 5)
    for k in ("perm", "inv_perm", "bin_keys", "bin_starts", "bin_of"):
        assert np.array_equal(getattr(plan, k), g[f"{tag}_{k}"]), k
    keys = og.allocate_blocks(x, h)
    assert np.array_equal(keys, g[f"{tag}_block_keys"])
    assert np.array_equal(og.unpack_blocks(keys), g[f"{tag}_block_coords"])
    st = og.make_stencil(x, keys, h)
    assert np.array_equal(st.nodes, g[f"{tag}_nodes"])
    assert np.array_equal(st.weights, g[f"{tag}_weights"])
    assert np.array_equal(st.dpos, g[f"{tag}_dpos"])
    assert og.staleness(plan, g[f"{tag}_moved"], h) == float(g[f"{tag}_staleness"])


def test_morton_known_answers():
    # reference test_transfer.py:22-31 locality KAT
    cells = og.base_cells(np.array([[0.05, 0.05, 0.05], [0.15, 0.05, 0.05], [3.05, 0.05, 0.05]]),
                          0.1)
    k = og.morton10(cells)
    assert k.dtype == np.uint16
    assert abs(int(k[0]) - int(k[1])) < abs(int(k[0]) - int(k[2]))


def test_lookup_outside_allocation_raises():
    keys = og.allocate_blocks(np.array([[0.5, 0.5, 0.5]]), 0.1)
    with pytest.raises(og.OracleAllocationError):
        og.lookup_nodes(keys, np.array([[900, 900, 900]]))


def _mats(g):
    return [SimpleNamespace(youngs_modulus=E, poisson_ratio=nu, density=r)
            for E, nu, r in zip(g["mat_E"], g["mat_nu"], g["mat_rho"])]


@pytest.mark.parametrize("tag", ["a", "b"])
def test_p2g_grid_g2p_match_reference(golden, tag):
    g = golden("p2g_g2p")
    mats = _mats(g)
    x, h, dt = g[f"{tag}_x"], float(g[f"{tag}_h"]), float(g[f"{tag}_dt"])
    tau = om.stresses(g[f"{tag}_f"], g[f"{tag}_mid"], mats)
    np.testing.assert_allclose(tau, g[f"{tag}_tau"], rtol=1e-12, atol=1e-9)
    keys = og.allocate_blocks(x, h)
    assert np.array_equal(keys, g[f"{tag}_block_keys"])
    st = og.make_stencil(x, keys, h)
    n_nodes = keys.shape[0] * 64
    m, ma, mf = om.p2g(x, g[f"{tag}_v"], g[f"{tag}_f"], g[f"{tag}_c"], g[f"{tag}_mass"],
                       g[f"{tag}_vol"], g[f"{tag}_mid"], mats, st, dt, n_nodes)
    assert np.abs(m - g[f"{tag}_gmass"]).max() <= 1e-13 * g[f"{tag}_mass"].max()
    assert np.abs(ma - g[f"{tag}_mom_apic"]).max() <= 1e-12 * np.abs(g[f"{tag}_mom_apic"]).max()
    assert np.abs(mf - g[f"{tag}_mom_force"]).max() <= 1e-12 * np.abs(g[f"{tag}_mom_force"]).max()
    act, vk, vs = om.grid_update(m, ma, mf, (0.0, 0.0, -9.81), dt)
    assert np.array_equal(act, g[f"{tag}_active"])
    np.testing.assert_allclose(vk, g[f"{tag}_v_k"], rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(vs, g[f"{tag}_v_star"], rtol=1e-11, atol=1e-12)
    x1, v1, c1, f1, k = om.g2p(x, g[f"{tag}_f"], st, g[f"{tag}_v_next"], dt)
    np.testing.assert_allclose(x1, g[f"{tag}_x1"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(v1, g[f"{tag}_v1"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(c1, g[f"{tag}_c1"], rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(f1, g[f"{tag}_f1"], rtol=1e-12, atol=1e-13)
    assert k == int(g[f"{tag}_nclamp"])


def test_clamp_matches_reference(golden):
    g = golden("p2g_g2p")
    out, k = om.clamp_inverted(g["clamp_in"])
    assert k == int(g["clamp_n"])
    np.testing.assert_allclose(out, g["clamp_out"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("name", ["halfspace", "sphere", "box", "capsule"])
def test_sdf_matches_reference(golden, name):
    g = golden("sdf_contacts")
    shapes = {"halfspace": ("halfspace", (0.0, 0.6, 0.8), 0.05), "sphere": ("sphere", 0.3),
              "box": ("box", (0.15, 0.1, 0.25)), "capsule": ("capsule", 0.05, 0.2)}
    phi, nrm, wit = osdf.query(shapes[name], g[f"{name}_pts"])
    np.testing.assert_allclose(phi, g[f"{name}_phi"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(nrm, g[f"{name}_normal"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(wit, g[f"{name}_witness"], rtol=0, atol=1e-15)


def test_frames_match_reference(golden):
    g = golden("sdf_contacts")
    np.testing.assert_allclose(osdf.frames(g["frames_normals"]), g["frames"], rtol=0, atol=1e-15)


def test_detect_with_bias_cache_matches_reference(golden):
    from scenes import oracle_bodies
    g = golden("sdf_contacts")
    scene = load_scene_json(g["scene_json"])
    bodies = oracle_bodies(scene)
    cache = ocm.FirstSightBias()
    c1 = ocm.detect(g["det_x"], bodies, 0.01, cache)
    bodies[1].v = g["det_body1_v2"]
    c2 = ocm.detect(g["det_x2"], bodies, 0.01, cache)
    for tag, c in (("c1", c1), ("c2", c2)):
        for k in ("particle", "body", "geom"):
            assert np.array_equal(getattr(c, k), g[f"{tag}_{k}"]), (tag, k)
        for k in ("phi", "normal", "witness", "frames", "bias", "mu"):
            np.testing.assert_allclose(getattr(c, k), g[f"{tag}_{k}"], rtol=0, atol=1e-14,
                                       err_msg=f"{tag} {k}")


def _problem(g, s):
    pre = f"s{s}_"
    k, tau_d, eps_v, dt = g[pre + "cparams"]
    return osv.Problem(g[pre + "m"], g[pre + "v_star"], g[pre + "v_init"], g[pre + "nodes"],
                       g[pre + "w"], g[pre + "frames"], g[pre + "bias"], g[pre + "phi"],
                       g[pre + "mu"], g[pre + "gamma_lag"], k, tau_d, eps_v, dt)


def _mnorm(v, m):
    return float(np.sqrt(np.sum(m[:, None] * v * v)))


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_solver_matches_reference(golden, seed):
    g = golden("solver")
    prob = _problem(g, seed)
    for tag, par in (("tight", osv.Params(eps_r=1e-10, max_iters=3000)),
                     ("loose", osv.Params(eps_r=5e-2))):
        v, gam, rep = osv.minimise(prob, par)
        pre = f"s{seed}_{tag}_"
        assert rep.converged == bool(g[pre + "conv"])
        ref_it = int(g[pre + "iters"])
        assert abs(rep.iterations - ref_it) <= max(1, ref_it // 50)
        assert _mnorm(v - g[pre + "v"], prob.m) <= 1e-9 * max(1.0, _mnorm(g[pre + "v"], prob.m))
        np.testing.assert_allclose(rep.residual[0], g[pre + "residual"][0], rtol=1e-12)
        np.testing.assert_allclose(rep.objective[0], g[pre + "objective"][0], rtol=1e-12)


@pytest.mark.parametrize("seed", [0, 1])
def test_dense_newton_matches_reference(golden, seed):
    g = golden("solver")
    prob = _problem(g, seed)
    v, _, rep = osv.minimise(prob, osv.Params(eps_r=1e-10, max_iters=3000), dense=True)
    assert rep.converged
    ref = g[f"s{seed}_dense_v"]
    assert _mnorm(v - ref, prob.m) <= 1e-8 * _mnorm(ref, prob.m)


def test_line_search_known_answers():
    # reference test_solver.py:59-82
    a, ev, _ = osv.exact_line_search(lambda a: (2 * (a - 3.0), 2.0))
    assert a == pytest.approx(3.0, rel=1e-8) and ev <= 3
    a, _, _ = osv.exact_line_search(
        lambda a: (a - 1.0 if a < 1.0 else 5.0 * (a - 1.0), 1.0 if a < 1.0 else 5.0))
    assert a == pytest.approx(1.0, abs=1e-7)
    a, _, _ = osv.exact_line_search(lambda a: (0.5 * (a - 40.0), 0.5))
    assert a == pytest.approx(40.0, rel=1e-8)
    with pytest.raises(osv.LineSearchError):
        osv.exact_line_search(lambda a: (1.0, 2.0))


@pytest.mark.parametrize("tag", ["rest", "press"])
def test_steps_match_reference(golden, tag):
    g = golden("steps")
    scene = load_scene_json(g[f"{tag}_scene_json"])
    s = oracle_state(scene, g[f"{tag}_x0"], g[f"{tag}_v0"], g[f"{tag}_f0"], g[f"{tag}_c0"],
                     g[f"{tag}_mass"], g[f"{tag}_vol"], g[f"{tag}_mid"])
    nsteps = g[f"{tag}_wrench"].shape[0]
    for i in range(nsteps):
        out = ostep.step(s)
        np.testing.assert_allclose(out["wrench"], g[f"{tag}_wrench"][i], rtol=1e-7, atol=1e-9)
        assert out["n_contacts_mean"] == g[f"{tag}_contacts_mean"][i]
        assert out["staleness"] == g[f"{tag}_staleness"][i]
        np.testing.assert_allclose(s.x, g[f"{tag}_xs"][i], rtol=0, atol=1e-12)
    np.testing.assert_allclose(s.v, g[f"{tag}_v1"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(s.f, g[f"{tag}_f1"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(np.array([b.position for b in s.bodies]),
                               g[f"{tag}_bodies_pos"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array([b.v for b in s.bodies]), g[f"{tag}_bodies_v"],
                               rtol=0, atol=1e-9)
