"""GPU parity at the BASELINE configurations (the sizes the bench measures).

* configs[0] (C1): the 8,000-particle elastic cube, all 100 rigid steps,
  against the trajectory recorded by running the UNMODIFIED reference
  (tests/golden/make_golden.py gen_c1; coupling.py:168-219).
* configs[1] (C2, 256k sand) and the 1M north-star sand scene: one substep
  from a pusher-loaded mid-window state, GPU vs the CPU oracle from the same
  state: grid momentum, contact set, contact impulses, the solver's residual
  test and the particle update.

Tolerances are stated per test and explained where they are set.  Each test
also writes its measured deviations to ``gpurun_out/parity_configs.jsonl``
(the numbers DESIGN.md §5 quotes).
"""

import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from scenes import load_scene_json, oracle_state  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _record(name, **kw):
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    with open(out / "parity_configs.jsonl", "a") as fh:
        fh.write(json.dumps(dict(test=name, **kw)) + "\n")


@pytest.fixture(scope="module")
def mp():
    import paper_2503_05046_b200 as m
    return m


def test_c1_cube_100_steps_match_reference(mp, golden):
    """configs[0] end to end: 100 fused rigid steps vs the reference run.

    The cube lands at step ~45; from then on the solves take 13-46 iterations
    and stop anywhere below eps_r = 5e-2 of the residual scale, so a
    trajectory becomes sensitive to the float summation order.  The
    fixture holds the reference run twice: in its default deterministic mode
    and in its own "fast" mode (a different summation order the reference
    tolerates, test_transfer.py:85-93).  Bars:

    * steps 1-44 (before the first multi-iteration solve, where the
      reference's two modes agree to 1e-6): contact counts exact, wrench per
      step within 1e-6 of its largest component, x at steps 10/25 to 1e-12 m;
    * steps 45-100: x at steps 50/75/100 within the larger of 10x the
      reference's own fast-vs-deterministic deviation at that step and 0.02 h
      (chaotic sensitivity to summation order, see below); the impulse integrated
      over the 100 steps within 5x the reference's fast-vs-deterministic
      difference (of its largest component); total solver iterations within
      10%."""
    from paper_2503_05046_b200 import scenes
    g = golden("c1_cube")
    scene = load_scene_json(g["scene_json"])
    state = scenes.build_state(scene)
    np.testing.assert_array_equal(np_(state.particles.x), g["x0"])  # same seeding
    nsteps = g["wrench"].shape[0]
    pre = 44
    d_nc, werr, xerr, wr, its = [], [], {}, [], []
    for i in range(nsteps):
        s = mp.advance_step(state)
        wr.append(s.wrench)
        its.append(s.iterations_mean)
        d_nc.append(abs(s.n_contacts_mean - g["contacts_mean"][i]))
        ws = np.abs(g["wrench"][i]).max()
        werr.append(float(np.abs(s.wrench - g["wrench"][i]).max() / max(ws, 1e-30)))
        k = i + 1
        if f"x_{k}" in g:
            xerr[k] = float(np.abs(np_(state.particles.x) - g[f"x_{k}"]).max())
    fast_x = {k: float(np.abs(g[f"fast_x_{k}"] - g[f"x_{k}"]).max()) for k in xerr}
    W, Wf, Wg = g["wrench"].sum(0), g["fast_wrench"].sum(0), np.sum(wr, axis=0)
    imp_fast = float(np.abs(Wf - W).max() / np.abs(W).max())
    imp_gpu = float(np.abs(Wg - W).max() / np.abs(W).max())
    it_gpu, it_ref = float(np.sum(its)), float(g["iters_mean"].sum())
    _record("c1_cube_100", pre_steps=pre, contacts_absdiff_max_pre=max(d_nc[:pre]),
            wrench_relerr_max_pre=max(werr[:pre]), contacts_absdiff_max=max(d_nc),
            x_err_gpu=xerr, x_err_ref_fast_mode=fast_x, impulse_relerr_gpu=imp_gpu,
            impulse_relerr_ref_fast_mode=imp_fast, iters_total_gpu=it_gpu,
            iters_total_ref=it_ref, iters_total_ref_fast=float(g["fast_iters_mean"].sum()))
    assert max(d_nc[:pre]) == 0
    assert max(werr[:pre]) <= 1e-6
    assert xerr[10] <= 1e-12 and xerr[25] <= 1e-12
    # after landing the trajectory is sensitive to summation order (the
    # reference's own fast mode moves x by up to 4e-5 m).  A single fast-mode
    # sample is a noisy scale (4.1e-5 at step 75, 1.4e-5 at step 100), so the
    # scale at step k is the envelope max_{j <= k} of the samples, and the bar
    # the larger of 10x the envelope and 0.02 h (each solve stops anywhere below
    # eps_r = 5e-2 of the residual scale; the fused P2G's float64 atomics make
    # the GPU's own roundoff seed differ run to run: 1.2e-4 to 2.2e-4 at step 100)
    h = scene["h"]
    env = 0.0
    for k in (50, 75, 100):
        env = max(env, fast_x[k])
        assert xerr[k] <= max(10.0 * env, 0.02 * h), (k, xerr[k], fast_x[k], env)
    assert imp_gpu <= 5.0 * imp_fast
    assert abs(it_gpu - it_ref) <= 0.1 * it_ref
    np.testing.assert_allclose(np.array([b.position for b in state.bodies]), g["bodies_pos"],
                               rtol=0, atol=1e-12)


def _oracle_from_gpu(scene_1sub, st):
    """The oracle's state built from the GPU state (particles, plastic, body
    poses/velocities at the same step)."""
    p = st.particles.numpy()
    ref = oracle_state(scene_1sub, p["x"], p["v"], p["f"], p["c"], p["mass"], p["volume0"],
                       p["material_id"])
    ref.plastic = p["plastic"].copy()
    for b, gb in zip(ref.bodies, st.bodies):
        b.position, b.quat = gb.position.copy(), gb.quat.copy()
        b.v, b.omega = gb.v.copy(), gb.omega.copy()
    ref.time = st.time
    return ref


def _loaded_substep_parity(mp, half, settle_steps, name):
    """Advance the sand scene on the GPU until the pusher is loaded, then run
    ONE substep from that state on the GPU (op-by-op path, which exposes the
    grid and the solve) and on the oracle, and compare."""
    import copy

    from oracle import step as ostep
    from paper_2503_05046_b200 import scenes
    from paper_2503_05046_b200.coupling import _advance_substep
    scene = scenes.sand_pile_scene(half=half, gap=0.0)
    st = scenes.build_state(scene)
    for _ in range(settle_steps):
        mp.advance_step(st)
    sc1 = copy.deepcopy(scene)
    sc1["dt"] = scene["dt"] / scene["substeps"]
    sc1["substeps"] = 1
    ref = _oracle_from_gpu(sc1, st)
    gst = scenes.build_state(sc1, particles=st.particles.copy())
    for b, gb in zip(gst.bodies, st.bodies):
        b.position, b.quat, b.v, b.omega = gb.position.copy(), gb.quat.copy(), gb.v.copy(), gb.omega.copy()
    gst.time, gst.step_index = st.time, st.step_index
    plan = mp.build_sort_plan(gst.particles.x, gst.h, gst.step_index)
    gst._bias_cache.clear()
    gst._accum.reset()
    info = _advance_substep(gst, sc1["dt"], plan, gst.step_index)
    # the oracle's own sensitivity to summation order: the same substep on a
    # random permutation of the particles (identical physics; P2G and the
    # solver's scatters sum in another order)
    perm = np.random.default_rng(7).permutation(st.particles.n)
    refp = _oracle_from_gpu(sc1, st)
    for k in ("x", "v", "f", "c", "mass", "vol0", "material_id", "plastic"):
        setattr(refp, k, getattr(refp, k)[perm].copy())
    for o in (ref, refp):
        o.cache.clear()
        o.acc_lin[:] = 0.0
        o.acc_ang[:] = 0.0
    r = ostep.substep(ref, sc1["dt"])
    rp = ostep.substep(refp, sc1["dt"])
    grid = info["grid"]
    # grid channels by node id (the block order is bit-exact, so node ids agree)
    n_act = int(np_(grid.active).sum())
    gm = np_(grid.mass)
    mom = np_(grid.mom_apic) + np_(grid.mom_force)
    assert gm.shape == r["mass"].shape
    np.testing.assert_array_equal(np_(grid.active), r["active"])
    mass_err = float(np.abs(gm - r["mass"]).max() / np.abs(r["mass"]).max())
    rmom = r["mom_apic"] + r["mom_force"]
    mom_err = float(np.abs(mom - rmom).max() / np.abs(rmom).max())
    # contacts: identical sets, in the reference's lexsorted order
    nc = info["n_contacts"]
    con = r["contacts"]
    assert nc == con.n, (nc, con.n)
    np.testing.assert_array_equal(np_(info["contacts"].particle), con.particle)
    # impulses: world-frame contact impulses, relative to the largest
    gam = np_(info["gamma_world"])
    rgam = r["gamma_world"]
    gam_err = float(np.abs(gam - rgam).max() / np.abs(rgam).max())
    tot_err = float(np.abs(gam.sum(0) - rgam.sum(0)).max() / np.abs(rgam.sum(0)).max())
    rep, orep = info["report"], r["report"]
    x_err = float(np.abs(np_(gst.particles.x) - ref.x).max())
    # oracle vs permuted oracle, matched by (original particle, body, geom)
    cp = rp["contacts"]
    inv = perm[cp.particle]
    order = np.lexsort((cp.geom, cp.body, inv))
    assert np.array_equal(inv[order], con.particle)
    pgam = rp["gamma_world"][order]
    o_gam = float(np.abs(pgam - rgam).max() / np.abs(rgam).max())
    o_tot = float(np.abs(pgam.sum(0) - rgam.sum(0)).max() / np.abs(rgam.sum(0)).max())
    xp = np.empty_like(refp.x)
    xp[perm] = refp.x
    o_x = float(np.abs(xp - ref.x).max())
    # the fused path (the one the bench times) from the same state
    fst = scenes.build_state(sc1, particles=st.particles.copy())
    for b, gb in zip(fst.bodies, st.bodies):
        b.position, b.quat, b.v, b.omega = gb.position.copy(), gb.quat.copy(), gb.v.copy(), gb.omega.copy()
    fst.time, fst.step_index = st.time, st.step_index
    fs = mp.advance_step(fst)
    fx_err = float(np.abs(np_(fst.particles.x) - ref.x).max())
    rw = np.concatenate([ref.acc_lin, ref.acc_ang], axis=1) / sc1["dt"]
    fw_err = float(np.abs(fs.wrench - rw).max() / np.abs(rw).max())
    assert fs.n_contacts_mean == con.n
    _record(name, n=int(st.particles.n), contacts=int(nc), n_active=n_act,
            iters_gpu=int(rep.iterations), iters_oracle=int(orep.iterations),
            converged_gpu=bool(rep.converged), converged_oracle=bool(orep.converged),
            residual_gpu=float(rep.residual_trace[-1]) if rep.residual_trace else None,
            threshold_gpu=float(rep.threshold_trace[-1]) if rep.threshold_trace else None,
            mass_relerr=mass_err, momentum_relerr=mom_err, gamma_relerr=gam_err,
            gamma_total_relerr=tot_err, x_err=x_err, fused_iters=int(fs.iterations_max),
            fused_x_err=fx_err, fused_wrench_relerr=fw_err,
            oracle_permuted_iters=int(rp["report"].iterations),
            oracle_permuted_gamma_relerr=o_gam, oracle_permuted_gamma_total_relerr=o_tot,
            oracle_permuted_x_err=o_x)
    return dict(mass=mass_err, mom=mom_err, gam=gam_err, tot=tot_err, x=x_err, rep=rep,
                orep=orep, fx=fx_err, fw=fw_err, fconv=fs.all_converged, o_gam=o_gam,
                o_tot=o_tot, o_x=o_x)


@pytest.mark.parametrize("half,settle,name", [
    ((0.2, 0.2, 0.1), 12, "c2_sand_256k_loaded"),
    ((0.4, 0.4, 0.1), 6, "sand_1m_loaded"),
])
def test_sand_loaded_substep_matches_oracle(mp, half, settle, name):
    """configs[1] and the 1M north-star scene, one pusher-loaded substep.

    Bars: node mass and momentum within 1e-12 relative (the reference's own
    fast-vs-deterministic bound, test_transfer.py:85-93); identical contact
    sets; both solves converge.  The solve stops anywhere below eps_r = 5e-2
    of its residual scale, and loaded frictional problems are ill-conditioned
    in the split of the impulse among contacts, so round-off in the summation
    order can move individual impulses far more than round-off.  The oracle
    is therefore also run on a permutation of the particles (same physics,
    another summation order).  When the GPU's solve takes the oracle's path
    (iteration counts within 2), its deviation is held to the larger of 10x the
    permuted oracle's and a floor: world impulses 2e-2 of the largest, their
    total 1e-2, particle positions 1e-7 m (1e-5 h).  Whether it takes that
    path depends on the round-off seed (the fused path's float64 atomics change
    it every run); in every case the aggregates the stopping rule determines
    are held to it: total impulse and fused wrench within eps_r, positions
    within 10 eps_r x 0.2 m/s x dt (2e-5 m, 2e-3 h)."""
    if os.environ.get("MPMRB_SKIP_LARGE"):
        pytest.skip("MPMRB_SKIP_LARGE set")
    d = _loaded_substep_parity(mp, half, settle, name)
    assert d["rep"].converged and d["orep"].converged and d["fconv"]
    assert d["mass"] <= 1e-12 and d["mom"] <= 1e-12
    eps_r = 5e-2  # the scene's stopping tolerance (scenes.sand_pile_scene)
    # the round-off seed decides whether the GPU's iterates follow the
    # oracle's path; when they do, the strict bars hold
    if abs(d["rep"].iterations - d["orep"].iterations) <= 2:
        assert d["gam"] <= max(2e-2, 10 * d["o_gam"])
        assert d["tot"] <= max(1e-2, 10 * d["o_tot"])
        assert d["x"] <= max(1e-7, 10 * d["o_x"])
    # otherwise both stop at different points below the tolerance: the split of
    # the impulse among contacts is not determined (per-contact error up to
    # O(1) of the largest, measured 0.87 with 86 vs 96 iterations), the
    # aggregates are, to about the tolerance: the total impulse to eps_r, x to
    # 10 eps_r x 0.2 m/s x dt (the pusher speed over one substep; measured
    # 4.6e-6 m with 84 vs 91 iterations at 256k)
    xtol = 10 * eps_r * 0.2 * 2e-4
    assert d["tot"] <= max(eps_r, 10 * d["o_tot"])
    assert d["x"] <= max(xtol, 10 * d["o_x"])
    assert d["fw"] <= max(eps_r, 10 * d["o_tot"])
    assert d["fx"] <= max(xtol, 10 * d["o_x"])


def test_tshirt_unconverged_solves_match_oracle(mp):
    """configs[3] (the T-shirt fold) at 16^2 vertices, with its own contact
    stiffness (1e5) and tolerance (eps_r = 5e-2), the sheet dropped onto the
    table: the light cloth's contact solves stop at max_iters = 500 on the
    GPU, and they do so on the oracle too, in the same substeps with the same
    contact counts and iteration counts.  The unconverged solves of the
    full-size bench scene (27 of 80 in its window) are therefore a property of
    the reference algorithm on this scene, not of the port.  Positions agree
    to 1e-5 m (1.3e-3 h; measured 4e-7 to 1.4e-6 m, the unconverged solves'
    stopping points depend on the round-off seed); the wrench is not compared:
    an unconverged solve leaves the split of the impulse undetermined (20-110%
    apart here)."""
    from oracle import step as ostep
    from paper_2503_05046_b200 import scenes
    sc = scenes.tshirt_fold_scene(n_side=16)
    sc["cloth"][0]["center"] = [0.0, 0.0, 0.0012]
    sc["cloth"][0]["velocity"] = [0.0, 0.0, -0.3]
    st = scenes.build_state(sc)
    p0 = st.particles.numpy()
    ref = oracle_state(sc, p0["x"], p0["v"], p0["f"], p0["c"], p0["mass"], p0["volume0"],
                       p0["material_id"])
    rows = []
    for i in range(3):
        s = mp.advance_step(st)
        r = ostep.step(ref)
        dx = float(np.abs(np_(st.particles.x) - ref.x).max())
        rows.append(dict(step=i, contacts=s.n_contacts_mean, iters_mean=s.iterations_mean,
                         iters_max=s.iterations_max, converged=bool(s.all_converged),
                         oracle_contacts=r["n_contacts_mean"],
                         oracle_iters_mean=r["iterations_mean"],
                         oracle_iters_max=r["iterations_max"],
                         oracle_converged=bool(r["all_converged"]), dx=dx))
        assert s.n_contacts_mean == r["n_contacts_mean"], i
        assert s.iterations_max == r["iterations_max"], i
        assert bool(s.all_converged) == bool(r["all_converged"]), i
        assert abs(s.iterations_mean - r["iterations_mean"]) <= 0.02 * r["iterations_mean"], i
        assert dx <= 1e-5, (i, dx)
    assert any(not row["converged"] for row in rows)  # the case this test is about
    _record("tshirt16_unconverged", steps=rows)


def test_sand_256k_first_loaded_step_matches_oracle(mp):
    """configs[1] at full size: step 1 of the bench window (the pusher's first
    loaded rigid step: 10 substeps, one of which stops at max_iters = 500)
    from the GPU state after step 0, on the fused GPU path and on the oracle.
    Contact counts, the max_iters solve and the iteration counts match, and x
    agrees to 1e-16 m in the recorded runs; the bar on x is the
    tolerance-derived 10 eps_r x 0.2 m/s x dt (2e-5 m) of the loaded-substep
    test, since an unconverged solve's stopping point depends on the
    round-off seed."""
    if os.environ.get("MPMRB_SKIP_LARGE"):
        pytest.skip("MPMRB_SKIP_LARGE set")
    from oracle import step as ostep
    from paper_2503_05046_b200 import scenes
    sc = scenes.sand_pile_scene(gap=0.0)  # bench.py workload "sand"
    st = scenes.build_state(sc)
    mp.advance_step(st)
    p = st.particles.numpy()
    ref = oracle_state(sc, p["x"], p["v"], p["f"], p["c"], p["mass"], p["volume0"],
                       p["material_id"])
    ref.plastic = p["plastic"].copy()
    for b, gb in zip(ref.bodies, st.bodies):
        b.position, b.quat = gb.position.copy(), gb.quat.copy()
        b.v, b.omega = gb.v.copy(), gb.omega.copy()
    ref.time, ref.step_index = st.time, st.step_index
    s = mp.advance_step(st)
    r = ostep.step(ref)
    dx = float(np.abs(np_(st.particles.x) - ref.x).max())
    _record("c2_sand_256k_step1", contacts=s.n_contacts_mean, oracle_contacts=r["n_contacts_mean"],
            iters_mean=s.iterations_mean, oracle_iters_mean=r["iterations_mean"],
            iters_max=s.iterations_max, oracle_iters_max=r["iterations_max"],
            converged=bool(s.all_converged), oracle_converged=bool(r["all_converged"]), x_err=dx)
    assert s.n_contacts_mean == r["n_contacts_mean"]
    assert s.iterations_max == r["iterations_max"]
    assert bool(s.all_converged) == bool(r["all_converged"])
    assert abs(s.iterations_mean - r["iterations_mean"]) <= 0.05 * r["iterations_mean"]
    assert dx <= 10 * 5e-2 * 0.2 * 2e-4
