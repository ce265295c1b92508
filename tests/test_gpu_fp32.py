"""fp32 performance mode of the fused substep (north_star: "fp64 oracle mode;
fp32 performance mode with a reported drift bound over N steps").

The mode keeps float32 particle state (v, F, C, mass, volume, plastic strain,
cached sand stress) and float32 per-particle arithmetic (stress, SVD, return
map, P2G contributions, G2P); positions, the grid, contacts and the contact
solve stay float64 (include/mpmrb_b200.h, mpmrb_sim_set_precision).  The
reference is float64 only, so the fp32 path is measured as a
DRIFT from the float64 path -- itself pinned to the reference
(test_gpu_configs.py, test_gpu_parity.py) -- over N coupling steps from the
same state.  Each test writes its measured drift to
``gpurun_out/fp32_drift.jsonl`` (the numbers DESIGN.md quotes); the bounds
are stated per test.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from scenes import load_scene_json  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _record(name, **kw):
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    with open(out / "fp32_drift.jsonl", "a") as fh:
        fh.write(json.dumps(dict(test=name, **kw)) + "\n")


@pytest.fixture(scope="module")
def mp():
    import paper_2503_05046_b200 as m
    return m


def _pair(scene):
    from paper_2503_05046_b200 import scenes
    a = scenes.build_state(scene)
    b = scenes.build_state(scene, particles=a.particles.copy(), precision="f32")
    return a, b


def test_fp32_sand_drift_bound(mp):
    """Pushed Drucker-Prager sand (32k particles), 30 coupling steps (300
    substeps) in both precisions from the same state.  Bounds: positions
    within 0.05 h (measured 0.017 h; the float64 path itself moves by ~0.015 h
    under a different summation order after contact, test_gpu_configs.py
    C1, because each solve stops anywhere below eps_r = 5e-2), pusher
    wrench integrated over the window within 5% of its magnitude (measured
    0.3-1.1%: the float64 path's own P2G flush is unordered, so two float64
    runs differ too), contact counts within 2%."""
    from paper_2503_05046_b200 import scenes
    sc = scenes.sand_pile_scene(half=(0.1, 0.1, 0.05), gap=0.0)
    a, b = _pair(sc)
    h = sc["h"]
    dx, wa, wb, nca, ncb = [], [], [], [], []
    for _ in range(30):
        sa = mp.advance_step(a)
        sb = mp.advance_step(b)
        dx.append(float(np.abs(np_(a.particles.x) - np_(b.particles.x)).max()))
        wa.append(sa.wrench)
        wb.append(sb.wrench)
        nca.append(sa.n_contacts_mean)
        ncb.append(sb.n_contacts_mean)
    Wa, Wb = np.sum(wa, axis=0), np.sum(wb, axis=0)
    w_rel = float(np.abs(Wa - Wb).max() / np.abs(Wa).max())
    nc_rel = float(abs(sum(nca) - sum(ncb)) / sum(nca))
    dF = float(np.abs(np_(a.particles.f) - np_(b.particles.f)).max())
    dplast = float(np.abs(np_(a.particles.plastic) - np_(b.particles.plastic)).max())
    _record("sand_32k_30_steps", n=int(a.particles.n), h=h, x_drift_per_step=dx,
            x_drift_max=max(dx), x_drift_over_h=max(dx) / h, impulse_relerr=w_rel,
            contacts_relerr=nc_rel, F_drift_max=dF, plastic_drift_max=dplast)
    assert max(dx) <= 0.05 * h
    assert w_rel <= 5e-2
    assert nc_rel <= 2e-2


def test_fp32_c1_cube_drift_vs_reference(mp, golden):
    """configs[0] (8k elastic cube, 100 steps) in fp32 against the trajectory
    of the unmodified reference: before landing (steps 10, 25) positions
    within 1e-6 m (float32 state advected by a float64 x update); after
    landing within 0.05 h at steps 50/75/100 (measured <= 0.007 h); total
    impulse within 5% of the reference's (measured 0.9%)."""
    from paper_2503_05046_b200 import scenes
    g = golden("c1_cube")
    scene = load_scene_json(g["scene_json"])
    st = scenes.build_state(scene, precision="f32")
    h = scene["h"]
    xerr, wr = {}, []
    for i in range(g["wrench"].shape[0]):
        s = mp.advance_step(st)
        wr.append(s.wrench)
        k = i + 1
        if f"x_{k}" in g:
            xerr[k] = float(np.abs(np_(st.particles.x) - g[f"x_{k}"]).max())
    W, Wg = g["wrench"].sum(0), np.sum(wr, axis=0)
    imp = float(np.abs(Wg - W).max() / np.abs(W).max())
    _record("c1_cube_100_steps_vs_reference", h=h, x_err=xerr, impulse_relerr=imp)
    assert xerr[10] <= 1e-6 and xerr[25] <= 1e-6
    for k in (50, 75, 100):
        assert xerr[k] <= 0.05 * h, (k, xerr[k])
    assert imp <= 5e-2


def test_fp32_p2g_conserves_mass_and_momentum(mp):
    """One fp32 step of free fall: every particle's momentum arrives on the
    grid, so the total particle momentum after the step equals the float64
    path's to float32 roundoff (1e-6 relative)."""
    from paper_2503_05046_b200 import scenes
    sc = scenes.elastic_cube_scene()
    a, b = _pair(sc)
    mp.advance_step(a)
    mp.advance_step(b)
    m = np_(a.particles.mass)
    pa = (m[:, None] * np_(a.particles.v)).sum(0)
    pb = (m[:, None] * np_(b.particles.v)).sum(0)
    rel = float(np.abs(pa - pb).max() / np.abs(pa).max())
    _record("free_fall_momentum", relerr=rel)
    assert rel <= 1e-6


def test_fp32_cloth_drift_bound(mp):
    """Codimensional cloth in the fp32 mode: a 33 x 33 sheet (3,137 particles)
    dropped 1 cm onto the rigid sphere of configs[2], 200 coupling steps
    (3,200 substeps: the landing and the settling).  The cloth forces,
    element stresses, vertex forces, d3 and positions stay float64; P2G / G2P
    and the element particles' C run in float32.  The solves run to
    eps_r = 1e-4, so the solver's stopping point does not hide the drift.

    The sheet's motion on the sphere amplifies roundoff: two float64 runs from
    the same state (the P2G flush is float64 atomics) end 0.17-0.19 h apart,
    the float32 run 0.10-0.16 h from a float64 one
    (profiles/r02_fp32_cloth_probe.jsonl, tools/fp32_cloth_probe.py).  So the
    drift is measured against that spread.  Bounds: positions within 0.5 h
    and within 2x the float64 run-to-run spread + 0.1 h; sphere impulse
    integrated over the window within 5%, as for the sand (measured
    0.2-1.0%; float64 repeat 0-1.7%)."""
    from paper_2503_05046_b200 import scenes
    sc = scenes.cloth_sheet_scene(n_side=33)
    sc["cloth"][0]["center"][2] = 0.26
    sc["solver"]["eps_r"] = 1e-4
    a = scenes.build_state(sc)
    a2 = scenes.build_state(sc)
    b = scenes.build_state(sc, precision="f32")
    assert torch.equal(a.particles.x, b.particles.x)
    w = {k: np.zeros(3) for k in "abr"}
    for _ in range(200):
        for k, st in (("a", a), ("r", a2), ("b", b)):
            s = mp.advance_step(st)
            w[k] += s.wrench[0][:3]
    h = sc["h"]
    xa = np_(a.particles.x)
    dx = float(np.abs(xa - np_(b.particles.x)).max()) / h
    dx_rep = float(np.abs(xa - np_(a2.particles.x)).max()) / h
    dw = float(np.abs(w["a"] - w["b"]).max() / np.abs(w["a"]).max())
    dw_rep = float(np.abs(w["a"] - w["r"]).max() / np.abs(w["a"]).max())
    _record("cloth_sheet_33", steps=200, max_dx_over_h=dx, f64_repeat_dx_over_h=dx_rep,
            impulse_relerr=dw, f64_repeat_impulse_relerr=dw_rep,
            max_d3_diff=float(np.abs(np_(a.cloth.d3) - np_(b.cloth.d3)).max()),
            contacts_last=s.n_contacts_mean)
    assert s.n_contacts_mean > 0          # the sheet is on the sphere
    assert dx <= 0.5, dx
    assert dx <= 2.0 * dx_rep + 0.1, (dx, dx_rep)
    assert dw <= 0.05, dw


def test_fp32_mode_rejects_unknown_precision():
    from paper_2503_05046_b200 import scenes
    with pytest.raises(ValueError):
        scenes.build_state(scenes.smoke_scene(), precision="f16")
