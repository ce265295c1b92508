"""Known-answer tests of the cloth oracle (oracle/cloth.py; parity unpinned:
the reference has no cloth).  The forces must be the exact negative gradient
of the energy, the rest state must be stress free, and the return mapping
must land on the friction cone."""

import numpy as np
import pytest

from oracle import cloth as oc


def _mesh(seed=0, n_side=4, jitter=0.02, d3_jitter=0.1):
    p = oc.params_from(3.2e6, 0.4, friction=0.3)
    x, mass, vol, mid, mesh = oc.sheet([0.0, 0.0, 0.3], (0.1, 0.1), n_side, 1e-3, 1500.0, p, 0)
    rng = np.random.default_rng(seed)
    x = x + jitter * 0.1 * rng.normal(size=x.shape)
    mesh.d3 = mesh.d3 + d3_jitter * rng.normal(size=mesh.d3.shape)
    return x, mesh


def test_rest_state_is_stress_free():
    p = oc.params_from(1e5, 0.3)
    x, _, _, _, mesh = oc.sheet([0, 0, 0.1], (0.2, 0.1), 5, 1e-3, 1000.0, p, 0)
    fext, tau, P = oc.forces(x, mesh)
    assert np.abs(fext).max() < 1e-9
    assert np.abs(P).max() < 1e-9
    assert oc.energy(x, mesh) == pytest.approx(0.0, abs=1e-18)


def test_qr_reconstructs_and_is_orthonormal():
    x, mesh = _mesh(1)
    F = oc.deformation(x, mesh)
    Q, R = oc.qr_gs(F)
    np.testing.assert_allclose(Q @ R, F, atol=1e-13)
    np.testing.assert_allclose(np.swapaxes(Q, 1, 2) @ Q, np.tile(np.eye(3), (len(F), 1, 1)),
                               atol=1e-13)
    assert np.all(np.tril(R, -1) == 0.0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_vertex_forces_are_minus_energy_gradient(seed):
    x, mesh = _mesh(seed)
    fext, _, _ = oc.forces(x, mesh)
    eps = 1e-7
    verts = np.unique(mesh.tri)
    rng = np.random.default_rng(seed + 10)
    for i in rng.choice(verts, size=6, replace=False):
        for d in range(3):
            xp, xm = x.copy(), x.copy()
            xp[i, d] += eps
            xm[i, d] -= eps
            g = (oc.energy(xp, mesh) - oc.energy(xm, mesh)) / (2 * eps)
            assert fext[i, d] == pytest.approx(-g, rel=1e-5, abs=1e-6 * np.abs(fext).max())


@pytest.mark.parametrize("seed", [0, 3])
def test_transverse_stress_is_energy_gradient_in_d3(seed):
    x, mesh = _mesh(seed, d3_jitter=0.3)
    _, tau, P = oc.forces(x, mesh)
    eps = 1e-7
    for e in range(0, len(mesh.vol), 5):
        for d in range(3):
            dp, dm = mesh.d3.copy(), mesh.d3.copy()
            dp[e, d] += eps
            dm[e, d] -= eps
            g = (oc.energy(x, mesh, dp) - oc.energy(x, mesh, dm)) / (2 * eps)
            assert mesh.vol[e] * P[e, d, 2] == pytest.approx(g, rel=1e-5, abs=1e-9)
    # tau_e = (P e3) d3^T
    np.testing.assert_allclose(tau, P[:, :, 2][:, :, None] * mesh.d3[:, None, :])


def test_return_map_separation_and_friction_cone():
    p = oc.params_from(1e5, 0.3, friction=0.3)
    F = np.tile(np.eye(3), (3, 1, 1))
    F[0, :, 2] = [0.3, 0.0, 1.5]      # separated: r33 > 1 -> (0, 0, 1)
    F[1, :, 2] = [0.5, 0.0, 0.6]      # compressed with large shear -> scaled onto the cone
    F[2, :, 2] = [1e-6, 0.0, 0.6]     # inside the cone: unchanged
    d3 = oc.return_map(F, p)
    np.testing.assert_allclose(d3[0], [0, 0, 1], atol=1e-15)
    lim = p.friction * p.k_normal * (1 - 0.6) ** 2 / p.gamma_shear
    np.testing.assert_allclose(d3[1], [lim, 0, 0.6], rtol=1e-12)
    np.testing.assert_allclose(d3[2], F[2, :, 2], rtol=1e-12)


def test_vertex_forces_are_internal():
    """The in-plane forces of every triangle sum to zero force (the torque is
    balanced by the transverse term acting through d3, not checked here)."""
    x, mesh = _mesh(4, jitter=0.05)
    fext, _, _ = oc.forces(x, mesh)
    assert np.abs(fext.sum(axis=0)).max() <= 1e-10 * np.abs(fext).max()


def test_oracle_cloth_step_conserves_momentum_in_free_space():
    """No gravity, no bodies: a stretched, spinning sheet keeps its linear
    momentum through full coupling steps (P2G/G2P and the cloth forces are
    momentum conserving); element particles stay at their face centroids."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from oracle import step as ostep
    from paper_2503_05046_b200 import scenes as S
    from scenes import oracle_state
    sc = S.cloth_sheet_scene(n_side=10)
    sc["bodies"] = []
    sc["gravity"] = [0.0, 0.0, 0.0]
    a = S.cloth_arrays(sc)[0]
    n = a["x"].shape[0]
    x = a["x"].copy()
    x[:, 0] *= 1.04
    v = 0.3 * np.cross([0.0, 0.0, 1.0], x - x.mean(axis=0))
    st = oracle_state(sc, x, v, np.tile(np.eye(3), (n, 1, 1)), np.zeros((n, 3, 3)),
                      a["mass"], a["vol"], a["mid"])
    p0 = (st.mass[:, None] * st.v).sum(axis=0)
    for _ in range(3):
        ostep.step(st)
    p1 = (st.mass[:, None] * st.v).sum(axis=0)
    np.testing.assert_allclose(p1, p0, atol=1e-12 * (1.0 + np.abs(st.mass[:, None] * st.v).sum()))
    np.testing.assert_allclose(st.x[st.cloth.epart], st.x[st.cloth.tri].mean(axis=1), atol=1e-15)
