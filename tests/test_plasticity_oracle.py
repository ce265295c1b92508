"""Known-answer tests of the Drucker–Prager oracle (oracle/plasticity.py).

The reference has no plasticity, so these KATs are what
pins the sand model of configs[1]/[4] ("yield-surface
projection, FD-consistent stress").  They are stated independently of the
oracle's vectorised code: scalar math for the expected values, finite
differences of the Hencky energy for the stress, and the yield condition in
stress space for the projection.

Model (Klár et al. 2016, cited at /root/reference/PAPER.md:28):
  psi(F) = mu |log sigma|^2 + lam/2 (tr log sigma)^2,   tau = dpsi/dF F^T
  yield: |dev tau| + alpha tr tau <= 0,  alpha = sqrt(2/3) 2 sin(phi) / (3 - sin(phi))
"""

import math

import numpy as np
import pytest

from oracle import plasticity as P
from oracle.mpm import lame

E, NU = 3.5e5, 0.3
MU, LAM = lame(E, NU)
ALPHA = P.dp_alpha(30.0)


def _rot(axis, ang):
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(ang) * k + (1 - math.cos(ang)) * (k @ k)


def _scalar_project(sig):
    """Scalar restatement of the return map for one particle (KAT source)."""
    eps = [math.log(s) for s in sig]
    tr = sum(eps)
    eh = [e - tr / 3.0 for e in eps]
    en = math.sqrt(sum(e * e for e in eh))
    if tr > 0.0:
        return [1.0, 1.0, 1.0], math.sqrt(sum(e * e for e in eps))
    dg = en + (3 * LAM + 2 * MU) / (2 * MU) * tr * ALPHA
    if dg <= 0.0 or en == 0.0:
        return list(sig), 0.0
    out = [e - dg / en * h for e, h in zip(eps, eh)]
    return [math.exp(e) for e in out], math.sqrt(sum((a - b) ** 2 for a, b in zip(eps, out)))


def _yield(sig):
    """|dev tau| + alpha tr tau for principal stretches sig (stress space)."""
    eps = np.log(sig)
    tau = 2 * MU * eps + LAM * eps.sum()
    dev = tau - tau.mean()
    return np.linalg.norm(dev) + ALPHA * tau.sum(), tau


def test_alpha_kat():
    # 30 deg: sin = 1/2 -> alpha = sqrt(2/3) * 2 * 0.5 / 2.5 = 0.4 sqrt(2/3)
    assert P.dp_alpha(30.0) == pytest.approx(0.4 * math.sqrt(2.0 / 3.0), rel=1e-15)
    assert P.dp_alpha(0.0) == 0.0


def test_case_ii_tension_projects_to_tip():
    s = np.array([[1.02, 1.01, 0.995], [1.1, 1.1, 1.1]])
    sig, dq = P.project(s, MU, LAM, ALPHA)
    np.testing.assert_array_equal(sig, np.ones_like(s))
    np.testing.assert_allclose(dq, np.linalg.norm(np.log(s), axis=1), rtol=1e-15)
    val, tau = _yield(sig[0])
    assert val == 0.0 and np.all(tau == 0.0)


def test_case_i_inside_cone_is_kept():
    # pure compression (ehat = 0) and a mildly sheared compressed state
    s = np.array([[0.98, 0.98, 0.98], [0.97, 0.975, 0.972], [1.0, 1.0, 1.0]])
    sig, dq = P.project(s, MU, LAM, ALPHA)
    np.testing.assert_array_equal(sig, s)
    np.testing.assert_array_equal(dq, 0.0)
    for row in s:
        assert _yield(row)[0] <= 1e-12 * MU


def test_case_iii_projects_onto_the_yield_surface():
    s = np.array([[0.95, 1.0, 1.03], [0.9, 0.99, 1.04], [0.98, 0.97, 1.02], [0.93, 1.0, 1.02]])
    before = np.array([_yield(r)[0] for r in s])
    assert np.all(before > 0)  # outside the cone
    sig, dq = P.project(s, MU, LAM, ALPHA)
    for row_in, row in zip(s, sig):
        val, tau = _yield(row)
        assert abs(val) <= 1e-9 * np.abs(tau).max()          # on the surface
        # volume (trace of log strain) is preserved by the deviatoric return
        assert np.log(row).sum() == pytest.approx(np.log(row_in).sum(), abs=1e-15)
        # the deviatoric direction is preserved (radial return)
        e0 = np.log(row_in) - np.log(row_in).mean()
        e1 = np.log(row) - np.log(row).mean()
        cos = e0 @ e1 / (np.linalg.norm(e0) * np.linalg.norm(e1))
        assert cos == pytest.approx(1.0, abs=1e-12)
    assert np.all(dq > 0)


def test_scalar_kats_match():
    cases = [[0.95, 1.0, 1.03], [1.02, 1.01, 0.995], [0.98, 0.98, 0.98], [0.9, 0.99, 1.04],
             [0.97, 0.975, 0.972], [1.0, 0.8, 1.3], [0.5, 0.6, 0.7]]
    s = np.array(cases)
    sig, dq = P.project(s, MU, LAM, ALPHA)
    for k, row in enumerate(cases):
        es, eq = _scalar_project(row)
        np.testing.assert_allclose(sig[k], es, rtol=1e-14)
        assert dq[k] == pytest.approx(eq, rel=1e-13, abs=1e-16)


def test_projection_is_idempotent():
    rng = np.random.default_rng(3)
    s = np.exp(rng.normal(0.0, 0.05, size=(500, 3)))
    sig, _ = P.project(s, MU, LAM, ALPHA)
    sig2, dq2 = P.project(sig, MU, LAM, ALPHA)
    np.testing.assert_allclose(sig2, sig, rtol=1e-12)
    assert np.all(dq2 <= 1e-12)
    vals = np.array([_yield(r)[0] for r in sig])
    tau_scale = np.array([np.abs(_yield(r)[1]).max() for r in sig]) + 1.0
    assert np.all(vals <= 1e-9 * tau_scale)  # every output is admissible


def _psi(f):
    s = np.linalg.svd(f, compute_uv=False)
    e = np.log(s)
    return MU * (e @ e) + 0.5 * LAM * e.sum() ** 2


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_hencky_stress_is_fd_consistent(seed):
    rng = np.random.default_rng(seed)
    f = np.eye(3) + 0.1 * rng.normal(size=(3, 3))
    assert np.linalg.det(f) > 0
    hstep = 1e-6
    dpsi = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            d = np.zeros((3, 3))
            d[i, j] = hstep
            dpsi[i, j] = (_psi(f + d) - _psi(f - d)) / (2 * hstep)
    tau_fd = dpsi @ f.T
    tau = P.hencky_stress(f[None], MU, LAM)[0]
    np.testing.assert_allclose(tau, tau_fd, rtol=1e-6, atol=1e-6 * np.abs(tau).max())
    np.testing.assert_allclose(tau, tau.T, atol=1e-9 * np.abs(tau).max())  # symmetric


def test_return_map_is_objective_and_keeps_rotation():
    u, v = _rot([1, 2, 3], 0.4), _rot([-2, 1, 0.5], 1.1)
    sig = np.array([0.93, 1.0, 1.04])
    f = u @ np.diag(sig) @ v.T
    q = _rot([0.3, -1, 2], 0.7)
    mats = [type("M", (), dict(model="sand", youngs_modulus=E, poisson_ratio=NU,
                               friction_angle=30.0))()]
    fs = np.stack([f, q @ f])
    out, dq = P.return_map(fs, np.zeros(2), np.zeros(2, np.int64), mats)
    np.testing.assert_allclose(out[1], q @ out[0], atol=1e-13)
    exp_sig, exp_dq = _scalar_project(list(sig))
    np.testing.assert_allclose(out[0], u @ np.diag(exp_sig) @ v.T, atol=1e-13)
    np.testing.assert_allclose(dq, [exp_dq, exp_dq], rtol=1e-12)
    # elastic materials are untouched
    mats_e = [type("M", (), dict(model="elastic", youngs_modulus=E, poisson_ratio=NU))()]
    out_e, dq_e = P.return_map(fs, np.zeros(2), np.zeros(2, np.int64), mats_e)
    np.testing.assert_array_equal(out_e, fs)
    np.testing.assert_array_equal(dq_e, 0.0)


def test_signed_svd_reconstructs_with_rotations():
    rng = np.random.default_rng(11)
    f = rng.normal(size=(64, 3, 3))
    u, s, vt = P.signed_svd(f)
    np.testing.assert_allclose(u @ (s[..., None] * vt), f, atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(u), 1.0, atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(vt), 1.0, atol=1e-12)
    assert np.all(s[:, :2] >= 0)
    np.testing.assert_array_equal(np.sign(s[:, 2]), np.sign(np.linalg.det(f)))
