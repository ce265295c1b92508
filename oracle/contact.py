"""Oracle: particle-vs-geometry contact detection and the lagged convex
contact model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  quaternion -> matrix      /root/reference/pkg/src/mpmrb/rotations.py:33-39
  BiasCache first sight     collision.py:55-85
  detect_contacts           collision.py:88-132 (phi < margin; lexsort particle, body, geom)
  contact_velocities        collision.py:135-143
  gain / target / gamma_n   contact_model.py:42-55
  energy / gradient / Hessian / fused grad+Hessian   contact_model.py:62-138

Bodies are duck-typed: any object with ``position, quat (w,x,y,z), v, omega``
and ``geoms`` whose items have ``shape, position, quat, mu`` works (the
product's and the reference's RigidBody both qualify).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import sdf


def quat_matrix(q) -> np.ndarray:
    w, x, y, z = (float(a) for a in q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


@dataclass
class Contacts:
    particle: np.ndarray
    body: np.ndarray
    geom: np.ndarray
    phi: np.ndarray
    normal: np.ndarray
    witness: np.ndarray
    frames: np.ndarray
    bias: np.ndarray
    mu: np.ndarray
    gamma_lag: np.ndarray

    @property
    def n(self) -> int:
        return int(self.phi.shape[0])


def empty_contacts() -> Contacts:
    z = np.zeros(0)
    zi = np.zeros(0, dtype=np.int64)
    return Contacts(zi, zi.copy(), zi.copy(), z, np.zeros((0, 3)), np.zeros((0, 3)),
                    np.zeros((0, 3, 3)), np.zeros((0, 3)), z.copy(), z.copy())


class FirstSightBias:
    """Bias memo keyed by (body, geom) -> {particle: bias}; cleared each step."""

    def __init__(self):
        self.memo: dict[tuple[int, int], dict[int, np.ndarray]] = {}

    def clear(self):
        self.memo.clear()

    def resolve(self, key, pids, fresh):
        table = self.memo.setdefault(key, {})
        out = fresh.copy()
        for i, pid in enumerate(pids.tolist()):
            if pid in table:
                out[i] = table[pid]
            else:
                table[pid] = fresh[i].copy()
        return out


def detect(x: np.ndarray, bodies, margin: float, cache: FirstSightBias | None = None) -> Contacts:
    """All (particle, body, geom) with phi < margin, lexsorted by that triple."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] == 0 or not bodies:
        return empty_contacts()
    chunks = []
    for bi, body in enumerate(bodies):
        rb = quat_matrix(body.quat)
        bpos = np.asarray(body.position, dtype=np.float64)
        for gi, g in enumerate(body.geoms):
            rg = rb @ quat_matrix(g.quat)
            pg = bpos + rb @ np.asarray(g.position, dtype=np.float64)
            loc = (x - pg) @ rg
            phi, n_loc, w_loc = sdf.query(g.shape, loc)
            hit = np.flatnonzero(phi < margin)
            if hit.size == 0:
                continue
            nrm = n_loc[hit] @ rg.T
            wit = w_loc[hit] @ rg.T + pg
            fr = sdf.frames(nrm)
            vpt = np.asarray(body.v, dtype=np.float64) + np.cross(
                np.asarray(body.omega, dtype=np.float64), wit - bpos)
            fresh = -np.einsum("cij,cj->ci", fr, vpt)
            bias = fresh if cache is None else cache.resolve((bi, gi), hit, fresh)
            chunks.append((hit, np.full(hit.size, bi), np.full(hit.size, gi), phi[hit], nrm,
                           wit, fr, bias, np.full(hit.size, float(g.mu))))
    if not chunks:
        return empty_contacts()
    cols = [np.concatenate([c[i] for c in chunks]) for i in range(9)]
    order = np.lexsort((cols[2], cols[1], cols[0]))
    cols = [c[order] for c in cols]
    return Contacts(cols[0].astype(np.int64), cols[1].astype(np.int64),
                    cols[2].astype(np.int64), cols[3], cols[4], cols[5], cols[6], cols[7],
                    cols[8], np.zeros(cols[3].shape[0]))


def gather_velocity(weights, nodes, frames, bias, v_grid) -> np.ndarray:
    """v_c = R (sum_i w_i v_i) + b for (nc,27) stencils (collision.py:135-143)."""
    if frames.shape[0] == 0:
        return np.zeros((0, 3))
    vp = np.einsum("ck,cki->ci", weights, v_grid[nodes])
    return np.einsum("cij,cj->ci", frames, vp) + bias


# ------------------------------------------------------------ contact model

def gain(k: float, tau_d: float, dt: float) -> float:
    return dt * (dt + tau_d) * k


def target_velocity(phi, tau_d: float, dt: float):
    return -np.asarray(phi) / (dt + tau_d)


def lagged_normal(v_n, phi, k, tau_d, dt):
    """gamma_n = K max(0, vhat - v_n) (contact_model.py:50-55)."""
    return gain(k, tau_d, dt) * np.maximum(0.0, target_velocity(phi, tau_d, dt) - np.asarray(v_n))


def _slip(vc):
    return np.sqrt(vc[:, 0] * vc[:, 0] + vc[:, 1] * vc[:, 1])


def energy(vc, phi, gamma_lag, mu, k, tau_d, eps_v, dt):
    K = gain(k, tau_d, dt)
    gap = np.maximum(0.0, target_velocity(phi, tau_d, dt) - vc[:, 2])
    s = _slip(vc)
    hub = np.where(s <= eps_v, s * s / (2.0 * eps_v), s - 0.5 * eps_v)
    return 0.5 * K * gap * gap + mu * gamma_lag * hub


def gradient(vc, phi, gamma_lag, mu, k, tau_d, eps_v, dt):
    g = np.empty((vc.shape[0], 3))
    g[:, 2] = -lagged_normal(vc[:, 2], phi, k, tau_d, dt)
    a = mu * gamma_lag / np.maximum(_slip(vc), eps_v)
    g[:, 0] = a * vc[:, 0]
    g[:, 1] = a * vc[:, 1]
    return g


def hessian(vc, phi, gamma_lag, mu, k, tau_d, eps_v, dt):
    """PSD contact-frame blocks; normal uses the active side at v_n == vhat."""
    n = vc.shape[0]
    G = np.zeros((n, 3, 3))
    on = vc[:, 2] <= target_velocity(phi, tau_d, dt)
    G[:, 2, 2] = np.where(on, gain(k, tau_d, dt), 0.0)
    s = _slip(vc)
    a = mu * gamma_lag / np.maximum(s, eps_v)
    b = np.where(s > eps_v, a / np.maximum(s * s, eps_v * eps_v), 0.0)
    G[:, 0, 0] = a - b * vc[:, 0] * vc[:, 0]
    G[:, 1, 1] = a - b * vc[:, 1] * vc[:, 1]
    G[:, 0, 1] = G[:, 1, 0] = -b * vc[:, 0] * vc[:, 1]
    return G


def grad_hess(vc, phi, gamma_lag, mu, k, tau_d, eps_v, dt):
    """Fused variant used by the line search (contact_model.py:114-138).

    Normal activity is tested as gap >= 0, equivalent to v_n <= vhat.
    """
    K = gain(k, tau_d, dt)
    gap = target_velocity(phi, tau_d, dt) - vc[:, 2]
    n = vc.shape[0]
    g = np.empty((n, 3))
    G = np.zeros((n, 3, 3))
    g[:, 2] = -K * np.maximum(0.0, gap)
    G[:, 2, 2] = np.where(gap >= 0.0, K, 0.0)
    s = _slip(vc)
    a = mu * gamma_lag / np.maximum(s, eps_v)
    g[:, 0] = a * vc[:, 0]
    g[:, 1] = a * vc[:, 1]
    b = np.where(s > eps_v, a / np.maximum(s * s, eps_v * eps_v), 0.0)
    G[:, 0, 0] = a - b * vc[:, 0] * vc[:, 0]
    G[:, 1, 1] = a - b * vc[:, 1] * vc[:, 1]
    G[:, 0, 1] = G[:, 1, 0] = -b * vc[:, 0] * vc[:, 1]
    return g, G
