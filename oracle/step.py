"""Oracle: one coupling substep and one coupling step (async time splitting).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates /root/reference/pkg/src/mpmrb/coupling.py:
  impulse accumulation   :47-66, gamma_world / arms :141-144
  _advance_substep       :115-150 (zero contacts -> v_next = v_star bitwise)
  health check           :153-165
  advance_step           :168-219 (plan once per step, wrench = accum / dt)
and the host-side rigid update it calls (bodies.py:116-137, rotations.py:41-84),
which the CUDA path also keeps on the host.

State is held in ``OracleState`` (plain NumPy arrays) so the oracle never
touches the product's device tensors.  Bodies are duck-typed objects with
mutable ``position, quat, v, omega`` plus ``kinematic, mass, inertia_body,
trajectory, geoms`` (the product's ``RigidBody`` qualifies); the oracle mutates
them, so tests hand it a deep copy.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import cloth as ocl
from . import contact as cm
from . import grid as og
from . import mpm as om
from . import plasticity as opl
from . import solver as osv
from .contact import quat_matrix


class OracleDiverged(RuntimeError):
    pass


@dataclass
class OracleState:
    x: np.ndarray
    v: np.ndarray
    f: np.ndarray
    c: np.ndarray
    mass: np.ndarray
    vol0: np.ndarray
    material_id: np.ndarray
    materials: list            # objects with youngs_modulus, poisson_ratio (+ optional DP fields)
    bodies: list
    h: float
    dt: float
    substeps: int = 1
    gravity: tuple = (0.0, 0.0, -9.81)
    k: float = 1e5
    tau_d: float = 1e-3
    eps_v: float = 1e-4
    margin: float | None = None
    solver: osv.Params = field(default_factory=osv.Params)
    time: float = 0.0
    step_index: int = 0
    plastic: np.ndarray | None = None   # per-particle DP hardening / log-volume state
    cloth: object | None = None         # oracle.cloth.ClothMesh (codimensional cloth)

    def __post_init__(self):
        self.cache = cm.FirstSightBias()
        nb = len(self.bodies)
        self.acc_lin = np.zeros((nb, 3))
        self.acc_ang = np.zeros((nb, 3))
        if self.plastic is None:
            self.plastic = np.zeros(self.x.shape[0])

    @property
    def det_margin(self) -> float:
        return self.h if self.margin is None else self.margin


def check_health(s: OracleState):
    if s.x.shape[0] == 0:
        return
    if not (np.isfinite(s.x).all() and np.isfinite(s.v).all()):
        raise OracleDiverged(f"non-finite particle state after step {s.step_index}")
    if np.abs(s.x).max() >= s.h * float(2 ** 20 - 2):
        raise OracleDiverged(f"particles left the representable region after step {s.step_index}")


def substep(s: OracleState, dt_s: float) -> dict:
    """One substep (coupling.py:115-150). Returns a dict of intermediates."""
    keys = og.allocate_blocks(s.x, s.h)
    n_nodes = keys.shape[0] * og.NODES_PER_BLOCK
    st = og.make_stencil(s.x, keys, s.h)
    extra_tau = fext = keep_f = None
    if s.cloth is not None:  # mesh forces before the transfer (oracle/cloth.py)
        fext, tau_e, _ = ocl.forces(s.x, s.cloth)
        extra_tau = np.zeros((s.x.shape[0], 3, 3))
        extra_tau[s.cloth.epart] = tau_e
        keep_f = s.cloth.roles(s.x.shape[0]) != ocl.ROLE_NONE
    mass, mom_apic, mom_force = om.p2g(s.x, s.v, s.f, s.c, s.mass, s.vol0, s.material_id,
                                       s.materials, st, dt_s, n_nodes, extra_tau, fext)
    active, v_k, v_star = om.grid_update(mass, mom_apic, mom_force, s.gravity, dt_s)
    con = cm.detect(s.x, s.bodies, s.det_margin, s.cache)
    gamma_world = np.zeros((0, 3))
    report = osv.Report(converged=True, n_dofs=3 * int(active.sum()))
    if con.n == 0:
        v_next = v_star
    else:
        vcs = cm.gather_velocity(st.weights[con.particle], st.nodes[con.particle], con.frames,
                                 con.bias, v_k)
        con.gamma_lag = cm.lagged_normal(vcs[:, 2], con.phi, s.k, s.tau_d, dt_s)
        prob, act = osv.restrict(active, mass, v_star, v_k, st.nodes, st.weights, con, s.k,
                                 s.tau_d, s.eps_v, dt_s)
        v_sol, gamma, report = osv.minimise(prob, s.solver)
        v_next = np.zeros((n_nodes, 3))
        v_next[act] = v_sol
        gamma_world = np.einsum("ci,cij->cj", gamma, con.frames)
        arms = con.witness - np.stack([np.asarray(s.bodies[b].position, dtype=np.float64)
                                       for b in con.body])
        moments = np.cross(arms, gamma_world)
        nb = len(s.bodies)
        for d in range(3):
            s.acc_lin[:, d] -= np.bincount(con.body, weights=gamma_world[:, d], minlength=nb)
            s.acc_ang[:, d] -= np.bincount(con.body, weights=moments[:, d], minlength=nb)
    x_old = s.x
    s.x, s.v, s.c, f_new, clamped = om.g2p(s.x, s.f, st, v_next, dt_s, keep_f)
    s.f, s.plastic = opl.return_map(f_new, s.plastic, s.material_id, s.materials)
    if s.cloth is not None:
        s.x = ocl.post_g2p(s.x, s.c, s.cloth, dt_s)
    return dict(keys=keys, stencil=st, mass=mass, mom_apic=mom_apic, mom_force=mom_force,
                active=active, v_k=v_k, v_star=v_star, v_next=v_next, contacts=con,
                report=report, gamma_world=gamma_world, clamped=clamped, x_old=x_old)


# ------------------------------------------------------------ host rigid update

def _qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def _qaxis(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    n = np.linalg.norm(axis)
    if n == 0.0:
        return np.array([1.0, 0.0, 0.0, 0.0])
    return np.concatenate(([np.cos(0.5 * angle)], np.sin(0.5 * angle) * axis / n))


def _qslerp(a, b, t):
    dot = float(np.dot(a, b))
    if dot < 0.0:
        b, dot = -b, -dot
    if dot > 1.0 - 1e-12:
        q = a + t * (b - a)
        return q / np.linalg.norm(q)
    th = np.arccos(np.clip(dot, -1.0, 1.0))
    return (np.sin((1.0 - t) * th) * a + np.sin(t * th) * b) / np.sin(th)


def _qlog_rate(q0, q1, dt):
    dq = _qmul(q1, np.array([q0[0], -q0[1], -q0[2], -q0[3]]))
    if dq[0] < 0.0:
        dq = -dq
    s = np.linalg.norm(dq[1:])
    if s < 1e-15:
        return np.zeros(3)
    return (2.0 * np.arctan2(s, dq[0]) / dt) * (dq[1:] / s)


def sample_trajectory(tr, t):
    """(pos, quat, v, omega), held constant outside the keyframes (bodies.py:56-74)."""
    T = np.asarray(tr.times, dtype=np.float64)
    P = np.asarray(tr.positions, dtype=np.float64)
    Q = np.asarray(tr.quats, dtype=np.float64)
    if t <= T[0]:
        return P[0].copy(), Q[0].copy(), np.zeros(3), np.zeros(3)
    if t >= T[-1]:
        return P[-1].copy(), Q[-1].copy(), np.zeros(3), np.zeros(3)
    i = int(np.searchsorted(T, t, side="right") - 1)
    seg = T[i + 1] - T[i]
    u = (t - T[i]) / seg
    return (P[i] + u * (P[i + 1] - P[i]), _qslerp(Q[i], Q[i + 1], u), (P[i + 1] - P[i]) / seg,
            _qlog_rate(Q[i], Q[i + 1], seg))


def rigid_update(body, lin, ang, gravity, dt, t_new):
    """Kinematic snap to trajectory or free-body impulse integration (bodies.py:116-137)."""
    if body.kinematic:
        if body.trajectory is None:
            body.v = np.zeros(3)
            body.omega = np.zeros(3)
        else:
            body.position, body.quat, body.v, body.omega = sample_trajectory(body.trajectory, t_new)
        return
    body.v = body.v + lin / body.mass + dt * np.asarray(gravity, dtype=np.float64)
    R = quat_matrix(body.quat)
    Iw = R @ body.inertia_body @ R.T
    L = Iw @ body.omega + ang
    w_half = np.linalg.solve(Iw, L)
    th = np.linalg.norm(w_half) * dt
    if th != 0.0:
        q = _qmul(_qaxis(w_half, th), body.quat)
        body.quat = q / np.linalg.norm(q)
    R = quat_matrix(body.quat)
    body.omega = np.linalg.solve(R @ body.inertia_body @ R.T, L)
    body.position = body.position + dt * body.v


def step(s: OracleState) -> dict:
    """One coupling step (coupling.py:168-219). Returns summary dict."""
    check_health(s)
    plan = og.sort_plan(s.x, s.h, s.step_index)
    s.cache.clear()
    s.acc_lin[:] = 0.0
    s.acc_ang[:] = 0.0
    dt_s = s.dt / s.substeps
    ncs, its, acts, clamped, conv = [], [], [], 0, True
    for _ in range(s.substeps):
        info = substep(s, dt_s)
        ncs.append(info["contacts"].n)
        its.append(info["report"].iterations)
        acts.append(int(info["active"].sum()))
        clamped += info["clamped"]
        conv &= info["report"].converged
        check_health(s)
    t_new = s.time + s.dt
    wrench = np.concatenate([s.acc_lin / s.dt, s.acc_ang / s.dt], axis=1)
    for bi, body in enumerate(s.bodies):
        rigid_update(body, s.acc_lin[bi], s.acc_ang[bi], s.gravity, s.dt, t_new)
        if not body.kinematic and not (np.isfinite(body.position).all()
                                       and np.isfinite(body.v).all()):
            raise OracleDiverged("non-finite rigid state")
    out = dict(step_index=s.step_index, time=t_new, n_contacts_mean=float(np.mean(ncs)),
               n_contacts_max=int(np.max(ncs)), iterations_mean=float(np.mean(its)),
               iterations_max=int(np.max(its)), n_active_nodes=float(np.mean(acts)),
               all_converged=conv, clamped=clamped, wrench=wrench,
               staleness=og.staleness(plan, s.x, s.h), plan=plan)
    s.time = t_new
    s.step_index += 1
    return out
