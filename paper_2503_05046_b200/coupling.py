"""Asynchronous MPM / rigid-body coupling — the host scheduler.

``advance_step`` keeps the reference's scheduler on the host
(coupling.py:168-219): N substeps of dt/N against rigid poses frozen at the
step start, then the rigid update.  Each substep is the fused device pipeline
(csrc/sim.cu) replayed as one CUDA graph; the host synchronises once per
step (sizing + statistics), never per substep, solver iteration or
line-search evaluation.

``_advance_substep`` composes the fine-grained GPU operators exactly like the
reference's coupling.py:115-150 (used by tests that inspect intermediates).
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bodies import advance_kinematic_body, geom_structs, integrate_free_body
from .collision import BiasCache, contact_velocities, detect_contacts
from .contact_model import ContactParams, normal_impulse
from .grid import SparseGrid
from .materials import Material, material_table
from .mpm import build_stencil, grid_to_particle, grid_update, particle_to_grid
from .particles import ParticleSet
from .solver import SolveReport, SolverParams, build_contact_problem, quasi_newton_solve
from .transfer import build_sort_plan, plan_staleness

log = logging.getLogger(__name__)


class SimulationDiverged(RuntimeError):
    """Non-finite state was produced; the previous step is the last good one."""


@dataclass(frozen=True)
class StepConfig:
    dt: float
    substeps: int = 1
    gravity: tuple = (0.0, 0.0, -9.81)

    def __post_init__(self):
        if not self.dt > 0:
            raise ValueError("coupling dt must be positive")
        if self.substeps < 1:
            raise ValueError("substeps must be >= 1")


class ImpulseAccumulator:
    """Per-body world-frame impulse totals for the current step (coupling.py:47-66)."""

    def __init__(self, n_bodies: int):
        self.linear = np.zeros((n_bodies, 3))
        self.angular = np.zeros((n_bodies, 3))

    def reset(self):
        self.linear[:] = 0.0
        self.angular[:] = 0.0

    def add_reactions(self, body_ids, gamma_world, arms):
        b = np.asarray(_lib.to_numpy(body_ids), dtype=np.int64)
        gw = np.asarray(_lib.to_numpy(gamma_world), dtype=np.float64)
        arm = np.asarray(_lib.to_numpy(arms), dtype=np.float64)
        mom = np.cross(arm, gw)
        nb = self.linear.shape[0]
        for d in range(3):
            self.linear[:, d] -= np.bincount(b, weights=gw[:, d], minlength=nb)
            self.angular[:, d] -= np.bincount(b, weights=mom[:, d], minlength=nb)


@dataclass
class StepSummary:
    step_index: int
    time: float
    n_particles: int
    n_active_nodes: float = 0.0
    n_contacts_mean: float = 0.0
    n_contacts_max: int = 0
    iterations_mean: float = 0.0
    iterations_max: int = 0
    all_converged: bool = True
    staleness: float = 0.0
    clamped_gradients: int = 0
    wrench: np.ndarray = None
    wall_ms: float | None = None
    ls_evals: int = 0
    # solves that stopped at max_iters (solver.py:358-362) and their iterations
    substeps_unconverged: int = 0
    iterations_unconverged: int = 0


@dataclass
class SimState:
    particles: ParticleSet
    materials: list
    bodies: list
    h: float
    step: StepConfig
    contact_params: ContactParams = field(default_factory=ContactParams)
    solver_params: SolverParams = field(default_factory=SolverParams)
    mode: str = "deterministic"
    workers: int | None = None
    cloth: object | None = None  # cloth.ClothMesh (NEW: codimensional cloth)
    # NEW (north_star): "f64" is the reference's float64 throughout; "f32" is
    # the performance mode of the fused path (float32 particle state and
    # arithmetic; positions, grid and contact solve float64), see
    # include/mpmrb_b200.h mpmrb_sim_set_precision
    precision: str = "f64"
    time: float = 0.0
    step_index: int = 0
    plan_builds: int = 0
    last_report: SolveReport | None = None

    def __post_init__(self):
        self._bias_cache = BiasCache()
        self._accum = ImpulseAccumulator(len(self.bodies))
        if not self.h > 0:
            raise ValueError("grid spacing h must be positive")
        if self.precision not in ("f64", "f32"):
            raise ValueError("precision must be 'f64' or 'f32'")
        self._sim = None
        self._ctx = None  # the state's own library context (stream, scratch, status)
        self._stream = None

    @property
    def margin(self) -> float:
        m = self.contact_params.margin
        return self.h if m is None else m

    def __del__(self):
        sim = getattr(self, "_sim", None)
        ctx = getattr(self, "_ctx", None)
        try:
            if sim is not None:
                _lib.lib().mpmrb_sim_destroy(sim)
            if ctx is not None:
                _lib.free_ctx(ctx)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


# ------------------------------------------------------------------ fused path

def _ensure_sim(state: SimState):
    """The state's fused simulator, on a library context of its own, so that
    several states (batched environments) can step concurrently from
    different host threads, each on its own stream."""
    if state._sim is None:
        L = _lib.lib()
        state._ctx = _lib.new_ctx()
        _lib.bind_stream(state._ctx, _stream_of(state))
        h = C.c_void_p()
        _lib.check(L.mpmrb_sim_create(state._ctx, C.byref(h)))
        state._sim = h
    return state._sim


def _stream_of(state: SimState) -> torch.cuda.Stream:
    if state._stream is None:
        state._stream = torch.cuda.Stream(device=_lib.device())
    return state._stream


def _configure_sim(state: SimState, sim, dt_s: float) -> None:
    """Hand the state's particles, materials, cloth, bodies and parameters to
    the fused simulator (on the state's stream; advance_step and slab.py)."""
    L = _lib.lib()
    p = state.particles
    nb = len(state.bodies)
    pv = p.view()
    _lib.check(L.mpmrb_sim_set_precision(
        sim, _lib.PREC_F32 if state.precision == "f32" else _lib.PREC_F64))
    _lib.check(L.mpmrb_sim_set_particles(sim, C.byref(pv)))
    tab, nm = material_table(state.materials)
    _lib.check(L.mpmrb_sim_set_materials(sim, tab, nm))
    cl = state.cloth
    if cl is not None and cl.n_elements > 0:
        _lib.check(L.mpmrb_sim_set_cloth(sim, cl.n_elements, _lib.ptr(cl.tri),
                                         _lib.ptr(cl.epart), _lib.ptr(cl.dm_inv),
                                         _lib.ptr(cl.vol), _lib.ptr(cl.d3),
                                         _lib.ptr(cl.role)))
    else:
        _lib.check(L.mpmrb_sim_set_cloth(sim, 0, None, None, None, None, None, None))
    gs = geom_structs(state.bodies)
    garr = (_lib.Geom * max(1, len(gs)))(*gs)
    _lib.check(L.mpmrb_sim_set_geoms(sim, garr, len(gs), nb))
    cp, sp = state.contact_params, state.solver_params
    g = (C.c_double * 3)(*[float(a) for a in state.step.gravity])
    spc = sp.to_struct()
    _lib.check(L.mpmrb_sim_set_params(sim, float(state.h), float(dt_s), g,
                                      float(cp.stiffness), float(cp.tau_d), float(cp.eps_v),
                                      float(state.margin), C.byref(spc)))


STAGES = ("grid_build", "p2g", "grid_update", "contacts", "solve", "reactions", "g2p")


def advance_step(state: SimState, profile: dict | None = None) -> StepSummary:
    """Advance one coupling step of size dt (N fused substeps + rigid update).

    ``profile``: if a dict is given, the step's first substep runs with direct
    launches and CUDA events between its stages; the dict receives the stage
    times (ms) and sizes (used by bench.py's live roofline)."""
    L = _lib.lib()
    p = state.particles
    sim = _ensure_sim(state)
    stream = _stream_of(state)
    stream.wait_stream(torch.cuda.current_stream())
    n = state.step.substeps
    dt = state.step.dt
    dt_s = dt / n
    epoch = state.step_index
    stats = _lib.StepStats()
    nb = len(state.bodies)
    imp = (C.c_double * (6 * max(nb, 1)))()
    with torch.cuda.stream(stream):
        _lib.bind_stream(state._ctx, stream)
        _configure_sim(state, sim, dt_s)
        rc = L.mpmrb_sim_begin_step(sim, epoch, n)
        if rc == _lib.E_DIVERGED:
            raise SimulationDiverged(
                f"non-finite or out-of-range particle state after step {state.step_index}")
        _lib.check(rc)
        state.plan_builds += 1
        for k in range(n):
            if profile is not None and k == 0:
                ms = (C.c_float * 7)()
                sz = (C.c_int32 * 5)()
                if profile.get("ncu"):  # bracket exactly this substep for ncu
                    torch.cuda.synchronize()
                    torch.cuda.profiler.start()
                _lib.check(L.mpmrb_sim_profile_substep(sim, ms, sz))
                if profile.get("ncu"):
                    torch.cuda.synchronize()
                    torch.cuda.profiler.stop()
                profile["stage_ms"] = dict(zip(STAGES, [float(a) for a in ms]))
                profile.update(n_blocks=int(sz[0]), n_active=int(sz[1]), n_contacts=int(sz[2]),
                               iterations=int(sz[3]), ls_evals=int(sz[4]))
                continue
            _lib.check(L.mpmrb_sim_substep(sim))
        rc = L.mpmrb_sim_end_step(sim, C.byref(stats), imp)
    if rc == _lib.E_DIVERGED:
        raise SimulationDiverged(f"non-finite particle state after step {state.step_index}")
    _lib.check(rc)
    acc = np.frombuffer(imp, dtype=np.float64)[: 6 * nb].reshape(nb, 6) if nb else np.zeros((0, 6))
    state._accum.linear[:] = acc[:, 0:3]
    state._accum.angular[:] = acc[:, 3:6]
    if stats.regularized:
        log.warning("regularized %d near-singular Hessian blocks this step", stats.regularized)
    if not stats.all_converged:
        log.warning("contact solve hit max_iters=%d in %d of %d substeps of step %d",
                    state.solver_params.max_iters, stats.substeps_unconverged, n,
                    state.step_index)
    if stats.clamped:
        log.warning("clamped %d inverted deformation gradients (singular value floor %.2f)",
                    stats.clamped, 0.05)
    new_time = state.time + dt
    wrench = np.concatenate([state._accum.linear / dt, state._accum.angular / dt], axis=1)
    _rigid_update(state, new_time)
    summary = StepSummary(
        step_index=state.step_index, time=new_time, n_particles=p.n,
        n_active_nodes=float(stats.n_active_mean), n_contacts_mean=float(stats.n_contacts_mean),
        n_contacts_max=int(stats.n_contacts_max), iterations_mean=float(stats.iterations_mean),
        iterations_max=int(stats.iterations_max), all_converged=bool(stats.all_converged),
        staleness=_last_staleness(state), clamped_gradients=int(stats.clamped), wrench=wrench,
        ls_evals=int(stats.ls_evals), substeps_unconverged=int(stats.substeps_unconverged),
        iterations_unconverged=int(stats.iterations_unconverged))
    state.last_report = SolveReport(converged=bool(stats.all_converged),
                                    iterations=int(stats.iterations_max),
                                    n_contacts=int(stats.n_contacts_max),
                                    n_dofs=int(3 * stats.n_active_mean))
    state.time = new_time
    state.step_index += 1
    return summary


def _last_staleness(state: SimState) -> float:
    return float(_staleness_c(state._sim))


def _staleness_c(sim) -> float:
    # staleness is computed in end_step and kept inside the sim; expose via a
    # tiny accessor so the summary matches coupling.py:212
    return _lib.lib().mpmrb_sim_staleness(sim)


def _rigid_update(state: SimState, new_time: float):
    dt = state.step.dt
    for b_idx, body in enumerate(state.bodies):
        if body.kinematic:
            advance_kinematic_body(body, new_time)
        else:
            integrate_free_body(body, state._accum.linear[b_idx], state._accum.angular[b_idx],
                                state.step.gravity, dt)
            if not (np.isfinite(body.position).all() and np.isfinite(body.v).all()):
                raise SimulationDiverged(
                    f"non-finite rigid state for {body.name!r} after step {state.step_index}")


# ------------------------------------------------------------------ op-by-op path

def _advance_substep(state: SimState, dt_s: float, plan, epoch: int) -> dict:
    """coupling.py:115-150 composed from the fine-grained GPU operators."""
    p = state.particles
    grid = SparseGrid.allocate(p.x, state.h)
    stencil = build_stencil(p.x, grid)
    particle_to_grid(p, grid, stencil, state.materials, dt_s, plan, epoch, mode=state.mode,
                     workers=state.workers)
    grid_update(grid, state.step.gravity, dt_s)
    contacts = detect_contacts(p, state.bodies, state.margin, state._bias_cache)
    gamma_world = _lib.zeros((0, 3))
    if contacts.n == 0:
        grid.v_next = grid.v_star
        report = SolveReport(converged=True, n_contacts=0,
                             n_dofs=3 * int(grid.active.sum()))
    else:
        vcs = contact_velocities(contacts, stencil, grid.v_k)
        contacts.gamma_lag = normal_impulse(vcs[:, 2], contacts.phi, state.contact_params, dt_s)
        problem, act = build_contact_problem(grid, stencil, contacts, state.contact_params, dt_s,
                                             plan, epoch, mode=state.mode, workers=state.workers)
        v_sol, gamma, report = quasi_newton_solve(problem, state.solver_params)
        grid.v_next = _lib.zeros((grid.n_nodes, 3))
        grid.v_next[act] = v_sol
        gamma_world = torch.einsum("ci,cij->cj", gamma, contacts.frames)
        bpos = torch.as_tensor(np.stack([np.asarray(b.position) for b in state.bodies]),
                               dtype=torch.float64, device=gamma.device)
        arms = contacts.witness - bpos[contacts.body]
        state._accum.add_reactions(contacts.body, gamma_world, arms)
    clamped = grid_to_particle(p, grid, stencil, dt_s, state.materials)
    state.last_report = report
    return dict(n_contacts=contacts.n, report=report, clamped=clamped,
                n_active=int(grid.active.sum()), contacts=contacts, gamma_world=gamma_world,
                grid=grid)


def _check_particle_health(state: SimState) -> None:
    p = state.particles
    if not p.n:
        return
    if not (bool(torch.isfinite(p.x).all()) and bool(torch.isfinite(p.v).all())):
        raise SimulationDiverged(f"non-finite particle state after step {state.step_index}")
    if float(p.x.abs().max()) >= state.h * float(2 ** 20 - 2):
        raise SimulationDiverged("particle positions left the representable grid region "
                                 f"after step {state.step_index}")


def advance_step_ops(state: SimState) -> StepSummary:
    """advance_step built from the fine-grained operators (no fused graph);
    the reference-shaped path, kept for parity tests and debugging."""
    p = state.particles
    _check_particle_health(state)
    epoch = state.step_index
    plan = build_sort_plan(p.x, state.h, epoch)
    state.plan_builds += 1
    state._bias_cache.clear()
    state._accum.reset()
    n = state.step.substeps
    dt_s = state.step.dt / n
    ncs, its, acts, clamped, conv = [], [], [], 0, True
    for _ in range(n):
        info = _advance_substep(state, dt_s, plan, epoch)
        ncs.append(info["n_contacts"])
        its.append(info["report"].iterations)
        acts.append(info["n_active"])
        conv &= info["report"].converged
        clamped += info["clamped"]
        _check_particle_health(state)
    dt = state.step.dt
    new_time = state.time + dt
    wrench = np.concatenate([state._accum.linear / dt, state._accum.angular / dt], axis=1)
    _rigid_update(state, new_time)
    summary = StepSummary(step_index=state.step_index, time=new_time, n_particles=p.n,
                          n_active_nodes=float(np.mean(acts)), n_contacts_mean=float(np.mean(ncs)),
                          n_contacts_max=int(np.max(ncs)), iterations_mean=float(np.mean(its)),
                          iterations_max=int(np.max(its)), all_converged=conv,
                          staleness=plan_staleness(plan, p.x, state.h),
                          clamped_gradients=clamped, wrench=wrench)
    state.time = new_time
    state.step_index += 1
    return summary
