"""Convex contact solve: block-preconditioned quasi-Newton with exact line
search, entirely on the GPU (reference solver.py:1-388).

``quasi_newton_solve`` launches ONE persistent kernel (csrc/solver.cu) that
runs every iteration and every line-search evaluation on the device, with
grid-wide reductions; the host reads back only the result and the traces.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .contact_model import ContactParams

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class SolverParams:
    eps_a: float = float(np.finfo(np.float64).eps)
    eps_r: float = 5e-2
    max_iters: int = 500
    ls_max_iters: int = 50
    ls_tol: float = 1e-8

    def __post_init__(self):
        if self.eps_a < 0 or self.eps_r < 0 or (self.eps_a == 0 and self.eps_r == 0):
            raise ValueError("need eps_a >= 0, eps_r >= 0, not both zero")
        if self.max_iters < 1 or self.ls_max_iters < 1:
            raise ValueError("iteration limits must be >= 1")
        if not self.ls_tol > 0:
            raise ValueError("ls_tol must be positive")

    def to_struct(self) -> _lib.SolverParamsC:
        s = _lib.SolverParamsC()
        s.eps_a, s.eps_r, s.ls_tol = self.eps_a, self.eps_r, self.ls_tol
        s.max_iters, s.ls_max_iters = self.max_iters, self.ls_max_iters
        return s


@dataclass
class SolveReport:
    converged: bool = False
    iterations: int = 0
    n_contacts: int = 0
    n_dofs: int = 0
    objective_trace: list = field(default_factory=list)
    residual_trace: list = field(default_factory=list)
    threshold_trace: list = field(default_factory=list)
    alpha_trace: list = field(default_factory=list)
    ls_evals: int = 0
    regularized: int = 0

    def log_lines(self) -> list[str]:
        out = [f"contact solve: {self.n_contacts} contacts, {self.n_dofs} dofs, "
               f"converged={self.converged} in {self.iterations} iterations"]
        for i, (o, r, t) in enumerate(zip(self.objective_trace, self.residual_trace,
                                          self.threshold_trace)):
            a = self.alpha_trace[i - 1] if 0 < i <= len(self.alpha_trace) else float("nan")
            out.append(f"  iter {i}: objective={o:.12e} residual={r:.6e} "
                       f"threshold={t:.6e} alpha={a:.6e}")
        return out


@dataclass
class ContactProblem:
    """One substep's solve restricted to active nodes (solver.py:75-110)."""

    m: torch.Tensor
    v_star: torch.Tensor
    v_init: torch.Tensor
    nodes: torch.Tensor
    w: torch.Tensor
    frames: torch.Tensor
    bias: torch.Tensor
    phi: torch.Tensor
    mu: torch.Tensor
    gamma_lag: torch.Tensor
    contact_params: ContactParams
    dt: float
    plan: object = None
    epoch: int = 0
    particle_ids: torch.Tensor | None = None
    mode: str = "deterministic"
    workers: int | None = None

    def __post_init__(self):
        for k in ("m", "v_star", "v_init", "w", "frames", "bias", "phi", "mu", "gamma_lag"):
            setattr(self, k, _lib.as_dev(getattr(self, k)))
        self.nodes = _lib.as_dev(self.nodes, torch.int64)

    @property
    def n_dofs(self) -> int:
        return 3 * int(self.m.shape[0])

    @property
    def n_contacts(self) -> int:
        return int(self.phi.shape[0])

    def contact_velocities(self, v) -> torch.Tensor:
        from .collision import _contact_velocities_raw
        if self.n_contacts == 0:
            return _lib.zeros((0, 3))
        return _contact_velocities_raw(self.nodes, self.w, self.frames, self.bias, v)

    def impulses(self, v) -> torch.Tensor:
        from .contact_model import contact_impulses
        if self.n_contacts == 0:
            return _lib.zeros((0, 3))
        return contact_impulses(self.contact_velocities(v), self.phi, self.gamma_lag, self.mu,
                                self.contact_params, self.dt)

    def to_struct(self) -> _lib.Problem:
        p = _lib.Problem()
        p.n_nodes = int(self.m.shape[0])
        p.n_contacts = self.n_contacts
        for k in ("m", "v_star", "v_init", "nodes", "w", "frames", "bias", "phi", "mu",
                  "gamma_lag"):
            setattr(p, k, _lib.ptr(getattr(self, k)))
        cp = self.contact_params
        p.stiffness, p.tau_d, p.eps_v, p.dt = cp.stiffness, cp.tau_d, cp.eps_v, float(self.dt)
        return p


def build_contact_problem(grid, stencil, contacts, contact_params: ContactParams, dt: float,
                          plan, epoch: int, mode: str = "deterministic",
                          workers: int | None = None):
    """Restrict the grid to active nodes (solver.py:197-221); returns (problem, act)."""
    act = torch.nonzero(grid.active, as_tuple=False).reshape(-1)
    remap = torch.full((grid.n_nodes,), -1, dtype=torch.int64, device=act.device)
    remap[act] = torch.arange(act.shape[0], device=act.device)
    if contacts.n:
        nodes = remap[stencil.nodes[contacts.particle]]
        w = stencil.weights[contacts.particle].clone()
        dead = nodes < 0
        w[dead] = 0.0
        nodes[dead] = 0
    else:
        nodes = torch.zeros((0, 27), dtype=torch.int64, device=act.device)
        w = _lib.zeros((0, 27))
    prob = ContactProblem(m=grid.mass[act], v_star=grid.v_star[act], v_init=grid.v_k[act],
                          nodes=nodes, w=w, frames=contacts.frames, bias=contacts.bias,
                          phi=contacts.phi, mu=contacts.mu, gamma_lag=contacts.gamma_lag,
                          contact_params=contact_params, dt=dt, plan=plan, epoch=epoch,
                          particle_ids=contacts.particle, mode=mode, workers=workers)
    return prob, act


@dataclass
class LineSearchResult:
    alpha: float
    evals: int
    derivative: float


def line_search(deriv, max_iters: int = 50, tol: float = 1e-8) -> LineSearchResult:
    """Scalar exact line search (solver.py:266-298), identical branch logic to
    the device kernel's P_ls phase; usable with any phi'(a), phi''(a) callable."""
    d0, _ = deriv(0.0)
    if not np.isfinite(d0) or d0 >= 0.0:
        raise ValueError(f"line search needs a descent direction, phi'(0) = {d0:.6e}")
    lo, hi, a, d = 0.0, np.inf, 1.0, d0
    for it in range(1, max_iters + 1):
        d, dd = deriv(a)
        if abs(d) <= tol * abs(d0):
            return LineSearchResult(alpha=a, evals=it, derivative=d)
        if d > 0.0:
            hi = a
        else:
            lo = a
        cand = a - d / dd if (np.isfinite(dd) and dd > 0.0) else np.nan
        if np.isfinite(hi):
            if not (lo < cand < hi) or not np.isfinite(cand):
                cand = 0.5 * (lo + hi)
        elif not np.isfinite(cand) or cand <= lo:
            cand = 2.0 * max(a, 1e-8)
        a = cand
    return LineSearchResult(alpha=lo if lo > 0.0 else a, evals=max_iters, derivative=d)


def quasi_newton_solve(problem: ContactProblem, params: SolverParams, v0=None):
    """Block-preconditioned solve on the device; returns (v, gamma, report)."""
    v, gamma, report, _ = _solve(problem, params, v0, None)
    return v, gamma, report


def quasi_newton_solve_ext(problem: ContactProblem, params: SolverParams, ext_free, v0=None):
    """The solve with contact-free nodes held elsewhere (slab decomposition,
    slab.py): ext_free = (S0, Q0, Q1) of those nodes (S0 = sum m|v0 - v*|^2,
    Q0 = sum m|v*|^2, Q1 = sum m v*.(v0 - v*)).  Returns (v, gamma, report, P)
    with P = prod(1 - alpha): the external nodes end at v* + P (v0 - v*)."""
    return _solve(problem, params, v0, ext_free)


def _solve(problem: ContactProblem, params: SolverParams, v0, ext_free):
    nd, nc = int(problem.m.shape[0]), problem.n_contacts
    v = _lib.empty((nd, 3))
    gamma = _lib.empty((nc, 3))
    T = params.max_iters + 1
    tr = _lib.empty((4, T))
    rep = _lib.SolveReportC()
    pr = problem.to_struct()
    sp = params.to_struct()
    v0d = _lib.as_dev(v0) if v0 is not None else None
    P = C.c_double(1.0)
    if ext_free is None:
        _lib.check(_lib.lib().mpmrb_qn_solve(_lib.ctx(), C.byref(pr), C.byref(sp), _lib.ptr(v0d),
                                             _lib.ptr(v), _lib.ptr(gamma), _lib.ptr(tr[0]),
                                             _lib.ptr(tr[1]), _lib.ptr(tr[2]), _lib.ptr(tr[3]),
                                             C.byref(rep)))
    else:
        ext = (C.c_double * 3)(*[float(e) for e in ext_free])
        _lib.check(_lib.lib().mpmrb_qn_solve_ext(
            _lib.ctx(), C.byref(pr), C.byref(sp), _lib.ptr(v0d), ext, _lib.ptr(v),
            _lib.ptr(gamma), _lib.ptr(tr[0]), _lib.ptr(tr[1]), _lib.ptr(tr[2]), _lib.ptr(tr[3]),
            C.byref(P), C.byref(rep)))
    it = int(rep.iterations)
    trh = _lib.to_numpy(tr)
    report = SolveReport(converged=bool(rep.converged), iterations=it, n_contacts=nc,
                         n_dofs=3 * nd, objective_trace=trh[0, : it + 1].tolist(),
                         residual_trace=trh[1, : it + 1].tolist(),
                         threshold_trace=trh[2, : it + 1].tolist(),
                         alpha_trace=trh[3, :it].tolist(), ls_evals=int(rep.ls_evals),
                         regularized=int(rep.regularized))
    if report.regularized:
        log.warning("regularized %d near-singular Hessian blocks", report.regularized)
    if not report.converged:
        log.warning("contact solve hit max_iters=%d (residual %.3e, threshold %.3e)",
                    params.max_iters, report.residual_trace[-1], report.threshold_trace[-1])
    return v, gamma, report, float(P.value)
