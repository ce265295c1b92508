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

    def impulses(self, v, vc=None) -> torch.Tensor:
        from .contact_model import contact_impulses
        if self.n_contacts == 0:
            return _lib.zeros((0, 3))
        vc = self.contact_velocities(v) if vc is None else _lib.as_dev(vc)
        return contact_impulses(vc, self.phi, self.gamma_lag, self.mu, self.contact_params,
                                self.dt)

    # ---- the reference's host-side building blocks of the solve
    # (solver.py:111-194), on the device: contact velocities, the contact model
    # and the ordered scatter are this package's kernels.  The fused solve
    # (k_qn_solve) evaluates the same quantities inside one kernel; these are
    # the API-level equivalents for callers of the reference's ContactProblem.

    def energy(self, v, vc=None) -> float:
        """solver.py:111-119: 1/2 |v - v*|_M^2 + sum of contact energies."""
        from .contact_model import contact_energy
        v = _lib.as_dev(v)
        dv = v - self.v_star
        e = 0.5 * float(torch.sum(self.m[:, None] * dv * dv))
        if self.n_contacts:
            vc = self.contact_velocities(v) if vc is None else _lib.as_dev(vc)
            e += float(torch.sum(contact_energy(vc, self.phi, self.gamma_lag, self.mu,
                                                self.contact_params, self.dt)))
        return e

    def _scatter_contact(self, vals) -> torch.Tensor:
        from .transfer import scatter_reduce
        return scatter_reduce(self.nodes, vals.contiguous(), int(self.m.shape[0]), self.plan,
                              self.epoch, mode=self.mode, workers=self.workers,
                              particle_ids=self.particle_ids)

    def gradient(self, v, vc=None):
        """solver.py:127-140: (total gradient, contact part J^T dl/dv_c)."""
        from .contact_model import contact_gradient
        v = _lib.as_dev(v)
        g = self.m[:, None] * (v - self.v_star)
        if self.n_contacts == 0:
            return g, torch.zeros_like(g)
        vc = self.contact_velocities(v) if vc is None else _lib.as_dev(vc)
        g_c = contact_gradient(vc, self.phi, self.gamma_lag, self.mu, self.contact_params,
                               self.dt)
        g_world = torch.einsum("ci,cij->cj", g_c, self.frames)  # R^T g_c per contact
        jt = self._scatter_contact(self.w[:, :, None] * g_world[:, None, :])
        return g + jt, jt

    def hessian_blocks(self, v, vc=None) -> torch.Tensor:
        """solver.py:151-167: m_i I + sum_c w_ic^2 R^T G R, (nd, 3, 3)."""
        from .contact_model import contact_hessian
        h = torch.diag_embed(self.m[:, None].expand(-1, 3).contiguous())
        if self.n_contacts == 0:
            return h
        v = _lib.as_dev(v)
        vc = self.contact_velocities(v) if vc is None else _lib.as_dev(vc)
        big_g = contact_hessian(vc, self.phi, self.gamma_lag, self.mu, self.contact_params,
                                self.dt)
        rgr = self.frames.transpose(1, 2) @ big_g @ self.frames
        vals = (self.w * self.w)[:, :, None] * rgr.reshape(-1, 1, 9)
        return h + self._scatter_contact(vals).reshape(-1, 3, 3)

    def dense_hessian(self, v) -> torch.Tensor:
        """solver.py:169-186: the full (3nd, 3nd) Hessian with cross-node
        coupling (oracle use; O(nd^2) memory)."""
        from .contact_model import contact_hessian
        nd = int(self.m.shape[0])
        h = torch.diag(self.m.repeat_interleave(3))
        if self.n_contacts == 0:
            return h
        v = _lib.as_dev(v)
        big_g = contact_hessian(self.contact_velocities(v), self.phi, self.gamma_lag, self.mu,
                                self.contact_params, self.dt)
        rgr = torch.einsum("cki,ckl,clj->cij", self.frames, big_g, self.frames)
        ww = self.w[:, :, None] * self.w[:, None, :]                      # (nc, 27, 27)
        blocks = ww[:, :, :, None, None] * rgr[:, None, None, :, :]       # (nc, 27, 27, 3, 3)
        rows = (3 * self.nodes[:, :, None] + torch.arange(3, device=h.device)).reshape(-1, 81)
        vals = blocks.permute(0, 1, 3, 2, 4).reshape(-1, 81, 81)
        flat = h.view(-1)
        idx = rows[:, :, None] * (3 * nd) + rows[:, None, :]
        flat.index_put_((idx.reshape(-1),), vals.reshape(-1), accumulate=True)
        return h

    def residual_threshold(self, v, g, g_contact, params: "SolverParams"):
        """solver.py:188-194: (||g||_M^-1, eps_a + eps_r max(||v||_M, ||J^T dl||_M^-1))."""
        v, g, gc = _lib.as_dev(v), _lib.as_dev(g), _lib.as_dev(g_contact)
        inv_m = 1.0 / self.m
        residual = float(torch.sqrt(torch.sum(g * g * inv_m[:, None])))
        p_norm = float(torch.sqrt(torch.sum(self.m[:, None] * v * v)))
        j_norm = float(torch.sqrt(torch.sum(gc * gc * inv_m[:, None])))
        return residual, params.eps_a + params.eps_r * max(p_norm, j_norm)

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


def solve_search_direction(h_blocks, g) -> torch.Tensor:
    """solver.py:224-256: d = -H^-1 g per SPD 3x3 block (device Cholesky,
    csrc/solver.cu k_search_direction), regularising near-singular blocks like
    the reference; FloatingPointError if one stays non-SPD."""
    h = _lib.as_dev(h_blocks).reshape(-1, 3, 3).contiguous()
    gg = _lib.as_dev(g).reshape(-1, 3).contiguous()
    d = _lib.empty(tuple(gg.shape))
    nreg = C.c_int32(0)
    _lib.check(_lib.lib().mpmrb_search_direction(_lib.ctx(), _lib.ptr(h), _lib.ptr(gg),
                                                 h.shape[0], _lib.ptr(d), C.byref(nreg)))
    if nreg.value:
        log.warning("regularizing %d near-singular Hessian blocks", nreg.value)
    return d


def _directional_derivatives(problem: ContactProblem, v, dv, vc0):
    """solver.py:301-325: phi'(a), phi''(a) along dv (device contact model)."""
    from .contact_model import contact_grad_hess
    mdv = problem.m[:, None] * dv
    a1 = float(torch.sum((v - problem.v_star) * mdv))
    a2 = float(torch.sum(dv * mdv))
    dvc = None
    if problem.n_contacts:
        dv_p = torch.einsum("ck,ckd->cd", problem.w, dv[problem.nodes])
        dvc = torch.einsum("cij,cj->ci", problem.frames, dv_p)

    def deriv(alpha: float):
        d, dd = a1 + a2 * alpha, a2
        if dvc is not None:
            g_c, big_g = contact_grad_hess(vc0 + alpha * dvc, problem.phi, problem.gamma_lag,
                                           problem.mu, problem.contact_params, problem.dt)
            d += float(torch.sum(g_c * dvc))
            dd += float(torch.sum(dvc * torch.einsum("cij,cj->ci", big_g, dvc)))
        return d, dd

    return deriv


def dense_newton_oracle(problem: ContactProblem, params: SolverParams, v0=None):
    """solver.py:385-389: full-Hessian Newton with the reference's test-last
    loop and exact line search (solver.py:328-365), driven from the host over
    device arrays -- a test oracle, O((3nd)^3) per iteration."""
    v = (problem.v_init if v0 is None else _lib.as_dev(v0)).clone()
    report = SolveReport(n_contacts=problem.n_contacts, n_dofs=problem.n_dofs)
    vc = problem.contact_velocities(v) if problem.n_contacts else None
    g, g_c = problem.gradient(v, vc)
    residual, threshold = problem.residual_threshold(v, g, g_c, params)
    report.objective_trace.append(problem.energy(v, vc))
    report.residual_trace.append(residual)
    report.threshold_trace.append(threshold)
    for it in range(params.max_iters):
        if residual < (threshold if it > 0 else params.eps_a):
            report.converged = True
            break
        dv = torch.linalg.solve(problem.dense_hessian(v), -g.reshape(-1)).reshape(-1, 3)
        ls = line_search(_directional_derivatives(problem, v, dv, vc),
                         max_iters=params.ls_max_iters, tol=params.ls_tol)
        v = v + ls.alpha * dv
        report.iterations += 1
        report.alpha_trace.append(ls.alpha)
        vc = problem.contact_velocities(v) if problem.n_contacts else None
        g, g_c = problem.gradient(v, vc)
        residual, threshold = problem.residual_threshold(v, g, g_c, params)
        report.objective_trace.append(problem.energy(v, vc))
        report.residual_trace.append(residual)
        report.threshold_trace.append(threshold)
    else:
        report.converged = residual < threshold
    if not bool(torch.isfinite(v).all()):
        raise FloatingPointError("contact solve produced non-finite velocities")
    return v, problem.impulses(v, vc), report


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
