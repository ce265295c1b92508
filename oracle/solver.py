"""Oracle: the block-diagonal quasi-Newton convex contact solve.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates /root/reference/pkg/src/mpmrb/solver.py:
  problem restriction to active nodes    :197-221 (dead slots -> w = 0, node 0)
  objective / gradient / Hessian blocks  :104-167
  residual + threshold                   :188-194
  3x3 Cholesky direction + regularise    :224-256
  exact line search                      :266-298
  directional derivatives                :301-325
  test-last minimisation loop            :328-365 (iteration 0 tests eps_a only)
  dense Newton (oracle of the oracle)    :169-186, 373-388
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import contact as cm


@dataclass
class Params:
    eps_a: float = float(np.finfo(np.float64).eps)
    eps_r: float = 5e-2
    max_iters: int = 500
    ls_max_iters: int = 50
    ls_tol: float = 1e-8


@dataclass
class Report:
    converged: bool = False
    iterations: int = 0
    n_contacts: int = 0
    n_dofs: int = 0
    objective: list = field(default_factory=list)
    residual: list = field(default_factory=list)
    threshold: list = field(default_factory=list)
    alpha: list = field(default_factory=list)
    ls_evals: list = field(default_factory=list)


class LineSearchError(ValueError):
    pass


@dataclass
class Problem:
    m: np.ndarray
    v_star: np.ndarray
    v_init: np.ndarray
    nodes: np.ndarray
    w: np.ndarray
    frames: np.ndarray
    bias: np.ndarray
    phi: np.ndarray
    mu: np.ndarray
    gamma_lag: np.ndarray
    k: float
    tau_d: float
    eps_v: float
    dt: float

    @property
    def nc(self) -> int:
        return int(self.phi.shape[0])

    def _cm(self):
        return (self.phi, self.gamma_lag, self.mu, self.k, self.tau_d, self.eps_v, self.dt)

    def vc(self, v):
        if self.nc == 0:
            return np.zeros((0, 3))
        return cm.gather_velocity(self.w, self.nodes, self.frames, self.bias, v)

    def scatter(self, vals):
        from .grid import scatter_in_order
        return scatter_in_order(self.nodes, vals, self.m.shape[0])

    def objective(self, v, vc):
        d = v - self.v_star
        e = 0.5 * np.sum(self.m[:, None] * d * d)
        if self.nc:
            e += np.sum(cm.energy(vc, *self._cm()))
        return float(e)

    def grad(self, v, vc):
        g = self.m[:, None] * (v - self.v_star)
        if self.nc == 0:
            return g, np.zeros_like(g)
        gc = cm.gradient(vc, *self._cm())
        gw = np.einsum("ci,cij->cj", gc, self.frames)
        jt = self.scatter(self.w[:, :, None] * gw[:, None, :])
        return g + jt, jt

    def hess_blocks(self, v, vc):
        H = np.zeros((self.m.shape[0], 3, 3))
        for d in range(3):
            H[:, d, d] = self.m
        if self.nc == 0:
            return H
        G = cm.hessian(vc, *self._cm())
        rgr = np.swapaxes(self.frames, 1, 2) @ G @ self.frames
        vals = (self.w * self.w)[:, :, None] * rgr.reshape(-1, 1, 9)
        return H + self.scatter(vals).reshape(-1, 3, 3)

    def dense_hessian(self, v):
        nd = self.m.shape[0]
        H = np.diag(np.repeat(self.m, 3)).astype(np.float64)
        if self.nc == 0:
            return H
        G = cm.hessian(self.vc(v), *self._cm())
        rgr = np.einsum("cki,ckl,clj->cij", self.frames, G, self.frames)
        for c in range(self.nc):
            for a in range(27):
                for b in range(27):
                    wab = self.w[c, a] * self.w[c, b]
                    if wab == 0.0:
                        continue
                    ia, ib = 3 * self.nodes[c, a], 3 * self.nodes[c, b]
                    H[ia:ia + 3, ib:ib + 3] += wab * rgr[c]
        return H

    def residual_threshold(self, v, g, jt, p: Params):
        inv_m = 1.0 / self.m
        res = float(np.sqrt(np.sum(g * g * inv_m[:, None])))
        pn = float(np.sqrt(np.sum(self.m[:, None] * v * v)))
        jn = float(np.sqrt(np.sum(jt * jt * inv_m[:, None])))
        return res, p.eps_a + p.eps_r * max(pn, jn)

    def impulses(self, vc):
        if self.nc == 0:
            return np.zeros((0, 3))
        return -cm.gradient(vc, *self._cm())


def restrict(active, mass, v_star, v_k, st_nodes, st_w, contacts, k, tau_d, eps_v, dt):
    """Build the active-node problem (solver.py:197-221). Returns (problem, act)."""
    act = np.flatnonzero(active)
    remap = np.full(active.shape[0], -1, dtype=np.int64)
    remap[act] = np.arange(act.shape[0])
    if contacts.n:
        nodes = remap[st_nodes[contacts.particle]]
        w = st_w[contacts.particle].copy()
        dead = nodes < 0
        w[dead] = 0.0
        nodes[dead] = 0
    else:
        nodes = np.zeros((0, 27), dtype=np.int64)
        w = np.zeros((0, 27))
    prob = Problem(mass[act], v_star[act], v_k[act], nodes, w, contacts.frames, contacts.bias,
                   contacts.phi, contacts.mu, contacts.gamma_lag, k, tau_d, eps_v, dt)
    return prob, act


def cholesky_direction(H, g):
    """d = -H^-1 g per 3x3 block; bad blocks get +1e-12 max(tr,1) 10^a (a<4)."""
    H = H
    for attempt in range(4):
        with np.errstate(invalid="ignore", divide="ignore"):
            l11 = np.sqrt(H[:, 0, 0])
            l21 = H[:, 1, 0] / l11
            l31 = H[:, 2, 0] / l11
            l22 = np.sqrt(H[:, 1, 1] - l21 * l21)
            l32 = (H[:, 2, 1] - l31 * l21) / l22
            l33 = np.sqrt(H[:, 2, 2] - l31 * l31 - l32 * l32)
            good = (np.isfinite(l11) & np.isfinite(l22) & np.isfinite(l33)
                    & (l11 > 0) & (l22 > 0) & (l33 > 0))
        if good.all():
            break
        if attempt == 3:
            raise FloatingPointError("Hessian block not SPD after regularization")
        H = H.copy()
        bad = ~good
        tr = H[bad, 0, 0] + H[bad, 1, 1] + H[bad, 2, 2]
        bump = 1e-12 * np.maximum(tr, 1.0) * (10.0 ** attempt)
        for d in range(3):
            H[bad, d, d] += bump
    y1 = -g[:, 0] / l11
    y2 = (-g[:, 1] - l21 * y1) / l22
    y3 = (-g[:, 2] - l31 * y1 - l32 * y2) / l33
    x3 = y3 / l33
    x2 = (y2 - l32 * x3) / l22
    x1 = (y1 - l21 * x2 - l31 * x3) / l11
    return np.stack([x1, x2, x3], axis=1)


def exact_line_search(deriv, max_evals=50, tol=1e-8):
    """1-D Newton on phi'(alpha) with bracketing (solver.py:266-298).

    Returns (alpha, evals, phi'(alpha)).
    """
    d0, _ = deriv(0.0)
    if not np.isfinite(d0) or d0 >= 0.0:
        raise LineSearchError(f"line search needs a descent direction, phi'(0) = {d0:.6e}")
    lo, hi, a, d = 0.0, np.inf, 1.0, d0
    for ev in range(1, max_evals + 1):
        d, dd = deriv(a)
        if abs(d) <= tol * abs(d0):
            return a, ev, d
        if d > 0.0:
            hi = a
        else:
            lo = a
        nxt = a - d / dd if (np.isfinite(dd) and dd > 0.0) else np.nan
        if np.isfinite(hi):
            if not np.isfinite(nxt) or not (lo < nxt < hi):
                nxt = 0.5 * (lo + hi)
        elif not np.isfinite(nxt) or nxt <= lo:
            nxt = 2.0 * max(a, 1e-8)
        a = nxt
    return (lo if lo > 0.0 else a), max_evals, d


def _deriv_along(prob: Problem, v, dv, vc0):
    mdv = prob.m[:, None] * dv
    a1 = float(np.sum((v - prob.v_star) * mdv))
    a2 = float(np.sum(dv * mdv))
    if prob.nc:
        dvc = np.einsum("cij,cj->ci", prob.frames,
                        np.einsum("ck,cki->ci", prob.w, dv[prob.nodes]))
    else:
        dvc = None

    def deriv(alpha):
        d, dd = a1 + a2 * alpha, a2
        if dvc is not None:
            g, G = cm.grad_hess(vc0 + alpha * dvc, *prob._cm())
            d += float(np.sum(g * dvc))
            dd += float(np.sum(dvc * np.einsum("cij,cj->ci", G, dvc)))
        return d, dd

    return deriv


def minimise(prob: Problem, p: Params, v0=None, dense=False):
    """Test-last quasi-Newton loop (solver.py:328-365). Returns (v, gamma, report)."""
    v = (prob.v_init if v0 is None else v0).copy()
    rep = Report(n_contacts=prob.nc, n_dofs=3 * prob.m.shape[0])
    vc = prob.vc(v) if prob.nc else None
    g, jt = prob.grad(v, vc)
    res, thr = prob.residual_threshold(v, g, jt, p)
    rep.objective.append(prob.objective(v, vc))
    rep.residual.append(res)
    rep.threshold.append(thr)
    converged_early = False
    for it in range(p.max_iters):
        if res < (thr if it > 0 else p.eps_a):
            converged_early = True
            break
        if dense:
            dv = np.linalg.solve(prob.dense_hessian(v), -g.ravel()).reshape(-1, 3)
        else:
            dv = cholesky_direction(prob.hess_blocks(v, vc), g)
        alpha, evals, _ = exact_line_search(_deriv_along(prob, v, dv, vc),
                                            p.ls_max_iters, p.ls_tol)
        v = v + alpha * dv
        rep.iterations += 1
        rep.alpha.append(alpha)
        rep.ls_evals.append(evals)
        vc = prob.vc(v) if prob.nc else None
        g, jt = prob.grad(v, vc)
        res, thr = prob.residual_threshold(v, g, jt, p)
        rep.objective.append(prob.objective(v, vc))
        rep.residual.append(res)
        rep.threshold.append(thr)
    rep.converged = converged_early or res < thr
    if not np.isfinite(v).all():
        raise FloatingPointError("contact solve produced non-finite velocities")
    return v, prob.impulses(vc) if prob.nc else np.zeros((0, 3)), rep
