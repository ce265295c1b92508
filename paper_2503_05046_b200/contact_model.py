"""Lagged convex contact model (reference contact_model.py:1-144).

Per contact, with v_c = (v_t1, v_t2, v_n): gamma_n = K max(0, vhat - v_n),
K = dt (dt + tau_d) k, vhat = -phi / (dt + tau_d); friction potential
mu gamma_lag huber_eps_v(|v_t|).  The per-contact energy / gradient / Hessian
below are evaluated by the SAME device functions the solver kernel inlines
(csrc/contact.cuh: cm_energy, cm_gradient, cm_hessian).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class ContactParams:
    stiffness: float = 1e5
    tau_d: float = 1e-3
    eps_v: float = 1e-4
    margin: float | None = None

    def __post_init__(self):
        if not self.stiffness > 0:
            raise ValueError("contact stiffness must be positive")
        if self.tau_d < 0:
            raise ValueError("tau_d must be non-negative")
        if not self.eps_v > 0:
            raise ValueError("eps_v must be positive")


def impulse_gain(params: ContactParams, dt: float) -> float:
    return dt * (dt + params.tau_d) * params.stiffness


def stabilization_velocity(phi, params: ContactParams, dt: float):
    return -_lib.as_dev(phi) / (dt + params.tau_d)


def normal_impulse(v_n, phi, params: ContactParams, dt: float) -> torch.Tensor:
    """gamma_n = K max(0, vhat - v_n) (contact_model.py:50-55)."""
    vhat = stabilization_velocity(phi, params, dt)
    return impulse_gain(params, dt) * torch.clamp(vhat - _lib.as_dev(v_n), min=0.0)


def _eval(v_c, phi, gamma_lag, mu, params, dt, want):
    vc = _lib.as_dev(v_c).reshape(-1, 3).contiguous()
    n = vc.shape[0]
    ph, gl, m = _lib.as_dev(phi), _lib.as_dev(gamma_lag), _lib.as_dev(mu)
    e = _lib.empty((n,)) if "e" in want else None
    g = _lib.empty((n, 3)) if "g" in want else None
    H = _lib.empty((n, 3, 3)) if "h" in want else None
    _lib.check(_lib.lib().mpmrb_contact_model(
        _lib.ctx(), _lib.ptr(vc), _lib.ptr(ph), _lib.ptr(gl), _lib.ptr(m), n,
        float(params.stiffness), float(params.tau_d), float(params.eps_v), float(dt),
        _lib.ptr(e), _lib.ptr(g), _lib.ptr(H)))
    return e, g, H


def contact_energy(v_c, phi, gamma_lag, mu, params: ContactParams, dt: float) -> torch.Tensor:
    return _eval(v_c, phi, gamma_lag, mu, params, dt, "e")[0]


def contact_gradient(v_c, phi, gamma_lag, mu, params: ContactParams, dt: float) -> torch.Tensor:
    return _eval(v_c, phi, gamma_lag, mu, params, dt, "g")[1]


def contact_hessian(v_c, phi, gamma_lag, mu, params: ContactParams, dt: float) -> torch.Tensor:
    return _eval(v_c, phi, gamma_lag, mu, params, dt, "h")[2]


def contact_grad_hess(v_c, phi, gamma_lag, mu, params: ContactParams, dt: float):
    _, g, H = _eval(v_c, phi, gamma_lag, mu, params, dt, "gh")
    return g, H


def contact_impulses(v_c, phi, gamma_lag, mu, params: ContactParams, dt: float) -> torch.Tensor:
    return -contact_gradient(v_c, phi, gamma_lag, mu, params, dt)
