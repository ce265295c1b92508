"""Particle-vs-rigid-geometry contact detection on the GPU.

``detect_contacts`` (collision.py:88-132): one count kernel, a device scan and
one emit kernel produce the contact SoA already in (particle, body, geom)
order.  ``BiasCache`` (collision.py:55-85) keeps the first-sight bias per
(body, geom, particle) as stamped device slots; ``clear()`` bumps the stamp,
so clearing is O(1).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bodies import geom_structs


@dataclass
class ContactSet:
    """SoA contact data ordered by (particle, body, geom); CUDA tensors."""

    particle: torch.Tensor
    body: torch.Tensor
    geom: torch.Tensor
    phi: torch.Tensor
    normal: torch.Tensor
    witness: torch.Tensor
    frames: torch.Tensor
    bias: torch.Tensor
    mu: torch.Tensor
    gamma_lag: torch.Tensor = field(default=None)

    def __post_init__(self):
        if self.gamma_lag is None:
            self.gamma_lag = torch.zeros_like(self.phi)

    @property
    def n(self) -> int:
        return int(self.phi.shape[0])

    @classmethod
    def empty(cls) -> "ContactSet":
        z = _lib.zeros((0,))
        zi = torch.zeros(0, dtype=torch.int64, device=z.device)
        return cls(zi, zi.clone(), zi.clone(), z, _lib.zeros((0, 3)), _lib.zeros((0, 3)),
                   _lib.zeros((0, 3, 3)), _lib.zeros((0, 3)), z.clone())


class BiasCache:
    """Per-step memo of contact-frame bias vectors keyed by (body, geom, particle)."""

    def __init__(self):
        self._stamp = None
        self._store = None
        self._shape = (0, 0)
        self._epoch = 1

    def clear(self):
        self._epoch += 1

    def _slots(self, n_geoms: int, n: int):
        """(geom, particle) slots for this call's geoms and particle count.
        A change of either re-lays the slots, carrying every cached entry
        whose (geom, particle) index still exists: the reference keys the
        cache by particle id (collision.py:55-85), so a particle keeps its
        first-sight bias when others join or leave the set."""
        if self._stamp is None or self._shape != (n_geoms, n):
            stamp = torch.zeros(max(1, n_geoms * n), dtype=torch.int32, device=_lib.device())
            store = _lib.zeros((max(1, n_geoms * n), 3))
            og, on = self._shape
            if self._stamp is not None and og * on > 0 and n_geoms * n > 0:
                kg, kn = min(og, n_geoms), min(on, n)
                stamp[: n_geoms * n].view(n_geoms, n)[:kg, :kn] = \
                    self._stamp[: og * on].view(og, on)[:kg, :kn]
                store[: n_geoms * n].view(n_geoms, n, 3)[:kg, :kn] = \
                    self._store[: og * on].view(og, on, 3)[:kg, :kn]
            self._stamp, self._store = stamp, store
            self._shape = (n_geoms, n)
        return self._stamp, self._store


def detect_contacts(particles, bodies, margin: float,
                    bias_cache: BiasCache | None = None) -> ContactSet:
    """Contacts with phi < margin, ordered by (particle, body, geom)."""
    if particles.n == 0 or not bodies:
        return ContactSet.empty()
    gs = geom_structs(bodies)
    ng = len(gs)
    garr = (_lib.Geom * ng)(*gs)
    n = particles.n
    cap = n * ng
    dev = particles.x.device
    out = dict(particle=torch.empty(cap, dtype=torch.int64, device=dev),
               body=torch.empty(cap, dtype=torch.int64, device=dev),
               geom=torch.empty(cap, dtype=torch.int64, device=dev),
               phi=_lib.empty((cap,)), normal=_lib.empty((cap, 3)), witness=_lib.empty((cap, 3)),
               frames=_lib.empty((cap, 3, 3)), bias=_lib.empty((cap, 3)), mu=_lib.empty((cap,)))
    if bias_cache is not None:
        stamp, store = bias_cache._slots(ng, n)
        epoch = bias_cache._epoch
    else:
        stamp = store = None
        epoch = 0
    nc = C.c_int64()
    _lib.check(_lib.lib().mpmrb_detect_contacts(
        _lib.ctx(), _lib.ptr(particles.x), n, garr, ng, float(margin), _lib.ptr(stamp),
        _lib.ptr(store), epoch, cap, *[_lib.ptr(out[k]) for k in (
            "particle", "body", "geom", "phi", "normal", "witness", "frames", "bias", "mu")],
        C.byref(nc)))
    k = int(nc.value)
    return ContactSet(**{key: val[:k] for key, val in out.items()})


def contact_velocities(contacts: ContactSet, stencil, v_grid) -> torch.Tensor:
    """v_c = R (sum_i w_i v_i) + b (collision.py:135-143)."""
    if contacts.n == 0:
        return _lib.zeros((0, 3))
    nodes = stencil.nodes[contacts.particle].contiguous()
    w = stencil.weights[contacts.particle].contiguous()
    return _contact_velocities_raw(nodes, w, contacts.frames, contacts.bias, v_grid)


def _contact_velocities_raw(nodes, w, frames, bias, v_grid) -> torch.Tensor:
    nc = nodes.shape[0]
    vg = _lib.as_dev(v_grid).contiguous()
    out = _lib.empty((nc, 3))
    _lib.check(_lib.lib().mpmrb_contact_velocities(
        _lib.ctx(), _lib.ptr(nodes.contiguous()), _lib.ptr(w.contiguous()),
        _lib.ptr(frames.contiguous()), _lib.ptr(bias.contiguous()), nc, _lib.ptr(vg),
        _lib.ptr(out)))
    return out
