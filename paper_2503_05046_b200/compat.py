"""NumPy façade over the GPU package, with the reference's module layout.

    from paper_2503_05046_b200 import compat
    compat.install()      # sys.modules["mpmrb"], ["mpmrb.transfer"], ... -> this façade
    import mpmrb          # code written against the reference's ndarray API

The reference (``mpmrb``, pure NumPy) hands NumPy arrays in and out of every
function; this package keeps state in HBM as torch tensors.  The façade maps
one onto the other without touching the computation:

* arguments: NumPy arrays pass straight through (the package uploads them);
  façade objects are unwrapped to the package's own objects;
* results: device tensors come back as NumPy arrays (``DevArray``, a host copy
  that writes the whole array back to its device tensor on item assignment,
  so ``particles.v[:] = 0`` works as on the reference's arrays); objects
  holding device state (ParticleSet, SparseGrid, Stencil, ContactSet,
  ContactProblem, SortPlan, SimState) come back as proxies whose array
  attributes read as fresh host copies and whose attribute assignment uploads.

Every computation still runs in this package's CUDA kernels; the façade adds
host<->device copies at the boundary (it is the compatibility path for code
and tests written against ``mpmrb``, not a fast path).  Names the package does
not implement (the reference's out-of-scope CLI, scene, experiments, outputs
modules) are absent.
"""

from __future__ import annotations

import sys
import types

import numpy as np
import torch

from . import (_lib, bodies, collision, contact_model, coupling, geometry, grid, materials, mpm,
               particles, rotations, solver, transfer)

MODULES = {
    "transfer": transfer, "grid": grid, "mpm": mpm, "particles": particles,
    "materials": materials, "collision": collision, "contact_model": contact_model,
    "solver": solver, "coupling": coupling, "geometry": geometry, "bodies": bodies,
    "rotations": rotations,
}

# classes whose instances hold device tensors
_DEVICE_CLASSES = (particles.ParticleSet, grid.SparseGrid, mpm.Stencil, collision.ContactSet,
                   solver.ContactProblem, transfer.SortPlan, coupling.SimState)


class DevArray(np.ndarray):
    """Host copy of a device tensor.  Item assignment on the array itself
    (not on views or results derived from it) writes it back to the tensor."""

    def __array_finalize__(self, obj):
        self._dev = None

    def __setitem__(self, idx, value):
        super().__setitem__(idx, value)
        dev = getattr(self, "_dev", None)
        if dev is not None:
            host = torch.from_numpy(np.ascontiguousarray(self.view(np.ndarray)))
            dev.copy_(host.to(device=dev.device, dtype=dev.dtype))


def _host(t: torch.Tensor) -> DevArray:
    a = t.detach().cpu().numpy().view(DevArray)
    a._dev = t
    return a


class Proxy:
    """A device-state object seen through NumPy."""

    __slots__ = ("_obj",)

    def __init__(self, obj):
        object.__setattr__(self, "_obj", obj)

    def __getattr__(self, name):
        v = getattr(self._obj, name)
        if callable(v) and not isinstance(v, (type, torch.Tensor)):
            return _wrap_fn(v)
        return to_np(v)

    def __setattr__(self, name, value):
        cur = getattr(self._obj, name, None)
        value = from_np(value)
        if isinstance(cur, torch.Tensor) and not isinstance(value, torch.Tensor) and value is not None:
            value = _lib.as_dev(np.asarray(value), cur.dtype)
        setattr(self._obj, name, value)

    def __repr__(self):
        return f"<mpmrb façade of {self._obj!r}>"


def to_np(v):
    if isinstance(v, torch.Tensor):
        return _host(v)
    if isinstance(v, Proxy):
        return v
    if isinstance(v, _DEVICE_CLASSES):
        return Proxy(v)
    if isinstance(v, list):
        out = [to_np(x) for x in v]
        # keep the caller's list (and its identity) when nothing needed converting
        return v if all(a is b for a, b in zip(out, v)) else out
    if isinstance(v, tuple) and not hasattr(v, "_fields"):
        return tuple(to_np(x) for x in v)
    if isinstance(v, dict):
        return {k: to_np(x) for k, x in v.items()}
    return v


def from_np(v):
    if isinstance(v, Proxy):
        return v._obj
    if isinstance(v, DevArray):
        return np.asarray(v.view(np.ndarray))
    if isinstance(v, list):
        out = [from_np(x) for x in v]
        return v if all(a is b for a, b in zip(out, v)) else out
    if isinstance(v, tuple) and not hasattr(v, "_fields"):
        return tuple(from_np(x) for x in v)
    if isinstance(v, dict):
        return {k: from_np(x) for k, x in v.items()}
    return v


def _wrap_fn(f):
    def call(*args, **kwargs):
        return to_np(f(*from_np(args), **from_np(kwargs)))

    call.__name__ = getattr(f, "__name__", "call")
    call.__doc__ = getattr(f, "__doc__", None)
    call.__wrapped__ = f
    return call


class _ClassFacade:
    """Constructor and class attributes of a device-state class."""

    def __init__(self, cls):
        self._cls = cls
        self.__name__ = cls.__name__
        self.__doc__ = cls.__doc__

    def __call__(self, *args, **kwargs):
        return to_np(self._cls(*from_np(args), **from_np(kwargs)))

    def __getattr__(self, name):
        v = getattr(self._cls, name)
        return _wrap_fn(v) if callable(v) and not isinstance(v, type) else to_np(v)

    def __instancecheck__(self, obj):
        return isinstance(from_np(obj), self._cls)


def _method_facade(cls):
    """A subclass of a plain (parameter) class whose own public methods take
    and return NumPy (e.g. the shapes' query); instances still pass the
    package's isinstance checks."""
    own = {k: v for k, v in vars(cls).items()
           if not k.startswith("_") and callable(v) and not isinstance(v, (type, staticmethod,
                                                                          classmethod))}
    if not own:
        return cls
    ns = {k: _wrap_fn(v) for k, v in own.items()}
    ns["__doc__"] = cls.__doc__
    ns["__module__"] = cls.__module__
    return type(cls.__name__, (cls,), ns)


_FACADE_CLASSES: dict = {}


def _facade(name: str, mod) -> types.ModuleType:
    fm = types.ModuleType(f"mpmrb.{name}", mod.__doc__)
    for attr, v in vars(mod).items():
        if attr.startswith("__") or isinstance(v, types.ModuleType):
            continue
        if isinstance(v, type) and issubclass(v, _DEVICE_CLASSES):
            fv = _ClassFacade(v)
        elif isinstance(v, type) and not issubclass(v, BaseException):
            if v not in _FACADE_CLASSES:
                _FACADE_CLASSES[v] = _method_facade(v)
            fv = _FACADE_CLASSES[v]
        elif isinstance(v, type) or not callable(v):
            fv = v  # exceptions, constants
        else:
            fv = _wrap_fn(v)
        setattr(fm, attr, fv)
    return fm


def _advance_step_by_mode(state, *args, **kwargs):
    """The reference's advance_step honours ``state.mode`` (coupling.py:168-
    219 with transfer.py:9-14): "deterministic", its default, sums every
    scatter in particle-id order, so results are bitwise reproducible and
    independent of the sort plan (test_coupling.py::
    test_substep_equivalence_bitwise).  That is the operator pipeline with the
    ordered P2G fold (coupling.advance_step_ops); "fast" is the fused substep
    graph (coupling.advance_step), whose P2G tiles flush with float64 atomics."""
    if getattr(state, "mode", "deterministic") == "deterministic" and not args and not kwargs:
        return coupling.advance_step_ops(state)
    return coupling.advance_step(state, *args, **kwargs)


def install(alias: str = "mpmrb") -> types.ModuleType:
    """Register the façade as ``alias`` (and ``alias.<module>``) in sys.modules."""
    root = types.ModuleType(alias, __doc__)
    root.__path__ = []  # a package, so "from mpmrb.x import y" resolves
    for name, mod in MODULES.items():
        fm = _facade(name, mod)
        if name == "coupling":
            fm.advance_step = _wrap_fn(_advance_step_by_mode)
        fm.__name__ = f"{alias}.{name}"
        sys.modules[f"{alias}.{name}"] = fm
        setattr(root, name, fm)
        for attr in dir(fm):
            if not attr.startswith("_") and not hasattr(root, attr):
                setattr(root, attr, getattr(fm, attr))
    sys.modules[alias] = root
    return root
