"""ctypes binding of libmpmrb_b200.so (include/mpmrb_b200.h).

The product path has NO CPU fallback: if the library or a CUDA device is
missing, every call raises ``NativeUnavailable``.  Device memory is owned by
PyTorch tensors; the library receives raw pointers plus the current CUDA
stream.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np
import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_native" / "libmpmrb_b200.so"

OK = 0
E_ALLOCATION = 1
E_PLAN_EPOCH = 2
E_INVALID = 3
E_NOT_DESCENT = 4
E_NONFINITE = 5
E_DIVERGED = 6
E_CUDA = 7
E_CAPACITY = 8

MAT_ELASTIC = 0
MAT_SAND = 1
MAT_CLOTH = 2
CLOTH_NONE, CLOTH_VERTEX, CLOTH_ELEMENT = 0, 1, 2
PREC_F64, PREC_F32 = 0, 1
GEOM_HALFSPACE, GEOM_SPHERE, GEOM_BOX, GEOM_CAPSULE = 0, 1, 2, 3


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is missing; there is no CPU fallback."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ----------------------------------------------------------------- structs

class Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("mu", C.c_double),
                ("lam", C.c_double), ("dp_alpha", C.c_double), ("k_normal", C.c_double),
                ("gamma_shear", C.c_double), ("friction", C.c_double)]


class Geom(C.Structure):
    _fields_ = [("kind", C.c_int32), ("body", C.c_int32), ("geom", C.c_int32),
                ("pad_", C.c_int32), ("rot", C.c_double * 9), ("pos", C.c_double * 3),
                ("params", C.c_double * 4), ("mu", C.c_double), ("body_pos", C.c_double * 3),
                ("body_v", C.c_double * 3), ("body_omega", C.c_double * 3)]


class Particles(C.Structure):
    _fields_ = [("x", C.c_void_p), ("v", C.c_void_p), ("f", C.c_void_p), ("c", C.c_void_p),
                ("mass", C.c_void_p), ("volume0", C.c_void_p), ("material_id", C.c_void_p),
                ("plastic", C.c_void_p), ("n", C.c_int64)]


class GridView(C.Structure):
    _fields_ = [("block_keys", C.c_void_p), ("hash_keys", C.c_void_p),
                ("hash_vals", C.c_void_p), ("n_blocks", C.c_int64), ("hash_cap", C.c_int64),
                ("h", C.c_double)]


class Problem(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_contacts", C.c_int64), ("m", C.c_void_p),
                ("v_star", C.c_void_p), ("v_init", C.c_void_p), ("nodes", C.c_void_p),
                ("w", C.c_void_p), ("frames", C.c_void_p), ("bias", C.c_void_p),
                ("phi", C.c_void_p), ("mu", C.c_void_p), ("gamma_lag", C.c_void_p),
                ("stiffness", C.c_double), ("tau_d", C.c_double), ("eps_v", C.c_double),
                ("dt", C.c_double)]


class SolverParamsC(C.Structure):
    _fields_ = [("eps_a", C.c_double), ("eps_r", C.c_double), ("max_iters", C.c_int32),
                ("ls_max_iters", C.c_int32), ("ls_tol", C.c_double)]


class SolveReportC(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("ls_evals", C.c_int32),
                ("regularized", C.c_int32), ("status", C.c_int32), ("pad_", C.c_int32)]


class StepStats(C.Structure):
    _fields_ = [("substeps", C.c_int32), ("all_converged", C.c_int32),
                ("iterations_max", C.c_int32), ("n_contacts_max", C.c_int32),
                ("iterations_mean", C.c_double), ("n_contacts_mean", C.c_double),
                ("n_active_mean", C.c_double), ("clamped", C.c_int64), ("ls_evals", C.c_int64),
                ("regularized", C.c_int64), ("status", C.c_int32), ("status_detail", C.c_int32),
                ("status_aux", C.c_int64), ("substeps_unconverged", C.c_int32),
                ("reserved", C.c_int32), ("iterations_total", C.c_int64),
                ("iterations_unconverged", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
class SimViews(C.Structure):
    """mpmrb_sim_views (include/mpmrb_b200.h): the fused substep's internal
    grid and contact arrays, for slab.py's fused mode."""
    _fields_ = [("n_blocks", C.c_int64), ("n_active", C.c_int64), ("n_contacts", C.c_int64),
                ("nc_cap", C.c_int64)] + [(k, C.c_void_p) for k in (
                    "block_keys", "mass", "mom_apic", "mom_force", "v_star", "v_k", "v_next",
                    "act", "m_act", "v_star_act", "v_k_act", "cnodes", "cw", "frames", "bias",
                    "phi", "mu", "gamma_lag", "gamma")]


_SIGS = {
    "mpmrb_abi_version": ([], C.c_int),
    "mpmrb_last_error": ([], C.c_char_p),
    "mpmrb_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "mpmrb_destroy": ([_P], C.c_int),
    "mpmrb_set_stream": ([_P, _P], C.c_int),
    "mpmrb_sync": ([_P], C.c_int),
    "mpmrb_launch_count": ([_P], C.c_int64),
    "mpmrb_sort_plan": ([_P, _P, _I64, _D, _P, _P, _P, _P, _P, _P, C.POINTER(_I64)], C.c_int),
    "mpmrb_plan_staleness": ([_P, _P, _P, _I64, _D, C.POINTER(_D)], C.c_int),
    "mpmrb_base_cells": ([_P, _P, _I64, _D, _P], C.c_int),
    "mpmrb_grid_allocate": ([_P, _P, _I64, _D, _P, _I64, _P, _P, _I64, C.POINTER(_I64)], C.c_int),
    "mpmrb_node_ids": ([_P, C.POINTER(GridView), _P, _I64, _P], C.c_int),
    "mpmrb_build_stencil": ([_P, C.POINTER(GridView), _P, _I64, _P, _P, _P], C.c_int),
    "mpmrb_seed_box": ([_P, C.POINTER(_I64), C.POINTER(_I64), C.c_int32, _D, _D, C.POINTER(_D),
                        C.POINTER(_D), C.POINTER(C.c_uint64), _P, _I64, C.POINTER(_I64)], C.c_int),
    "mpmrb_scatter_reduce": ([_P, _P, _P, _I64, _I64, _I64, _I64, _P], C.c_int),
    "mpmrb_scatter_reduce_ordered": ([_P, _P, _P, _I64, _I64, _I64, _I64, _P], C.c_int),
    "mpmrb_compute_stresses": ([_P, _P, _P, _I64, C.POINTER(Material), C.c_int32, _P], C.c_int),
    "mpmrb_p2g": ([_P, C.POINTER(GridView), C.POINTER(Particles), C.POINTER(Material), C.c_int32,
                   _D, _P, _P, _P], C.c_int),
    "mpmrb_p2g_ordered": ([_P, C.POINTER(GridView), C.POINTER(Particles), C.POINTER(Material),
                           C.c_int32, _D, _P, _P, _P], C.c_int),
    "mpmrb_grid_update": ([_P, _I64, _P, _P, _P, C.POINTER(_D), _D, _P, _P, _P], C.c_int),
    "mpmrb_g2p": ([_P, C.POINTER(GridView), C.POINTER(Particles), C.POINTER(Material), C.c_int32,
                   _P, _D, C.POINTER(_I64)], C.c_int),
    "mpmrb_clamp_degenerate": ([_P, _P, _I64, _P, C.POINTER(_I64)], C.c_int),
    "mpmrb_contact_model": ([_P, _P, _P, _P, _P, _I64, _D, _D, _D, _D, _P, _P, _P], C.c_int),
    "mpmrb_sdf_query": ([_P, C.POINTER(Geom), _P, _I64, _P, _P, _P], C.c_int),
    "mpmrb_contact_frames": ([_P, _P, _I64, _P], C.c_int),
    "mpmrb_detect_contacts": ([_P, _P, _I64, C.POINTER(Geom), C.c_int32, _D, _P, _P, C.c_int32,
                               _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(_I64)],
                              C.c_int),
    "mpmrb_contact_velocities": ([_P, _P, _P, _P, _P, _I64, _P, _P], C.c_int),
    "mpmrb_qn_solve": ([_P, C.POINTER(Problem), C.POINTER(SolverParamsC), _P, _P, _P, _P, _P, _P,
                        _P, C.POINTER(SolveReportC)], C.c_int),
    "mpmrb_qn_solve_ext": ([_P, C.POINTER(Problem), C.POINTER(SolverParamsC), _P,
                            C.POINTER(C.c_double), _P, _P, _P, _P, _P, _P,
                            C.POINTER(C.c_double), C.POINTER(SolveReportC)], C.c_int),
    "mpmrb_solver_profile": ([_P, C.POINTER(C.c_uint64), C.c_int32], C.c_int),
    "mpmrb_solver_profile_cta": ([_P, C.POINTER(C.c_uint64)], C.c_int),
    "mpmrb_sim_create":([_P, C.POINTER(C.c_void_p)], C.c_int),
    "mpmrb_sim_destroy": ([_P], C.c_int),
    "mpmrb_sim_set_particles": ([_P, C.POINTER(Particles)], C.c_int),
    "mpmrb_sim_set_materials": ([_P, C.POINTER(Material), C.c_int32], C.c_int),
    "mpmrb_sim_set_geoms": ([_P, C.POINTER(Geom), C.c_int32, C.c_int32], C.c_int),
    "mpmrb_sim_set_params": ([_P, _D, _D, C.POINTER(_D), _D, _D, _D, _D,
                              C.POINTER(SolverParamsC)], C.c_int),
    "mpmrb_sim_set_cloth": ([_P, _I64, _P, _P, _P, _P, _P, _P], C.c_int),
    "mpmrb_sim_set_precision": ([_P, C.c_int32], C.c_int),
    "mpmrb_search_direction": ([_P, _P, _P, _I64, _P, C.POINTER(C.c_int32)], C.c_int),
    "mpmrb_polar_rotation": ([_P, _P, _I64, _P], C.c_int),
    "mpmrb_scan_exclusive_i32": ([_P, _P, _I64, _P, _P], C.c_int),
    "mpmrb_inverse_transpose3": ([_P, _P, _I64, _P], C.c_int),
    "mpmrb_sim_begin_step": ([_P, _I64, C.c_int32], C.c_int),
    "mpmrb_sim_substep": ([_P], C.c_int),
    "mpmrb_sim_end_step": ([_P, C.POINTER(StepStats), C.POINTER(_D)], C.c_int),
    "mpmrb_sim_staleness": ([_P], C.c_double),
    "mpmrb_sim_profile_substep": ([_P, C.POINTER(C.c_float), C.POINTER(C.c_int32)], C.c_int),
    "mpmrb_sim_last_grid":([_P, C.POINTER(_I64), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                             C.POINTER(_P)], C.c_int),
    "mpmrb_sim_last_contacts": ([_P, C.POINTER(_I64), C.POINTER(_P), C.POINTER(_P)], C.c_int),
    "mpmrb_sim_substep_part": ([_P, C.c_int32], C.c_int),
    "mpmrb_sim_get_views": ([_P, C.POINTER(SimViews)], C.c_int),
    "mpmrb_sim_set_solve_result": ([_P, C.POINTER(SolveReportC)], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()
_ctx = {}


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (but do not require a GPU for) the C-ABI library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # MPMRB_LIB_PATH: an alternative build of the same library (A/B
        # experiments, tools/build_variant.sh)
        p = Path(path) if path else Path(os.environ.get("MPMRB_LIB_PATH", LIB_PATH))
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing; build it with `python -m paper_2503_05046_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def lib() -> C.CDLL:
    return load_library()


def _exc_for(code: int, msg: str) -> Exception:
    from .grid import AllocationError
    from .transfer import PlanEpochError
    if code == E_ALLOCATION:
        return AllocationError(msg)
    if code == E_PLAN_EPOCH:
        return PlanEpochError(msg)
    if code in (E_INVALID, E_NOT_DESCENT):
        return ValueError(msg)
    if code == E_NONFINITE:
        return FloatingPointError(msg)
    if code == E_DIVERGED:
        from .coupling import SimulationDiverged
        return SimulationDiverged(msg)
    return NativeError(code, msg)


def check(code: int) -> None:
    if code != OK:
        msg = lib().mpmrb_last_error().decode(errors="replace")
        raise _exc_for(code, msg)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def ctx() -> C.c_void_p:
    """Per-device library context bound to the current torch stream."""
    dev = device()
    L = lib()
    key = dev.index
    h = _ctx.get(key)
    if h is None:
        out = C.c_void_p()
        check(L.mpmrb_create(key, C.byref(out)))
        h = out
        _ctx[key] = h
    check(L.mpmrb_set_stream(h, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return h


_own_ctx: list = []  # contexts owned by simulation states (coupling.SimState)


def new_ctx() -> C.c_void_p:
    """A library context of its own (stream, scratch, status), for a
    simulation state that may step concurrently with others on the device."""
    out = C.c_void_p()
    check(lib().mpmrb_create(device().index, C.byref(out)))
    with _lock:
        _own_ctx.append(out.value)
    return out


def free_ctx(h) -> None:
    with _lock:
        if h.value in _own_ctx:
            _own_ctx.remove(h.value)
    lib().mpmrb_destroy(h)


def bind_stream(h, stream: torch.cuda.Stream) -> None:
    check(lib().mpmrb_set_stream(h, C.c_void_p(stream.cuda_stream)))


def launch_count() -> int:
    """Kernels launched so far by every context on this device."""
    dev = device()
    h = _ctx.get(dev.index)
    n = int(lib().mpmrb_launch_count(h)) if h is not None else 0
    with _lock:
        own = list(_own_ctx)
    return n + sum(int(lib().mpmrb_launch_count(C.c_void_p(v))) for v in own)


# ----------------------------------------------------------------- tensors

def ptr(t: torch.Tensor | None) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    if not t.is_cuda:
        raise NativeUnavailable("tensor is not on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def as_dev(a, dtype=torch.float64, shape=None) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor of dtype (no copy if already there)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=dtype)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(a)), dtype=dtype, device=dev)
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def to_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def empty(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())
