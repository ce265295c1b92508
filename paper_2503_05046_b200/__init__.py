"""B200-native (sm_100a) hot path of the convex MPM–rigid-body coupling of
arXiv 2503.05046, as a drop-in for the reference package ``mpmrb``.

The public names mirror the reference's ``mpmrb/__init__.py:5-27``.  Particle,
grid and contact state live in HBM as float64 PyTorch tensors; every hot-path
operation runs in hand-written CUDA kernels in ``_native/libmpmrb_b200.so``
(C ABI: ``include/mpmrb_b200.h``).  There is no CPU fallback: without the
library or a CUDA device the operators raise ``NativeUnavailable``.

Out of scope (host-side, not on the hot path): scene YAML, run driver, frame
output and CLI.
"""

__version__ = "0.1.0"

from ._lib import NativeUnavailable  # noqa: F401
from .bodies import GeomAttachment, RigidBody, Trajectory, compose_geoms  # noqa: F401
from .collision import BiasCache, ContactSet, contact_velocities, detect_contacts  # noqa: F401
from .contact_model import ContactParams  # noqa: F401
from .coupling import (SimState, SimulationDiverged, StepConfig, StepSummary,  # noqa: F401
                       advance_step, advance_step_ops)
from .geometry import Box, Capsule, HalfSpace, Sphere, contact_frames  # noqa: F401
from .geometry import query_signed_distance  # noqa: F401
from .grid import AllocationError, SparseGrid  # noqa: F401
from .materials import Material  # noqa: F401
from .mpm import build_stencil, grid_to_particle, grid_update, particle_to_grid  # noqa: F401
from .particles import ParticleSet, concatenate, seed_box, seed_sphere  # noqa: F401
from .solver import (ContactProblem, SolverParams, SolveReport,  # noqa: F401
                     build_contact_problem, quasi_newton_solve)
from .transfer import (PlanEpochError, SortPlan, build_sort_plan,  # noqa: F401
                       plan_staleness, scatter_reduce)

__all__ = [
    "__version__",
    "AllocationError", "BiasCache", "Box", "Capsule", "ContactParams", "ContactProblem",
    "ContactSet", "GeomAttachment", "HalfSpace", "Material", "NativeUnavailable",
    "ParticleSet", "PlanEpochError", "RigidBody", "SimState", "SimulationDiverged",
    "SolveReport", "SolverParams", "SortPlan", "SparseGrid", "Sphere", "StepConfig",
    "StepSummary", "Trajectory", "advance_step", "advance_step_ops", "build_contact_problem",
    "build_sort_plan", "build_stencil", "compose_geoms", "concatenate", "contact_frames",
    "contact_velocities", "detect_contacts", "grid_to_particle", "grid_update",
    "particle_to_grid", "plan_staleness", "quasi_newton_solve", "query_signed_distance",
    "scatter_reduce", "seed_box", "seed_sphere",
]
