"""Synthetic scenes of the benchmark configurations as plain
JSON-able dicts, and the builder that turns one into a ``SimState``.

This is NOT the reference's YAML front-end (scene.py is out of scope); it is
the minimal scene vocabulary the tests, smoke() and bench.py share.  The dict
format is the one tests/golden/make_golden.py records.
"""

from __future__ import annotations

import copy

import numpy as np

from .bodies import GeomAttachment, RigidBody, Trajectory
from .contact_model import ContactParams
from .coupling import SimState, StepConfig
from .geometry import Box, Capsule, HalfSpace, Sphere
from .materials import Material
from .particles import concatenate
from .solver import SolverParams


def _shape(g):
    if g["shape"] == "halfspace":
        n = np.asarray(g["normal"], dtype=np.float64)
        return HalfSpace(normal=tuple(n / np.linalg.norm(n)), offset=float(g["offset"]))
    if g["shape"] == "sphere":
        return Sphere(radius=float(g["radius"]))
    if g["shape"] == "box":
        return Box(half_extents=tuple(float(a) for a in g["half_extents"]))
    return Capsule(radius=float(g["radius"]), half_length=float(g["half_length"]))


def build_bodies(scene) -> list:
    out = []
    for b in scene["bodies"]:
        geoms = [GeomAttachment(shape=_shape(g), position=np.asarray(g["position"], float),
                                quat=np.asarray(g["quat"], float), mu=float(g["mu"]))
                 for g in b["geoms"]]
        traj = None
        if b.get("trajectory"):
            t = b["trajectory"]
            quats = t.get("quats") or [[1.0, 0.0, 0.0, 0.0]] * len(t["times"])
            traj = Trajectory(times=np.asarray(t["times"]), positions=np.asarray(t["positions"]),
                              quats=np.asarray(quats))
        kw = {}
        if not b["kinematic"]:
            kw = dict(mass=float(b["mass"]), inertia_body=np.asarray(b["inertia"], float))
        body = RigidBody(name=b["name"], kinematic=bool(b["kinematic"]), geoms=geoms,
                         position=np.asarray(b["position"], float),
                         quat=np.asarray(b["quat"], float),
                         v=np.asarray(b.get("v", [0, 0, 0]), float),
                         omega=np.asarray(b.get("omega", [0, 0, 0]), float),
                         trajectory=traj, **kw)
        if body.kinematic and traj is not None:
            body.position, body.quat, body.v, body.omega = traj.sample(0.0)
        out.append(body)
    return out


def build_materials(scene) -> list:
    out = []
    for m in scene["materials"]:
        kw = {}
        if m.get("model") == "cloth":
            kw = dict(cloth_normal_stiffness=m.get("k_normal"),
                      cloth_shear_stiffness=m.get("gamma_shear"),
                      cloth_friction=m.get("cloth_friction", 0.3))
        out.append(Material(m["E"], m["nu"], m["rho"], model=m.get("model", "elastic"),
                            friction_angle=m.get("friction_angle", 30.0), **kw))
    return out


def cloth_arrays(scene) -> list:
    """Host arrays of the scene's cloth sheets (cloth.sheet_arrays), in scene
    order, each with its material id and initial velocity."""
    from .cloth import sheet_arrays
    out = []
    for c in scene.get("cloth", []):
        a = sheet_arrays(c["center"], c["size"], c["n_side"], c["thickness"],
                         scene["materials"][c["material"]]["rho"], c.get("normal_axis", 2))
        a["mid"] = np.full(a["x"].shape[0], c["material"], dtype=np.int64)
        a["v"] = np.tile(np.asarray(c.get("velocity", [0.0, 0.0, 0.0]), float),
                         (a["x"].shape[0], 1))
        out.append(a)
    return out


def build_particles(scene):
    """Particles of the scene's volumes followed by its cloth sheets; returns
    (ParticleSet, ClothMesh | None)."""
    from .cloth import ClothMesh
    from .particles import ParticleSet, seed_box_gpu
    mats = build_materials(scene)
    # seeded on the GPU, bit-identical to the reference's NumPy seeding
    sets = [seed_box_gpu(np.asarray(v["center"]), np.asarray(v["half"]), scene["h"],
                         mats[v["material"]], material_id=v["material"],
                         particles_per_cell=v["ppc"], jitter=v["jitter"],
                         velocity=tuple(v["velocity"]), seed=v["seed"])
            for v in scene["volumes"]]
    sheets = cloth_arrays(scene)
    for a in sheets:
        n = a["x"].shape[0]
        sets.append(ParticleSet(a["x"], a["v"], np.tile(np.eye(3), (n, 1, 1)),
                                np.zeros((n, 3, 3)), a["mass"], a["vol"], a["mid"]))
    particles = concatenate(sets)
    if not sheets:
        return particles, None
    n_total = particles.n
    first = particles.n - sum(a["x"].shape[0] for a in sheets)
    tri, ep, dmi, vol, d3 = [], [], [], [], []
    role = np.zeros(n_total, dtype=np.int8)
    for a in sheets:
        tri.append(a["tri"] + first)
        ep.append(a["epart"] + first)
        dmi.append(a["dm_inv"])
        vol.append(a["vol_e"])
        d3.append(a["d3"])
        role[first:first + a["x"].shape[0]] = a["role"]
        first += a["x"].shape[0]
    mesh = ClothMesh.from_arrays(np.concatenate(tri), np.concatenate(ep), np.concatenate(dmi),
                                 np.concatenate(vol), np.concatenate(d3), role)
    return particles, mesh


def build_state(scene, particles=None, cloth=None, precision: str = "f64") -> SimState:
    c = scene["contact"]
    s = scene["solver"]
    sp = SolverParams(eps_r=s.get("eps_r", 5e-2), max_iters=s.get("max_iters", 500))
    if particles is None:
        particles, cloth = build_particles(scene)
    return SimState(particles=particles, materials=build_materials(scene),
                    bodies=build_bodies(scene), h=scene["h"],
                    step=StepConfig(dt=scene["dt"], substeps=scene["substeps"],
                                    gravity=tuple(scene["gravity"])),
                    contact_params=ContactParams(stiffness=c["stiffness"], tau_d=c["tau_d"],
                                                 eps_v=c["eps_v"], margin=c.get("margin")),
                    solver_params=sp, cloth=cloth, precision=precision)


# ------------------------------------------------------------------ configs

def _floor(mu=0.5):
    return dict(name="floor", kinematic=True, position=[0, 0, 0], quat=[1, 0, 0, 0],
                geoms=[dict(shape="halfspace", normal=[0, 0, 1], offset=0.0, position=[0, 0, 0],
                            quat=[1, 0, 0, 0], mu=mu)])


def smoke_scene() -> dict:
    """~500 particles on a floor, pressed by a descending kinematic sphere."""
    return dict(h=0.01, dt=1e-3, substeps=2, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=1e-3, eps_v=1e-4, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=5e4, nu=0.3, rho=1000.0)],
                volumes=[dict(center=[0, 0, 0.0205], half=[0.02, 0.02, 0.02], material=0, ppc=8,
                              jitter=1.0, seed=0, velocity=[0, 0, -0.1])],
                bodies=[_floor(0.8),
                        dict(name="ball", kinematic=True, position=[0, 0, 0.07], quat=[1, 0, 0, 0],
                             trajectory=dict(times=[0.0, 1.0], positions=[[0, 0, 0.065],
                                                                          [0, 0, -0.235]]),
                             geoms=[dict(shape="sphere", radius=0.025, position=[0, 0, 0],
                                         quat=[1, 0, 0, 0], mu=0.5)])])


def elastic_cube_scene() -> dict:
    """C1: 8,000-particle elastic cube dropped on a kinematic ground box
    (the reference CPU scene, 100 rigid steps)."""
    dt = 1e-3
    return dict(h=0.01, dt=dt, substeps=10, gravity=[0, 0, -9.81], steps=100,
                contact=dict(stiffness=1e5, tau_d=dt, eps_v=1e-4, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=1e5, nu=0.3, rho=1000.0)],
                volumes=[dict(center=[0, 0, 0.06], half=[0.05, 0.05, 0.05], material=0, ppc=8,
                              jitter=1.0, seed=0, velocity=[0, 0, 0])],
                bodies=[dict(name="ground", kinematic=True, position=[0, 0, -0.05],
                             quat=[1, 0, 0, 0],
                             geoms=[dict(shape="box", half_extents=[0.3, 0.3, 0.05],
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.5)])])


# Friction regularisation of the sand workloads.  The survey's common
# setting is the dataclass default 1e-4 (contact_model.py:31); with it the
# solve of the first substep of every pusher-loaded step stops at
# max_iters = 500 (on the oracle as on the GPU: the pusher's pose jumps by
# v dt at each rigid step, coupling.py:1-8).  1e-3 (1 mm/s of regularised
# slip) is the value of the reference's own panel-grip experiment
# (experiments.py:32-69) and every solve converges
# (profiles/r02_convergence_study.txt).
SAND_EPS_V = 1e-3


def sand_pile_scene(half=(0.2, 0.2, 0.1), h=0.01, model="sand", eps_v=SAND_EPS_V,
                    gap=0.005) -> dict:
    """C2: Drucker–Prager sand block (256k particles at the default size) on a
    floor, pushed by a kinematic box starting ``gap`` clear at +0.2 m/s
    (DP parameters proposed there: 30 deg, c = 0, E = 3.5e5)."""
    dt = 2e-3
    hx, hy, hz = half
    push_half = (0.05, hy, 0.05)
    x0 = -hx - gap - push_half[0]
    z0 = push_half[2] + 0.005
    return dict(h=h, dt=dt, substeps=10, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=dt, eps_v=eps_v, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=3.5e5, nu=0.3, rho=1500.0, model=model, friction_angle=30.0)],
                volumes=[dict(center=[0, 0, hz + 0.002], half=list(half), material=0, ppc=8,
                              jitter=1.0, seed=0, velocity=[0, 0, 0])],
                bodies=[_floor(0.5),
                        dict(name="pusher", kinematic=True, position=[x0, 0, z0],
                             quat=[1, 0, 0, 0],
                             trajectory=dict(times=[0.0, 10.0],
                                             positions=[[x0, 0, z0], [x0 + 2.0, 0, z0]]),
                             geoms=[dict(shape="box", half_extents=list(push_half),
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.5)])])


def multi_material_scene(half=(0.25, 0.25, 0.125), h=0.005, substeps=20,
                         eps_v=SAND_EPS_V) -> dict:
    """C5: a block of two materials split at x = 0 (elastic on x < 0,
    Drucker-Prager sand on x > 0), 4.0M particles at the default size
    (100 x 100 x 50 cells x 8 ppc), on a floor and pushed from
    -x by a kinematic box starting 5 mm clear at +0.2 m/s.  N = 20 substeps
    keeps the sand's elastic wave CFL at h = 5 mm where C2 has it at 10 mm."""
    dt = 2e-3
    hx, hy, hz = half
    push_half = (0.05, hy, 0.05)
    x0 = -hx - 0.005 - push_half[0]
    z0 = push_half[2] + 0.005
    zc = hz + 0.002
    return dict(h=h, dt=dt, substeps=substeps, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=dt, eps_v=eps_v, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=1e5, nu=0.3, rho=1000.0, model="elastic"),
                           dict(E=3.5e5, nu=0.3, rho=1500.0, model="sand", friction_angle=30.0)],
                volumes=[dict(center=[-hx / 2, 0, zc], half=[hx / 2, hy, hz], material=0, ppc=8,
                              jitter=1.0, seed=0, velocity=[0, 0, 0]),
                         dict(center=[hx / 2, 0, zc], half=[hx / 2, hy, hz], material=1, ppc=8,
                              jitter=1.0, seed=1, velocity=[0, 0, 0])],
                bodies=[_floor(0.5),
                        dict(name="pusher", kinematic=True, position=[x0, 0, z0],
                             quat=[1, 0, 0, 0],
                             trajectory=dict(times=[0.0, 10.0],
                                             positions=[[x0, 0, z0], [x0 + 2.0, 0, z0]]),
                             geoms=[dict(shape="box", half_extents=list(push_half),
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.5)])])


def host_particles(scene: dict) -> dict:
    """Seed the scene's particle volumes on the HOST as NumPy arrays (the same
    jittered lattice as seed_box, particles.py:113-136): x, v, f, c, mass, vol,
    mid.  Used by bench.py (pinned host buffers, CPU baseline) and the
    multi-process tests; no device work."""
    from .particles import _jittered_lattice
    out = {k: [] for k in ("x", "v", "mass", "vol", "mid")}
    h = scene["h"]
    for v in scene["volumes"]:
        m = scene["materials"][v["material"]]
        c, half = np.asarray(v["center"], float), np.asarray(v["half"], float)
        rng = np.random.default_rng(v["seed"])
        lo = np.floor((c - half) / h).astype(np.int64)
        hi = np.ceil((c + half) / h).astype(np.int64)
        per_axis = max(1, round(v["ppc"] ** (1.0 / 3.0)))
        pts = _jittered_lattice(lo, hi, h, per_axis, v["jitter"], rng)
        pts = pts[np.all(np.abs(pts - c) <= half, axis=1)]
        n = pts.shape[0]
        vol = 8.0 * half.prod() / n
        out["x"].append(pts)
        out["v"].append(np.tile(np.asarray(v["velocity"], float), (n, 1)))
        out["mass"].append(np.full(n, m["rho"] * vol))
        out["vol"].append(np.full(n, vol))
        out["mid"].append(np.full(n, v["material"], dtype=np.int64))
    for a in cloth_arrays(scene):  # cloth sheets follow the volumes
        for k in ("x", "v", "mass", "vol", "mid"):
            out[k].append(a[k])
    out = {k: (val if val else [np.zeros((0, 3)) if k in ("x", "v") else np.zeros(0)])
           for k, val in out.items()}
    arr = {k: np.concatenate(val) for k, val in out.items()}
    arr["mid"] = arr["mid"].astype(np.int64)
    n = arr["x"].shape[0]
    arr["f"] = np.tile(np.eye(3), (n, 1, 1))
    arr["c"] = np.zeros((n, 3, 3))
    return arr


def cloth_sheet_scene(n_side: int = 183, h: float = 1.0 / 128) -> dict:
    """C3: a square cloth sheet (n_side^2 vertices + 2 (n_side-1)^2 face
    particles; 183 -> 99,737 particles) draped over a rigid sphere r = 0.25,
    E = 3.2e6, nu = 0.4, rho = 1.5e3, mu = 0.6, dt = 2 ms
    (SURVEY.md §8d).  Vertex spacing h/2, thickness 1 mm (proposed).  N = 16
    substeps: with E = 3.2e6 the membrane wave speed sqrt(E/rho) = 46 m/s and
    the explicit transfer needs dt_s < spacing / c (N = 4 diverges in the
    oracle as well)."""
    dt = 2e-3
    side = (n_side - 1) * 0.5 * h
    return dict(h=h, dt=dt, substeps=16, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=dt, eps_v=1e-4, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=3.2e6, nu=0.4, rho=1.5e3, model="cloth")],
                volumes=[],
                cloth=[dict(material=0, center=[0.0, 0.0, 0.3], size=[side, side],
                            n_side=n_side, thickness=1e-3)],
                bodies=[dict(name="sphere", kinematic=True, position=[0, 0, 0],
                             quat=[1, 0, 0, 0],
                             geoms=[dict(shape="sphere", radius=0.25, position=[0, 0, 0],
                                         quat=[1, 0, 0, 0], mu=0.6)])])


def tshirt_fold_scene(n_side: int = 64, h: float = 1.0 / 128) -> dict:
    """C4 (synthetic stand-in for the paper's T-shirt): a
    sheet with the paper's particle count (64^2 vertices + 7,938 faces =
    12,034 particles) on a table, its near edge gripped by two kinematic box
    grippers that lift it and fold it over (keyframe trajectories), E = 1e5,
    nu = 0.3, rho = 1e3, gripper friction 0.6, dt = 2 ms, N = 4."""
    dt = 2e-3
    side = (n_side - 1) * 0.5 * h
    half = 0.5 * side
    grip_half = [0.02, 0.02, 0.01]
    z0 = 0.004 + grip_half[2] + 0.002
    keys = [0.0, 0.3, 0.8, 1.3]

    def gripper(name, y):
        p0 = [-half + 0.01, y, z0]
        return dict(name=name, kinematic=True, position=p0, quat=[1, 0, 0, 0],
                    trajectory=dict(times=keys,
                                    positions=[p0, [-half + 0.01, y, z0 - 0.004],
                                               [0.0, y, 0.12], [half - 0.03, y, 0.03]]),
                    geoms=[dict(shape="box", half_extents=grip_half, position=[0, 0, 0],
                                quat=[1, 0, 0, 0], mu=0.6)])
    return dict(h=h, dt=dt, substeps=4, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=dt, eps_v=1e-4, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=1e5, nu=0.3, rho=1e3, model="cloth")],
                volumes=[],
                cloth=[dict(material=0, center=[0.0, 0.0, 0.004], size=[side, side],
                            n_side=n_side, thickness=1e-3)],
                bodies=[_floor(0.5), gripper("gripper_a", -0.5 * half),
                        gripper("gripper_b", 0.5 * half)])


def scaled(scene: dict, **kw) -> dict:
    s = copy.deepcopy(scene)
    s.update(kw)
    return s


# ------------------------------------------------------------------ interop

def from_reference_state(ref) -> SimState:
    """Build a device ``SimState`` from a reference ``mpmrb.coupling.SimState``
    (coupling.py:87-112), duck-typed: particle arrays (particles.py:12-64) are
    uploaded once, materials (materials.py:24-46), bodies (bodies.py:20-113),
    step, contact and solver parameters are carried over field by field.
    Rigid bodies are re-created from their public fields (the GPU path only
    reads poses, velocities and geoms)."""
    from .particles import ParticleSet
    rp = ref.particles
    particles = ParticleSet(np.asarray(rp.x), np.asarray(rp.v), np.asarray(rp.f),
                            np.asarray(rp.c), np.asarray(rp.mass), np.asarray(rp.volume0),
                            np.asarray(rp.material_id, dtype=np.int64))
    mats = [Material(m.youngs_modulus, m.poisson_ratio, m.density,
                     model=getattr(m, "model", "elastic"),
                     friction_angle=getattr(m, "friction_angle", 30.0)) for m in ref.materials]
    shapes = {"HalfSpace": lambda s: HalfSpace(normal=tuple(s.normal), offset=float(s.offset)),
              "Sphere": lambda s: Sphere(radius=float(s.radius)),
              "Box": lambda s: Box(half_extents=tuple(float(a) for a in s.half_extents)),
              "Capsule": lambda s: Capsule(radius=float(s.radius),
                                           half_length=float(s.half_length))}
    bodies = []
    for b in ref.bodies:
        geoms = [GeomAttachment(shape=shapes[type(g.shape).__name__](g.shape),
                                position=np.asarray(g.position, float),
                                quat=np.asarray(g.quat, float), mu=float(g.mu)) for g in b.geoms]
        traj = None
        if getattr(b, "trajectory", None) is not None:
            t = b.trajectory
            traj = Trajectory(times=np.asarray(t.times), positions=np.asarray(t.positions),
                              quats=np.asarray(t.quats))
        kw = {} if b.kinematic else dict(mass=float(b.mass),
                                         inertia_body=np.asarray(b.inertia_body, float))
        bodies.append(RigidBody(name=b.name, kinematic=bool(b.kinematic), geoms=geoms,
                                position=np.asarray(b.position, float),
                                quat=np.asarray(b.quat, float), v=np.asarray(b.v, float),
                                omega=np.asarray(b.omega, float), trajectory=traj, **kw))
    cp, sp = ref.contact_params, ref.solver_params
    st = SimState(particles=particles, materials=mats, bodies=bodies, h=float(ref.h),
                  step=StepConfig(dt=float(ref.step.dt), substeps=int(ref.step.substeps),
                                  gravity=tuple(float(a) for a in ref.step.gravity)),
                  contact_params=ContactParams(stiffness=cp.stiffness, tau_d=cp.tau_d,
                                               eps_v=cp.eps_v, margin=cp.margin),
                  solver_params=SolverParams(eps_a=sp.eps_a, eps_r=sp.eps_r,
                                             max_iters=sp.max_iters,
                                             ls_max_iters=sp.ls_max_iters, ls_tol=sp.ls_tol))
    st.time = float(getattr(ref, "time", 0.0))
    st.step_index = int(getattr(ref, "step_index", 0))
    return st
