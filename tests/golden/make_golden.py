"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``mpmrb`` from /root/reference/pkg/src (and the
reference test helpers from /root/reference/pkg/tests), evaluates the hot-path
functions on seeded inputs, and writes compressed ``.npz`` fixtures next to this
script.  The fixtures are committed; nothing at test time reads
/root/reference.  Scene descriptions are stored as JSON so tests can rebuild
the same scenes for the oracle and for the CUDA path.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    import mpmrb  # noqa: F401
    return mpmrb


def save(name: str, **arrays):
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"wrote {path.name}: {path.stat().st_size / 1024:.1f} KiB")


def random_particle_arrays(rng, n, lo, hi, v_scale=1.0):
    x = rng.uniform(lo, hi, size=(n, 3))
    v = rng.normal(0.0, v_scale, size=(n, 3))
    f = np.broadcast_to(np.eye(3), (n, 3, 3)).copy() + 0.05 * rng.normal(size=(n, 3, 3))
    c = 0.1 * rng.normal(size=(n, 3, 3))
    vol = np.full(n, (0.5 * 0.05) ** 3)
    return x, v, f, c, 1000.0 * vol, vol


def gen_binning():
    from mpmrb.grid import SparseGrid, base_cells
    from mpmrb.mpm import build_stencil
    from mpmrb.transfer import build_sort_plan, morton_keys, plan_staleness
    out = {}
    cases = [("uniform", 0.05, (0.0, 1.0), 700, 1),
             ("negative", 0.013, (-0.37, 0.21), 900, 2),
             ("dense", 0.01, (0.0, 0.08), 1500, 3)]
    for tag, h, (lo, hi), n, seed in cases:
        rng = np.random.default_rng(seed)
        x = rng.uniform(lo, hi, size=(n, 3))
        plan = build_sort_plan(x, h, epoch=5)
        grid = SparseGrid.allocate(x, h)
        st = build_stencil(x, grid)
        moved = x + rng.normal(0.0, 0.3 * h, size=x.shape)
        out.update({
            f"{tag}_x": x, f"{tag}_h": np.float64(h),
            f"{tag}_cells": base_cells(x, h),
            f"{tag}_keys": morton_keys(base_cells(x, h)),
            f"{tag}_perm": plan.perm, f"{tag}_inv_perm": plan.inv_perm,
            f"{tag}_bin_keys": plan.bin_keys, f"{tag}_bin_starts": plan.bin_starts,
            f"{tag}_bin_of": plan.bin_of,
            f"{tag}_block_keys": grid.block_keys, f"{tag}_block_coords": grid.block_coords,
            f"{tag}_weights": st.weights, f"{tag}_nodes": st.nodes, f"{tag}_dpos": st.dpos,
            f"{tag}_moved": moved, f"{tag}_staleness": np.float64(plan_staleness(plan, moved, h)),
        })
    save("binning", **out)


def gen_p2g_g2p():
    from mpmrb.grid import SparseGrid
    from mpmrb.materials import Material, clamp_degenerate
    from mpmrb.mpm import (build_stencil, compute_stresses, grid_to_particle, grid_update,
                           particle_to_grid)
    from mpmrb.particles import ParticleSet
    from mpmrb.transfer import build_sort_plan
    mats = [Material(1e5, 0.4, 1000.0), Material(2e5, 0.3, 500.0)]
    out = {}
    for tag, n, h, dt, seed in [("a", 400, 0.08, 1e-4, 11), ("b", 1200, 0.03, 5e-4, 12)]:
        rng = np.random.default_rng(seed)
        x, v, f, c, m, vol = random_particle_arrays(rng, n, (0, 0, 0), (0.4, 0.4, 0.4))
        mid = (rng.uniform(size=n) < 0.5).astype(np.int64)
        p = ParticleSet(x=x.copy(), v=v.copy(), f=f.copy(), c=c.copy(), mass=m, volume0=vol,
                        material_id=mid)
        grid = SparseGrid.allocate(p.x, h)
        st = build_stencil(p.x, grid)
        plan = build_sort_plan(p.x, h, 0)
        tau = compute_stresses(p, mats)
        particle_to_grid(p, grid, st, mats, dt, plan, 0)
        g = np.array([0.0, 0.0, -9.81])
        grid_update(grid, g, dt)
        v_next = grid.v_star + rng.normal(0.0, 0.01, size=grid.v_star.shape)
        v_next[~grid.active] = 0.0
        grid.v_next = v_next
        nclamp = grid_to_particle(p, grid, st, dt)
        out.update({
            f"{tag}_x": x, f"{tag}_v": v, f"{tag}_f": f, f"{tag}_c": c, f"{tag}_mass": m,
            f"{tag}_vol": vol, f"{tag}_mid": mid, f"{tag}_h": np.float64(h),
            f"{tag}_dt": np.float64(dt), f"{tag}_tau": tau,
            f"{tag}_block_keys": grid.block_keys,
            f"{tag}_gmass": grid.mass, f"{tag}_mom_apic": grid.mom_apic,
            f"{tag}_mom_force": grid.mom_force, f"{tag}_active": grid.active,
            f"{tag}_v_k": grid.v_k, f"{tag}_v_star": grid.v_star, f"{tag}_v_next": v_next,
            f"{tag}_x1": p.x, f"{tag}_v1": p.v, f"{tag}_c1": p.c, f"{tag}_f1": p.f,
            f"{tag}_nclamp": np.int64(nclamp),
        })
    out["mat_E"] = np.array([m.youngs_modulus for m in mats])
    out["mat_nu"] = np.array([m.poisson_ratio for m in mats])
    out["mat_rho"] = np.array([m.density for m in mats])
    # clamp cases: healthy, inverted, non-finite, strongly compressed, random
    rng = np.random.default_rng(5)
    fs = [np.eye(3), np.diag([1.0, 1.0, -0.5]), np.array([[np.nan, 0, 0], [0, 1, 0], [0, 0, 1]]),
          np.diag([0.01, 0.5, 2.0])]
    rnd = rng.normal(size=(40, 3, 3))
    fs = np.concatenate([np.stack(fs), rnd])
    fixed, k = clamp_degenerate(fs)
    out["clamp_in"] = fs
    out["clamp_out"] = fixed
    out["clamp_n"] = np.int64(k)
    save("p2g_g2p", **out)


def gen_sdf_contacts():
    from mpmrb.bodies import GeomAttachment, RigidBody
    from mpmrb.collision import BiasCache, detect_contacts
    from mpmrb.geometry import Box, Capsule, HalfSpace, Sphere, contact_frames
    from mpmrb.particles import ParticleSet
    from mpmrb.rotations import quat_from_axis_angle
    rng = np.random.default_rng(21)
    out = {}
    shapes = {"halfspace": HalfSpace(normal=(0.0, 0.6, 0.8), offset=0.05),
              "sphere": Sphere(radius=0.3), "box": Box(half_extents=(0.15, 0.1, 0.25)),
              "capsule": Capsule(radius=0.05, half_length=0.2)}
    for name, sh in shapes.items():
        pts = rng.uniform(-0.45, 0.45, size=(400, 3))
        pts[:3] = 0.0  # degenerate centre cases
        pts[3] = [0.0, 0.0, 0.1]
        phi, nrm, wit = sh.query(pts)
        out.update({f"{name}_pts": pts, f"{name}_phi": phi, f"{name}_normal": nrm,
                    f"{name}_witness": wit})
    nrm = rng.normal(size=(300, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:6] = np.array([[0, 0, 1.0], [1.0, 0, 0], [0, 1.0, 0], [0, 0, -1.0],
                        [np.sqrt(0.5), np.sqrt(0.5), 0.0], [0.6, 0.0, 0.8]])
    out["frames_normals"] = nrm
    out["frames"] = contact_frames(nrm)

    # a multi-body scene; JSON-described so tests can rebuild it
    scene = dict(bodies=[
        dict(name="floor", kinematic=True, position=[0, 0, 0], quat=[1, 0, 0, 0],
             v=[0.01, -0.02, 0.0], omega=[0.0, 0.0, 0.3],
             geoms=[dict(shape="halfspace", normal=[0, 0, 1], offset=0.0, position=[0, 0, 0],
                         quat=[1, 0, 0, 0], mu=0.5)]),
        dict(name="tool", kinematic=True, position=[0.05, 0.02, 0.12],
             quat=list(quat_from_axis_angle(np.array([0.3, 1.0, 0.2]), 0.7)),
             v=[0.1, 0.0, -0.2], omega=[0.5, -0.3, 1.0],
             geoms=[dict(shape="sphere", radius=0.04, position=[0.0, 0.0, 0.0],
                         quat=[1, 0, 0, 0], mu=0.8),
                    dict(shape="box", half_extents=[0.05, 0.02, 0.03],
                         position=[0.03, -0.02, 0.01],
                         quat=list(quat_from_axis_angle(np.array([0, 0, 1.0]), 0.4)), mu=0.6),
                    dict(shape="capsule", radius=0.015, half_length=0.05,
                         position=[-0.04, 0.03, -0.02],
                         quat=list(quat_from_axis_angle(np.array([1.0, 0, 0]), 1.1)), mu=0.3)]),
    ])
    bodies = build_ref_bodies(scene)
    x = rng.uniform([-0.1, -0.1, -0.01], [0.15, 0.15, 0.2], size=(3000, 3))
    n = x.shape[0]
    ps = ParticleSet(x=x, v=np.zeros((n, 3)), f=np.broadcast_to(np.eye(3), (n, 3, 3)).copy(),
                     c=np.zeros((n, 3, 3)), mass=np.ones(n), volume0=np.ones(n))
    cache = BiasCache()
    cs = detect_contacts(ps, bodies, margin=0.01, bias_cache=cache)
    # second detection with moved particles and mutated body velocity: cache semantics
    bodies[1].v = np.array([-0.3, 0.2, 0.1])
    ps.x = x + rng.normal(0.0, 0.004, size=x.shape)
    cs2 = detect_contacts(ps, bodies, margin=0.01, bias_cache=cache)
    out["scene_json"] = np.array(json.dumps(scene))
    out["det_x"] = x
    out["det_x2"] = ps.x
    out["det_body1_v2"] = bodies[1].v
    for tag, c in (("c1", cs), ("c2", cs2)):
        for k in ("particle", "body", "geom", "phi", "normal", "witness", "frames", "bias", "mu"):
            out[f"{tag}_{k}"] = getattr(c, k)
    save("sdf_contacts", **out)


def build_ref_bodies(scene):
    from mpmrb.bodies import GeomAttachment, RigidBody, Trajectory
    from mpmrb.geometry import Box, Capsule, HalfSpace, Sphere
    bodies = []
    for b in scene["bodies"]:
        geoms = []
        for g in b["geoms"]:
            if g["shape"] == "halfspace":
                sh = HalfSpace(normal=tuple(g["normal"]), offset=g["offset"])
            elif g["shape"] == "sphere":
                sh = Sphere(radius=g["radius"])
            elif g["shape"] == "box":
                sh = Box(half_extents=tuple(g["half_extents"]))
            else:
                sh = Capsule(radius=g["radius"], half_length=g["half_length"])
            geoms.append(GeomAttachment(shape=sh, position=np.asarray(g["position"], float),
                                        quat=np.asarray(g["quat"], float), mu=g["mu"]))
        traj = None
        if b.get("trajectory"):
            t = b["trajectory"]
            traj = Trajectory(times=np.asarray(t["times"]), positions=np.asarray(t["positions"]),
                              quats=np.asarray(t["quats"]))
        kw = {}
        if not b["kinematic"]:
            kw = dict(mass=b["mass"], inertia_body=np.asarray(b["inertia"], float))
        bodies.append(RigidBody(name=b["name"], kinematic=b["kinematic"], geoms=geoms,
                                position=np.asarray(b["position"], float),
                                quat=np.asarray(b["quat"], float),
                                v=np.asarray(b.get("v", [0, 0, 0]), float),
                                omega=np.asarray(b.get("omega", [0, 0, 0]), float),
                                trajectory=traj, **kw))
    return bodies


def gen_solver():
    from conftest import make_random_problem
    from mpmrb.solver import SolverParams, dense_newton_oracle, quasi_newton_solve
    tight = SolverParams(eps_r=1e-10, max_iters=3000)
    loose = SolverParams(eps_r=5e-2)
    out = {}
    seeds = [0, 1, 2, 3]
    for s in seeds:
        prob, contacts, grid, act = make_random_problem(s)
        pre = f"s{s}_"
        for k in ("m", "v_star", "v_init", "nodes", "w", "frames", "bias", "phi", "mu",
                  "gamma_lag"):
            out[pre + k] = getattr(prob, k)
        cp = prob.contact_params
        out[pre + "cparams"] = np.array([cp.stiffness, cp.tau_d, cp.eps_v, prob.dt])
        out[pre + "particle"] = contacts.particle
        for tag, par in (("tight", tight), ("loose", loose)):
            v, gam, rep = quasi_newton_solve(prob, par)
            out[pre + tag + "_v"] = v
            out[pre + tag + "_gamma"] = gam
            out[pre + tag + "_iters"] = np.int64(rep.iterations)
            out[pre + tag + "_conv"] = np.bool_(rep.converged)
            out[pre + tag + "_residual"] = np.array(rep.residual_trace)
            out[pre + tag + "_threshold"] = np.array(rep.threshold_trace)
            out[pre + tag + "_objective"] = np.array(rep.objective_trace)
            out[pre + tag + "_alpha"] = np.array(rep.alpha_trace)
        if s < 2:
            v, gam, rep = dense_newton_oracle(prob, tight)
            out[pre + "dense_v"] = v
        print(f"solver seed {s}: {prob.n_contacts} contacts, {prob.n_dofs} dofs")
    out["seeds"] = np.array(seeds)
    save("solver", **out)


def scene_resting_box():
    """conftest.resting_box_state(drop=0.0005, dt=4e-4, substeps=4) as JSON."""
    return dict(h=0.01, dt=4e-4, substeps=4, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e5, tau_d=4e-4, eps_v=1e-4, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=5e4, nu=0.3, rho=1000.0)],
                volumes=[dict(center=[0, 0, 0.0205], half=[0.02] * 3, material=0, ppc=8,
                              jitter=1.0, seed=0, velocity=[0, 0, 0])],
                bodies=[dict(name="floor", kinematic=True, position=[0, 0, 0],
                             quat=[1, 0, 0, 0],
                             geoms=[dict(shape="halfspace", normal=[0, 0, 1], offset=0.0,
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.8)])])


def scene_presser():
    """Blob on a floor pressed by a moving kinematic capsule plus a free ball."""
    return dict(h=0.015, dt=1e-3, substeps=4, gravity=[0, 0, -9.81],
                contact=dict(stiffness=1e4, tau_d=1e-3, eps_v=1e-3, margin=None),
                solver=dict(eps_r=5e-2),
                materials=[dict(E=1e5, nu=0.35, rho=1000.0), dict(E=4e4, nu=0.3, rho=800.0)],
                volumes=[dict(center=[0, 0, 0.0305], half=[0.03, 0.03, 0.03], material=0,
                              ppc=8, jitter=1.0, seed=4, velocity=[0.05, 0, -0.1]),
                         dict(center=[0.0, 0.0, 0.075], half=[0.015, 0.015, 0.012], material=1,
                              ppc=8, jitter=0.5, seed=5, velocity=[0, 0, -0.2])],
                bodies=[dict(name="floor", kinematic=True, position=[0, 0, 0],
                             quat=[1, 0, 0, 0],
                             geoms=[dict(shape="halfspace", normal=[0, 0, 1], offset=0.0,
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.6)]),
                        dict(name="pin", kinematic=True, position=[-0.02, 0.0, 0.105],
                             quat=[np.cos(np.pi / 4), np.sin(np.pi / 4), 0, 0],
                             trajectory=dict(times=[0.0, 0.05], positions=[[-0.02, 0, 0.105],
                                                                           [0.01, 0, 0.09]],
                                             quats=[[np.cos(np.pi / 4), np.sin(np.pi / 4), 0, 0]] * 2),
                             geoms=[dict(shape="capsule", radius=0.01, half_length=0.05,
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.7)]),
                        dict(name="ball", kinematic=False, mass=0.05,
                             inertia=(np.eye(3) * 2e-6).tolist(), position=[0.03, 0.0, 0.08],
                             quat=[1, 0, 0, 0], v=[0, 0, -0.3], omega=[0, 2.0, 0],
                             geoms=[dict(shape="box", half_extents=[0.01, 0.01, 0.01],
                                         position=[0, 0, 0], quat=[1, 0, 0, 0], mu=0.5)])])


def build_ref_state(scene):
    from mpmrb.contact_model import ContactParams
    from mpmrb.coupling import SimState, StepConfig
    from mpmrb.materials import Material
    from mpmrb.particles import concatenate, seed_box
    from mpmrb.solver import SolverParams
    mats = [Material(m["E"], m["nu"], m["rho"]) for m in scene["materials"]]
    sets = [seed_box(np.asarray(v["center"]), np.asarray(v["half"]), scene["h"],
                     mats[v["material"]], material_id=v["material"],
                     particles_per_cell=v["ppc"], jitter=v["jitter"],
                     velocity=tuple(v["velocity"]), seed=v["seed"]) for v in scene["volumes"]]
    c = scene["contact"]
    return SimState(particles=concatenate(sets), materials=mats,
                    bodies=build_ref_bodies(scene), h=scene["h"],
                    step=StepConfig(dt=scene["dt"], substeps=scene["substeps"],
                                    gravity=tuple(scene["gravity"])),
                    contact_params=ContactParams(stiffness=c["stiffness"], tau_d=c["tau_d"],
                                                 eps_v=c["eps_v"], margin=c["margin"]),
                    solver_params=SolverParams(eps_r=scene["solver"]["eps_r"]))


def gen_steps():
    from mpmrb.coupling import advance_step
    out = {}
    for tag, scene, nsteps in (("rest", scene_resting_box(), 6), ("press", scene_presser(), 8)):
        st = build_ref_state(scene)
        p = st.particles
        out[f"{tag}_scene_json"] = np.array(json.dumps(scene))
        out[f"{tag}_x0"], out[f"{tag}_v0"] = p.x.copy(), p.v.copy()
        out[f"{tag}_f0"], out[f"{tag}_c0"] = p.f.copy(), p.c.copy()
        out[f"{tag}_mass"], out[f"{tag}_vol"] = p.mass.copy(), p.volume0.copy()
        out[f"{tag}_mid"] = p.material_id.copy()
        wr, nc, it, conv, act, stale = [], [], [], [], [], []
        xs = []
        for _ in range(nsteps):
            s = advance_step(st)
            wr.append(s.wrench)
            nc.append(s.n_contacts_mean)
            it.append(s.iterations_mean)
            conv.append(s.all_converged)
            act.append(s.n_active_nodes)
            stale.append(s.staleness)
            xs.append(st.particles.x.copy())
        out[f"{tag}_wrench"] = np.stack(wr)
        out[f"{tag}_contacts_mean"] = np.array(nc)
        out[f"{tag}_iters_mean"] = np.array(it)
        out[f"{tag}_conv"] = np.array(conv)
        out[f"{tag}_active_mean"] = np.array(act)
        out[f"{tag}_staleness"] = np.array(stale)
        out[f"{tag}_xs"] = np.stack(xs)
        out[f"{tag}_x1"], out[f"{tag}_v1"] = st.particles.x, st.particles.v
        out[f"{tag}_f1"], out[f"{tag}_c1"] = st.particles.f, st.particles.c
        out[f"{tag}_bodies_pos"] = np.array([b.position for b in st.bodies])
        out[f"{tag}_bodies_quat"] = np.array([b.quat for b in st.bodies])
        out[f"{tag}_bodies_v"] = np.array([b.v for b in st.bodies])
        out[f"{tag}_bodies_omega"] = np.array([b.omega for b in st.bodies])
        print(f"steps {tag}: n={p.n}, contacts {np.mean(nc):.1f}, iters {np.mean(it):.2f}")
    save("steps", **out)


def _c1_run(mode, workers):
    from mpmrb.coupling import advance_step
    from paper_2503_05046_b200.scenes import elastic_cube_scene
    scene = elastic_cube_scene()
    st = build_ref_state(scene)
    st.mode, st.workers = mode, workers
    p = st.particles
    out = dict(scene_json=np.array(json.dumps(scene)), x0=p.x.copy(), v0=p.v.copy())
    keep = (10, 25, 50, 75, 100)
    wr, nc, ncmax, it, itmax, conv, act = [], [], [], [], [], [], []
    for k in range(1, scene["steps"] + 1):
        s = advance_step(st)
        wr.append(s.wrench)
        nc.append(s.n_contacts_mean)
        ncmax.append(s.n_contacts_max)
        it.append(s.iterations_mean)
        itmax.append(s.iterations_max)
        conv.append(s.all_converged)
        act.append(s.n_active_nodes)
        if k in keep:
            out[f"x_{k}"] = st.particles.x.copy()
            out[f"v_{k}"] = st.particles.v.copy()
        if k % 10 == 0:
            print(f"c1 {mode} step {k}: contacts {s.n_contacts_mean:.1f} "
                  f"iters {s.iterations_mean:.2f}", flush=True)
    out.update(wrench=np.stack(wr), contacts_mean=np.array(nc), contacts_max=np.array(ncmax),
               iters_mean=np.array(it), iters_max=np.array(itmax), conv=np.array(conv),
               active_mean=np.array(act),
               bodies_pos=np.array([b.position for b in st.bodies]))
    return out


def gen_c1():
    """configs[0]: the 8,000-particle elastic cube dropped
    onto a kinematic ground box, h = 0.01, dt = 1e-3, N = 10, run for the full
    100 rigid steps through the reference's advance_step (coupling.py:168-219)
    in its default deterministic mode.  Stored per step: wrench, contact /
    iteration means, convergence, active nodes; particle x / v at steps 10,
    25, 50, 75, 100.

    The same run in the reference's own "fast" mode (transfer.py:204-248:
    bin-ordered chunks summed by 4 workers, then merged -- a different float
    summation order that the reference tolerates at <= 1e-12 per scatter,
    test_transfer.py:85-93) is stored under ``fast_*``: the trajectory
    divergence that reassociation alone causes in the reference itself."""
    import sys as _s
    _s.path.insert(0, str(Path(__file__).resolve().parents[2]))
    det = _c1_run("deterministic", None)
    fast = _c1_run("fast", 4)
    out = dict(det)
    for k, v in fast.items():
        if k not in ("scene_json", "x0", "v0"):
            out[f"fast_{k}"] = v
    save("c1_cube", **out)


def gen_outputs():
    """Reference frame bytes (outputs.py:33-42), CSV frame and contact log
    (outputs.py:61-105) for small seeded arrays."""
    import tempfile
    from mpmrb import outputs as ro
    rng = np.random.default_rng(77)
    x = rng.normal(size=(7, 3))
    v = rng.normal(size=(7, 3))
    wr = rng.normal(size=(2, 6))
    out = dict(x=x, v=v, wrench=wr, time=np.array(0.123456789))
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        ro.write_frame(d / "a.bin", 0.123456789, x, v)
        ro.write_frame(d / "b.bin", 0.5, x)
        ro.write_frame_csv(d / "c.csv", 0.123456789, x, v)
        log = ro.ContactLogWriter(d / "contacts.csv", ["ground", "pusher"])
        log.log_step(0.002, {"ground": wr[0], "pusher": wr[1]})
        log.log_step(0.004, {"ground": -wr[0], "pusher": 2 * wr[1]})
        log.close()
        out["frame_v"] = np.frombuffer((d / "a.bin").read_bytes(), dtype=np.uint8)
        out["frame_nov"] = np.frombuffer((d / "b.bin").read_bytes(), dtype=np.uint8)
        out["frame_csv"] = np.frombuffer((d / "c.csv").read_bytes(), dtype=np.uint8)
        out["contact_log"] = np.frombuffer((d / "contacts.csv").read_bytes(), dtype=np.uint8)
    save("outputs", **out)


if __name__ == "__main__":
    _import_reference()
    which = sys.argv[1:] or ["binning", "p2g_g2p", "sdf_contacts", "solver", "steps", "outputs"]
    for w in which:
        globals()[f"gen_{w}"]()
