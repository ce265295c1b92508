"""Scene builders shared by the oracle and the CUDA path in tests and bench.

A scene is a JSON-able dict (see tests/golden/make_golden.py).  The oracle gets
plain namespace bodies with tuple shapes; the product gets its own classes.
"""

from __future__ import annotations

import copy
import json
from types import SimpleNamespace

import numpy as np


def load_scene_json(s) -> dict:
    if isinstance(s, np.ndarray):
        s = str(s)
    return json.loads(s) if isinstance(s, str) else copy.deepcopy(s)


def _shape_tuple(g):
    if g["shape"] == "halfspace":
        return ("halfspace", tuple(g["normal"]), float(g["offset"]))
    if g["shape"] == "sphere":
        return ("sphere", float(g["radius"]))
    if g["shape"] == "box":
        return ("box", tuple(g["half_extents"]))
    return ("capsule", float(g["radius"]), float(g["half_length"]))


def _qnorm(q):
    q = np.asarray(q, dtype=np.float64)
    return q / np.linalg.norm(q)


def oracle_bodies(scene) -> list:
    out = []
    for b in scene["bodies"]:
        geoms = [SimpleNamespace(shape=_shape_tuple(g), position=np.asarray(g["position"], float),
                                 quat=_qnorm(g["quat"]), mu=float(g["mu"])) for g in b["geoms"]]
        traj = None
        if b.get("trajectory"):
            t = b["trajectory"]
            traj = SimpleNamespace(times=np.asarray(t["times"], float),
                                   positions=np.asarray(t["positions"], float),
                                   quats=np.stack([_qnorm(q) for q in (
                                       t.get("quats") or [[1.0, 0, 0, 0]] * len(t["times"]))]))
        ns = SimpleNamespace(name=b["name"], kinematic=bool(b["kinematic"]), geoms=geoms,
                             position=np.asarray(b["position"], float), quat=_qnorm(b["quat"]),
                             v=np.asarray(b.get("v", [0, 0, 0]), float),
                             omega=np.asarray(b.get("omega", [0, 0, 0]), float),
                             trajectory=traj,
                             mass=float(b.get("mass", 0.0)),
                             inertia_body=np.asarray(b.get("inertia", np.eye(3)), float))
        if ns.kinematic and traj is not None:
            from oracle.step import sample_trajectory
            ns.position, ns.quat, ns.v, ns.omega = sample_trajectory(traj, 0.0)
        out.append(ns)
    return out


def oracle_materials(scene) -> list:
    return [SimpleNamespace(youngs_modulus=m["E"], poisson_ratio=m["nu"], density=m["rho"],
                            model=m.get("model", "elastic"),
                            friction_angle=m.get("friction_angle", 30.0))
            for m in scene["materials"]]


def oracle_cloth(scene, n_total: int):
    """oracle.cloth.ClothMesh of the scene's sheets, which follow the volume
    particles at the end of the particle arrays (scenes.build_particles)."""
    if not scene.get("cloth"):
        return None
    from oracle import cloth as oc
    from paper_2503_05046_b200.scenes import cloth_arrays
    sheets = cloth_arrays(scene)
    first = n_total - sum(a["x"].shape[0] for a in sheets)
    tri, ep, dmi, vol, d3 = [], [], [], [], []
    for a in sheets:
        tri.append(a["tri"] + first)
        ep.append(a["epart"] + first)
        dmi.append(a["dm_inv"])
        vol.append(a["vol_e"])
        d3.append(a["d3"])
        first += a["x"].shape[0]
    m = scene["materials"][scene["cloth"][0]["material"]]
    params = oc.params_from(m["E"], m["nu"], m.get("k_normal"), m.get("gamma_shear"),
                            m.get("cloth_friction", 0.3))
    return oc.ClothMesh(tri=np.concatenate(tri), epart=np.concatenate(ep),
                        dm_inv=np.concatenate(dmi), vol=np.concatenate(vol),
                        d3=np.concatenate(d3), params=params)


def oracle_state(scene, x, v, f, c, mass, vol, mid):
    from oracle.solver import Params
    from oracle.step import OracleState
    con = scene["contact"]
    sp = Params(eps_r=scene["solver"].get("eps_r", 5e-2))
    if "max_iters" in scene["solver"]:
        sp.max_iters = scene["solver"]["max_iters"]
    return OracleState(x=np.array(x, float), v=np.array(v, float), f=np.array(f, float),
                       c=np.array(c, float), mass=np.array(mass, float),
                       vol0=np.array(vol, float), material_id=np.array(mid, np.int64),
                       materials=oracle_materials(scene), bodies=oracle_bodies(scene),
                       h=scene["h"], dt=scene["dt"], substeps=scene["substeps"],
                       gravity=tuple(scene["gravity"]), k=con["stiffness"], tau_d=con["tau_d"],
                       eps_v=con["eps_v"], margin=con.get("margin"), solver=sp,
                       cloth=oracle_cloth(scene, np.asarray(x).shape[0]))
