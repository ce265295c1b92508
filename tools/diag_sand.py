"""Diagnostics for the sand-pile workload: per-step solver iterations for
scene variants, and GPU-vs-oracle agreement on a hard (pusher-loaded) substep.

    python tools/diag_sand.py [steps]
"""

import copy
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2503_05046_b200 as mp  # noqa: E402
from paper_2503_05046_b200 import scenes  # noqa: E402


def run(scene, steps, label):
    st = scenes.build_state(scene)
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        s = mp.advance_step(st)
        its.append((round(s.iterations_mean, 1), s.iterations_max, round(s.n_contacts_mean)))
    torch.cuda.synchronize()
    print(label, f"{time.perf_counter() - t0:.2f}s", its, flush=True)
    return st


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    base = scenes.sand_pile_scene(half=(0.1, 0.1, 0.05))  # 32k particles, same physics
    run(base, steps, "base")
    v = copy.deepcopy(base)
    v["contact"]["eps_v"] = 1e-3
    run(v, steps, "eps_v=1e-3")
    v = copy.deepcopy(base)
    v["materials"][0]["model"] = "elastic"
    run(v, steps, "elastic")
    v = copy.deepcopy(base)
    v["bodies"][1]["geoms"][0]["mu"] = 0.0
    run(v, steps, "pusher mu=0")
    v = copy.deepcopy(base)
    v["contact"]["stiffness"] = 1e4
    run(v, steps, "k=1e4")

    # GPU vs oracle on a hard substep
    from oracle import step as ostep
    from scenes import oracle_state
    st = run(base, steps, "base again")
    p = st.particles.numpy()
    sc = copy.deepcopy(base)
    sc["dt"] = base["dt"] / base["substeps"]
    sc["substeps"] = 1
    ref = oracle_state(sc, p["x"], p["v"], p["f"], p["c"], p["mass"], p["volume0"],
                       p["material_id"])
    ref.plastic = p["plastic"].copy()
    from paper_2503_05046_b200.bodies import geom_structs  # noqa: F401
    ob = ref.bodies
    for b, gb in zip(ob, st.bodies):
        b.position, b.quat, b.v, b.omega = gb.position.copy(), gb.quat.copy(), gb.v.copy(), gb.omega.copy()
    gst = scenes.build_state(sc, particles=st.particles.copy())
    for b, gb in zip(gst.bodies, st.bodies):
        b.position, b.quat, b.v, b.omega = gb.position.copy(), gb.quat.copy(), gb.v.copy(), gb.omega.copy()
    t0 = time.perf_counter()
    r = ostep.step(ref)
    t_ref = time.perf_counter() - t0
    s = mp.advance_step(gst)
    print("oracle substep", f"{t_ref:.1f}s", "iters", r["iterations_mean"], "contacts",
          r["n_contacts_mean"], "| gpu iters", s.iterations_mean, "contacts", s.n_contacts_mean)
    print("max|dx|", float(np.abs(gst.particles.x.cpu().numpy() - ref.x).max()),
          "wrench", r["wrench"].tolist(), s.wrench.tolist())


if __name__ == "__main__":
    main()
