"""Convergence study of the sand-pile workload: per-step solver iterations,
unconverged solves and device time for scene variants.

    python tools/diag_converge.py [steps] [half_x,half_y,half_z] [variant ...]

Prints one JSON line per variant.
"""

import copy
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2503_05046_b200 as mp  # noqa: E402
from paper_2503_05046_b200 import scenes  # noqa: E402


def variant(base, name):
    v = copy.deepcopy(base)
    pusher = v["bodies"][1]
    if name == "base":
        pass
    elif name == "epsv1e-3":
        v["contact"]["eps_v"] = 1e-3
    elif name == "epsv1e-2":
        v["contact"]["eps_v"] = 1e-2
    elif name == "pmu0":
        pusher["geoms"][0]["mu"] = 0.0
    elif name == "k1e4":
        v["contact"]["stiffness"] = 1e4
    elif name == "slow":
        t = pusher["trajectory"]
        t["positions"][1][0] = t["positions"][0][0] + 0.5
    elif name == "raised":
        dz = 0.03
        pusher["position"][2] += dz
        for p in pusher["trajectory"]["positions"]:
            p[2] += dz
    elif name == "inside":
        # pusher starts 1 mm inside the sand: contact-loaded from t = 0
        for p in [pusher["position"]] + pusher["trajectory"]["positions"]:
            p[0] += 0.006
    elif name == "inside_raised":
        for p in [pusher["position"]] + pusher["trajectory"]["positions"]:
            p[0] += 0.006
            p[2] += 0.03
    elif name == "touch3":
        # the bench scene: eps_v = 1e-3, pusher face starting at the sand face
        v["contact"]["eps_v"] = 1e-3
        for p in [pusher["position"]] + pusher["trajectory"]["positions"]:
            p[0] += 0.005
    elif name == "inside3":
        v["contact"]["eps_v"] = 1e-3
        for p in [pusher["position"]] + pusher["trajectory"]["positions"]:
            p[0] += 0.006
    elif name == "elastic":
        v["materials"][0]["model"] = "elastic"
    elif name == "eps_r1e-1":
        v["solver"]["eps_r"] = 1e-1
    else:
        raise ValueError(name)
    return v


def run(scene, steps, label):
    st = scenes.build_state(scene)
    rows = []
    stream = None
    total_ms = 0.0
    for k in range(steps):
        if stream is None:
            mp.advance_step(st)  # creates the stream; counted as a step
            stream = st._stream
            continue
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s = mp.advance_step(st)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        total_ms += ms
        rows.append(dict(k=k, ms=round(ms, 2), it=round(s.iterations_mean, 1),
                         itmax=s.iterations_max, unconv=s.substeps_unconverged,
                         nc=round(s.n_contacts_mean)))
    its = sum(r["it"] for r in rows) * scene["substeps"]
    unc = sum(r["unconv"] for r in rows)
    print(json.dumps(dict(variant=label, n=st.particles.n, steps=len(rows),
                          ms_per_step=total_ms / max(1, len(rows)), iters_total=its,
                          substeps_unconverged=unc, rows=rows)), flush=True)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    half = tuple(float(a) for a in sys.argv[2].split(",")) if len(sys.argv) > 2 else (0.2, 0.2, 0.1)
    names = sys.argv[3:] or ["base"]
    base = scenes.sand_pile_scene(half=half, eps_v=1e-4)  # round-1 scene
    for nm in names:
        t0 = time.perf_counter()
        run(variant(base, nm), steps, nm)
        print(f"# {nm}: {time.perf_counter() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
