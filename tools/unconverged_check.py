"""Does the oracle also stop at max_iters where the GPU does?  The bench's
256k sand window has one solve at max_iters = 500 in its first loaded step.
This runs step 0 on the GPU, then step 1 from that state on the GPU (fused
path) and on the oracle, and prints both steps' solver summaries.

    python tools/unconverged_check.py [sand|sand1m] > gpurun_out/unconverged_check.txt
"""
import copy
import importlib
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
import paper_2503_05046_b200 as mp  # noqa: E402
from oracle import step as ostep  # noqa: E402

scenes = importlib.import_module("paper_2503_05046_b200.scenes")
oracle_state = importlib.import_module("scenes").oracle_state  # tests/scenes.py


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "sand"
    sc = bench.workload_scene(name)
    st = scenes.build_state(sc)
    s0 = mp.advance_step(st)
    print("step 0 gpu: iters max", s0.iterations_max, "mean", s0.iterations_mean,
          "converged", s0.all_converged, flush=True)
    p = st.particles.numpy()
    ref = oracle_state(sc, p["x"], p["v"], p["f"], p["c"], p["mass"], p["volume0"],
                       p["material_id"])
    ref.plastic = p["plastic"].copy()
    for b, gb in zip(ref.bodies, st.bodies):
        b.position, b.quat = gb.position.copy(), gb.quat.copy()
        b.v, b.omega = gb.v.copy(), gb.omega.copy()
    ref.time, ref.step_index = st.time, st.step_index
    s1 = mp.advance_step(st)
    print("step 1 gpu: contacts", s1.n_contacts_mean, "iters max", s1.iterations_max, "mean",
          s1.iterations_mean, "converged", s1.all_converged,
          "unconverged substeps", s1.substeps_unconverged, flush=True)
    t0 = time.time()
    r1 = ostep.step(ref)
    print("step 1 oracle: contacts", r1["n_contacts_mean"], "iters max", r1["iterations_max"],
          "mean", r1["iterations_mean"], "converged", r1["all_converged"],
          f"({time.time() - t0:.0f} s)", flush=True)
    print("x max diff after step 1:", float(np.abs(st.particles.numpy()["x"] - ref.x).max()))


if __name__ == "__main__":
    main()
