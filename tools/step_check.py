"""One rigid step of a bench workload on the GPU (fused path) and on the
oracle from the same GPU state.  The bench's 256k and 1M sand windows have one
solve at max_iters = 500 in their first loaded step (step 1): does the oracle
stop there too?  This runs STEP steps on the GPU, then one more from that
state on both, and prints both steps' solver summaries and the position
difference.

    python tools/step_check.py WORKLOAD [STEP] [NSTEPS] > gpurun_out/step_check.txt

NSTEPS > 1 continues both sides for NSTEPS steps (a trajectory comparison).
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
    nstep = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ncomp = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    sc = bench.workload_scene(name)
    st = scenes.build_state(sc)
    for i in range(nstep):
        s0 = mp.advance_step(st)
        print(f"step {i} gpu: iters max", s0.iterations_max, "mean", s0.iterations_mean,
              "converged", s0.all_converged, flush=True)
    p = st.particles.numpy()
    ref = oracle_state(sc, p["x"], p["v"], p["f"], p["c"], p["mass"], p["volume0"],
                       p["material_id"])
    ref.plastic = p["plastic"].copy()
    if st.cloth is not None:
        ref.cloth.d3 = st.cloth.d3.cpu().numpy().copy()
    for b, gb in zip(ref.bodies, st.bodies):
        b.position, b.quat = gb.position.copy(), gb.quat.copy()
        b.v, b.omega = gb.v.copy(), gb.omega.copy()
    ref.time, ref.step_index = st.time, st.step_index
    for k in range(nstep, nstep + ncomp):
        s1 = mp.advance_step(st)
        print(f"step {k} gpu: contacts", s1.n_contacts_mean, "iters max", s1.iterations_max,
              "mean", s1.iterations_mean, "converged", s1.all_converged,
              "unconverged substeps", s1.substeps_unconverged, flush=True)
        t0 = time.time()
        r1 = ostep.step(ref)
        print(f"step {k} oracle: contacts", r1["n_contacts_mean"], "iters max",
              r1["iterations_max"], "mean", r1["iterations_mean"], "converged",
              r1["all_converged"], f"({time.time() - t0:.0f} s)", flush=True)
        if st.cloth is not None:
            print("d3 max diff:", float(np.abs(st.cloth.d3.cpu().numpy() - ref.cloth.d3).max()))
        print("wrench rel diff:", float(np.abs(s1.wrench - r1["wrench"]).max()
                                        / max(np.abs(r1["wrench"]).max(), 1e-300)))
        print(f"x max diff after step {k}:",
              float(np.abs(st.particles.numpy()["x"] - ref.x).max()), flush=True)


if __name__ == "__main__":
    main()
