"""Convergence / speed study of a bench workload under scene-parameter and
solver-grid variants (diagnostics; bench.py measures the committed scenes):

    python tools/scene_study.py WORKLOAD STEPS [key=value ...]

keys: eps_v, stiffness (contact), ctas (MPMRB_SOLVER_CTAS).  Prints ms per
rigid step (device events), solver iterations per substep and the solves
that stopped at max_iters."""

import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    workload, steps = sys.argv[1], int(sys.argv[2])
    kv = dict(a.split("=") for a in sys.argv[3:])
    if "ctas" in kv:
        os.environ["MPMRB_SOLVER_CTAS"] = kv["ctas"]
    import bench
    import paper_2503_05046_b200 as mp
    from paper_2503_05046_b200 import scenes
    sc = bench.workload_scene(workload, 0)
    for k in ("eps_v", "stiffness"):
        if k in kv:
            sc["contact"][k] = float(kv[k])
    st = scenes.build_state(sc)
    ms, its, unconv = [], [], 0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st._stream if st._stream is not None else torch.cuda.current_stream())
        s = mp.advance_step(st)
        e1.record(st._stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        its.append(s.iterations_mean)
        unconv += s.substeps_unconverged
    print(f"{workload} {kv}: ms/step {np.mean(ms[1:]):.2f}  iters/substep {np.mean(its):.1f}  "
          f"unconverged solves {unconv} of {steps * sc['substeps']}", flush=True)


if __name__ == "__main__":
    main()
