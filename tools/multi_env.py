"""Batched independent environments on ONE GPU, stepped concurrently.

    python tools/multi_env.py [--envs E] [--workload sand] [--steps K] [--warmup W]

The contact solve is latency-bound: while its line-search group works, most
SMs wait (profiles/r01_ncu_solver_2m_stalls.txt).  E environments each get
their own library context, CUDA stream and host thread.  Each solver grid is
sized to 148 / E CTAs (MPMRB_SOLVER_CTAS), so that E cooperative solves are
co-resident, and their phases interleave.  The script prints the aggregate
particle-substeps/s for E = 1 and for the requested E."""

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=2)
    ap.add_argument("--workload", default="sand")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    ctas = os.environ.get("MPMRB_SOLVER_CTAS")
    if ctas is None:
        os.environ["MPMRB_SOLVER_CTAS"] = str(148 // a.envs) if a.envs > 1 else "0"
    import torch
    import bench
    import paper_2503_05046_b200 as mp
    from paper_2503_05046_b200 import scenes
    from paper_2503_05046_b200.distributed import env_scene
    states = [scenes.build_state(env_scene(bench.workload_scene(a.workload, 0), e))
              for e in range(a.envs)]
    n = sum(s.particles.n for s in states)
    N = states[0].step.substeps
    snaps = [{k: getattr(s.particles, k).clone() for k in
              ("x", "v", "f", "c", "plastic")} for s in states]

    def restore():
        for s, sn in zip(states, snaps):
            for k, t in sn.items():
                getattr(s.particles, k).copy_(t)
            s.time, s.step_index = 0.0, 0

    def run(steps):
        errs = []

        def worker(s):
            try:
                for _ in range(steps):
                    mp.advance_step(s)
            except BaseException as e:  # surfaced below
                errs.append(e)

        th = [threading.Thread(target=worker, args=(s,)) for s in states]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]

    run(a.warmup)
    restore()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(a.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps(dict(envs=a.envs, solver_ctas=os.environ["MPMRB_SOLVER_CTAS"],
                          workload=a.workload, particles_total=n, steps=a.steps,
                          ms_per_step=dt * 1e3 / a.steps,
                          value=n * N * a.steps / dt, unit="particle-substeps/s (wall)")))


if __name__ == "__main__":
    main()
