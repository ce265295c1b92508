"""Event-timed device solve on a pusher-loaded sand problem (diagnostics).

    python tools/solver_timing.py [steps] [half_x] [max_iters]
"""

import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import paper_2503_05046_b200 as mp  # noqa: E402
from solver_scaling import build_problem  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    hx = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    prob = build_problem(steps, hx)
    par = mp.SolverParams(eps_r=5e-2, max_iters=iters)
    a = torch.randn(4096, 4096, device="cuda")
    for rep_i in range(8):
        if rep_i >= 4:
            # keep the GPU busy right up to the solve (clock ramp-up check)
            t_end = time.perf_counter() + 0.3
            while time.perf_counter() < t_end:
                a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        v, g, rep = mp.quasi_newton_solve(prob, par)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(f"run {rep_i}: events {e0.elapsed_time(e1):8.3f} ms wall {wall * 1e3:8.3f} ms "
              f"iters={rep.iterations} ls={rep.ls_evals} conv={rep.converged}", flush=True)


if __name__ == "__main__":
    main()
