"""``bench-transfer`` on the GPU (the reference's
``mpmrb bench-transfer``, cli.py:48-82).

Same payload as the reference: n particles uniform in a 64h cube (seed 0),
the sparse grid and 27-node stencils, values ~ N(0, 1) of shape (n, 27, 7);
then the 7-channel scatter timed per call (CUDA events).  Modes (same CSV
columns as the reference, cli.py:60-82):
  deterministic / fast  — scatter_reduce: the ordered segmented fold, each
                          (node, channel) summed in particle-id order, bitwise
                          the reference's deterministic result
                          (transfer.py:135-145); both modes take this path,
  naive                 — scatter_naive: one float64 atomic per contribution
                          (transfer.py:251-260's per-row baseline),
and the relative difference against the deterministic result.

    python -m paper_2503_05046_b200.bench_transfer --particles 100000 [--mode all]
"""

from __future__ import annotations

import argparse
import sys

import numpy as np
import torch


def payload(n: int, seed: int = 0):
    from .grid import SparseGrid
    from .mpm import build_stencil
    rng = np.random.default_rng(seed)
    h = 0.01
    positions = rng.uniform(0.0, 64 * h, size=(n, 3))
    pos = torch.as_tensor(positions, device="cuda")
    grid = SparseGrid.allocate(pos, h)
    stencil = build_stencil(pos, grid)
    values = torch.as_tensor(rng.standard_normal((n, 27, 7)), device="cuda")
    return grid, stencil, values, pos, h


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench_transfer")
    ap.add_argument("--particles", type=int, default=100000)
    ap.add_argument("--mode", choices=["deterministic", "fast", "naive", "all"], default="all")
    ap.add_argument("--repeats", type=int, default=20)
    args = ap.parse_args(argv)
    from .transfer import build_sort_plan, scatter_naive, scatter_reduce
    n = args.particles
    grid, stencil, values, pos, h = payload(n)
    plan = build_sort_plan(pos, h, epoch=0)
    modes = ["deterministic", "fast", "naive"] if args.mode == "all" else [args.mode]
    ref = scatter_reduce(stencil.nodes, values, grid.n_nodes, plan, 0, mode="deterministic")
    scale = float(ref.abs().max())
    print("mode,particles,workers,ms_per_scatter,rel_diff_vs_deterministic")
    for mode in modes:
        def run():
            if mode == "naive":
                return scatter_naive(stencil.nodes, values, grid.n_nodes)
            return scatter_reduce(stencil.nodes, values, grid.n_nodes, plan, 0, mode=mode)
        out = run()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(max(1, args.repeats)):
            out = run()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / max(1, args.repeats)
        rel = float((out - ref).abs().max()) / scale
        print(f"{mode},{n},gpu,{ms:.3f},{rel:.3e}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
