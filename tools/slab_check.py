"""Slab decomposition at bench size against the undecomposed fused step, from
the same initial state: run under torchrun (gloo lets the ranks share one
GPU), rank 0 prints one JSON line with per-step contact counts, iterations,
wrench and the final max |x| difference.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/slab_check.py [--workload sand] [--steps 3] [--solve gather0] [--ops]
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="sand")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--solve", default="gather0", choices=("gather0", "allreduce"))
    ap.add_argument("--ops", action="store_true")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo")
    import bench
    from paper_2503_05046_b200 import coupling, scenes, slab
    sc = bench.workload_scene(a.workload, 0)
    st = scenes.build_state(sc)
    x0 = st.particles.x.clone()
    ss = slab.SlabState.from_state(st, solve=a.solve)
    step = slab.slab_advance_step if a.ops else slab.slab_advance_step_fused
    sums = [step(ss) for _ in range(a.steps)]
    allp = slab.gather_particles(ss)
    if rank == 0:
        ref_state = scenes.build_state(sc)
        assert torch.equal(ref_state.particles.x, x0)
        ref = [coupling.advance_step(ref_state) for _ in range(a.steps)]
        h = sc["h"]
        dx = float((allp["x"] - ref_state.particles.x).abs().max())
        rows = []
        for s, r in zip(sums, ref):
            ws = float(np.abs(r.wrench).max()) or 1.0
            rows.append(dict(contacts=[s.n_contacts_mean, r.n_contacts_mean],
                             active=[s.n_active_nodes, r.n_active_nodes],
                             iterations=[s.iterations_mean, r.iterations_mean],
                             wrench_relerr=float(np.abs(s.wrench - r.wrench).max()) / ws))
        print(json.dumps(dict(workload=a.workload, particles=int(x0.shape[0]), ranks=world,
                              substep="ops" if a.ops else "fused", solve=a.solve,
                              steps=a.steps, max_dx_m=dx, max_dx_over_h=dx / h, per_step=rows)),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
