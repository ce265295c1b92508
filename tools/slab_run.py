"""Run one scene slab-decomposed over the ranks of a torchrun job and print one
JSON line (rank 0) with the device time per rigid step (max over ranks):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/slab_run.py [--workload multi4m|sand|sand1m] [--steps K] [--warmup W]

NCCL when every rank has its own GPU; --backend gloo lets several ranks share
one GPU (functional runs only).  By default each rank runs the fused
simulator's kernels with the slab exchanges between the substep's parts
(slab_advance_step_fused); --ops composes the fine-grained device operators
instead (slab_advance_step); --solve picks the distributed contact solve."""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="multi4m")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--backend", default=None)
    ap.add_argument("--solve", default="gather0", choices=("gather0", "allreduce"))
    ap.add_argument("--single", action="store_true",
                    help="world 1 only: the undecomposed fused coupling.advance_step on the "
                         "same window, for comparison")
    ap.add_argument("--ops", action="store_true",
                    help="operator-by-operator substep (slab_advance_step) instead of the fused "
                         "simulator's kernels (slab_advance_step_fused)")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    backend = a.backend or ("nccl" if torch.cuda.device_count() >= world else "gloo")
    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        dist.init_process_group(backend)
    import bench
    from paper_2503_05046_b200 import scenes, slab
    sc = bench.workload_scene(a.workload, 0)
    st = scenes.build_state(sc)
    ss = slab.SlabState.from_state(st, solve=a.solve)
    step = slab.slab_advance_step if a.ops else slab.slab_advance_step_fused
    if a.single:
        from paper_2503_05046_b200 import coupling
        assert world == 1, "--single is the one-process reference run"
        step = lambda _ss: coupling.advance_step(st)  # noqa: E731
    for _ in range(a.warmup):
        step(ss)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sums = [step(ss) for _ in range(a.steps)]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:  # device time of the job = the slowest rank's
        tt = ss.comm.allgather(torch.tensor([[ms]], dtype=torch.float64))
        ms = max(float(x.item()) for x in tt)
    n = sums[-1].n_particles
    if rank == 0:
        print(json.dumps(dict(metric="MPM particle-substeps/sec incl. convex contact solve",
                              value=n * sc["substeps"] / (ms * 1e-3), unit="particle-substeps/s",
                              n_gpus=world, decomposition="slab", backend=backend, solve=a.solve,
                              substep="single" if a.single else ("ops" if a.ops else "fused"),
                              steps=a.steps, warmup=a.warmup, ms_per_step=ms,
                              wall_s=time.perf_counter() - t0,
                              config=dict(workload=a.workload, particles=n,
                                          substeps=sc["substeps"],
                                          contacts_mean=sums[-1].n_contacts_mean,
                                          solver_iters_mean=sums[-1].iterations_mean))),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
