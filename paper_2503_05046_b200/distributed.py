"""Multi-GPU host plumbing: batched independent environments, one per rank.

The coupling step shards naturally only across independent scenes
(SURVEY.md §8(e)): every rank advances its own environment, no data-path
collective is needed, and throughput is reported as weak scaling with the
device time reduced as the MAX over ranks.  One process per GPU, launched by
``torch.distributed.run``; NCCL for the timing/statistics reductions on the
GPU box, gloo for the CPU tests (tests/test_distributed.py).

Slab decomposition of one large scene (P2G halo exchange, the contact problem
gathered to one rank) is ``slab.py``; see DESIGN.md §7.
"""

from __future__ import annotations

import copy
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

ENV_SEED_STRIDE = 1000  # per-rank seed offset of the seeded particle volumes


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK of this process (torchrun's variables)."""
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None) -> RankInfo:
    """Join the process group when WORLD_SIZE > 1 (idempotent).  The default
    backend is NCCL with the rank's GPU bound, gloo without CUDA."""
    info = rank_info()
    if info.world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(info.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", info.local_rank))
        else:
            dist.init_process_group(backend)
    return info


def env_scene(scene: dict, rank: int) -> dict:
    """The independent environment of ``rank``: the same configuration with the
    particle-volume seeds offset by rank (distinct jittered lattices)."""
    sc = copy.deepcopy(scene)
    for v in sc["volumes"]:
        v["seed"] = int(v["seed"]) + ENV_SEED_STRIDE * rank
    return sc


def _device() -> torch.device:
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Device time of the job = the slowest rank's (contract: max over ranks)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(units_per_rank: list[int] | int, seconds_max: float) -> float:
    """Whole-job throughput: the units all ranks processed over the max time."""
    total = sum(units_per_rank) if isinstance(units_per_rank, list) else units_per_rank
    return float(total) / float(seconds_max)


def gather_stats(stats: dict) -> list[dict] | None:
    """Per-rank statistics (contacts, iterations, ...) gathered on rank 0."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return [stats]
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(stats, out, dst=0)
    return out


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def shutdown() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()
