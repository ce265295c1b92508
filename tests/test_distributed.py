"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host path:
batched independent environments, one per rank.

Each rank builds its environment with ``distributed.env_scene``, advances it
with the CPU oracle (test infrastructure; the GPU path is exercised by the
gpu tests), and the job-level reductions of bench.py (max-over-ranks time,
summed units, gathered statistics) are checked against single-process runs of
the same environments.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tiny_scene():
    from paper_2503_05046_b200 import scenes
    sc = scenes.smoke_scene()
    sc["volumes"][0]["half"] = [0.01, 0.01, 0.01]
    sc["volumes"][0]["center"] = [0.0, 0.0, 0.0105]
    return sc


def _run_env(scene):
    """Two coupling steps of one environment with the CPU oracle."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle import step as ostep
    from paper_2503_05046_b200.scenes import host_particles
    from scenes import oracle_state
    a = host_particles(scene)
    st = oracle_state(scene, a["x"], a["v"], a["f"], a["c"], a["mass"], a["vol"], a["mid"])
    out = [ostep.step(st) for _ in range(2)]
    return dict(n=int(a["x"].shape[0]), x=st.x.copy(), contacts=out[-1]["n_contacts_mean"],
                iters=out[-1]["iterations_mean"], wrench=np.asarray(out[-1]["wrench"]))


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    from paper_2503_05046_b200 import distributed as D
    info = D.init("gloo")
    assert (info.rank, info.world) == (rank, world)
    scene = D.env_scene(_tiny_scene(), rank)
    res = _run_env(scene)
    # fake per-rank device time: the job time is the slowest rank's
    t_rank = 1.0 + rank
    t_job = D.max_over_ranks(t_rank)
    n_all = D.sum_over_ranks(res["n"])
    stats = D.gather_stats(dict(rank=rank, n=res["n"], contacts=res["contacts"],
                                iters=res["iters"], x0=res["x"][:4].tolist(),
                                wrench=res["wrench"].tolist()))
    D.barrier()
    if rank == 0:
        np.savez(Path(outdir) / "dist.npz", t_job=t_job, n_all=n_all,
                 thr=D.job_throughput(int(n_all), t_job),
                 stats=np.array([repr(s) for s in stats]))
    D.shutdown()


def test_env_scene_seeds_are_independent():
    from paper_2503_05046_b200 import distributed as D
    sc = _tiny_scene()
    s0, s1 = D.env_scene(sc, 0), D.env_scene(sc, 1)
    assert s0["volumes"][0]["seed"] != s1["volumes"][0]["seed"]
    assert sc["volumes"][0]["seed"] == s0["volumes"][0]["seed"]  # input untouched
    from paper_2503_05046_b200.scenes import host_particles
    a, b = host_particles(s0), host_particles(s1)
    k = min(a["x"].shape[0], b["x"].shape[0])
    assert k > 0 and not np.allclose(a["x"][:k], b["x"][:k])


def test_single_process_reductions_are_identity():
    from paper_2503_05046_b200 import distributed as D
    assert D.max_over_ranks(2.5) == 2.5
    assert D.sum_over_ranks(7) == 7
    assert D.job_throughput([3, 5], 2.0) == 4.0
    assert D.gather_stats({"a": 1}) == [{"a": 1}]


@pytest.mark.timeout(600)
def test_two_rank_batched_envs_gloo(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    d = np.load(tmp_path / "dist.npz", allow_pickle=False)
    assert float(d["t_job"]) == 2.0          # max over ranks
    stats = [eval(s) for s in d["stats"]]    # noqa: S307 - our own repr of plain dicts
    assert [s["rank"] for s in stats] == [0, 1]
    n_all = sum(s["n"] for s in stats)
    assert int(d["n_all"]) == n_all
    assert float(d["thr"]) == pytest.approx(n_all / 2.0)
    # each rank advanced its own environment, bit-identical to a single-process run
    from paper_2503_05046_b200 import distributed as D
    for s in stats:
        ref = _run_env(D.env_scene(_tiny_scene(), s["rank"]))
        np.testing.assert_array_equal(np.asarray(s["x0"]), ref["x"][:4])
        np.testing.assert_array_equal(np.asarray(s["wrench"]), ref["wrench"])
        assert s["contacts"] == ref["contacts"]
    # and the environments differ
    assert stats[0]["x0"] != stats[1]["x0"]
