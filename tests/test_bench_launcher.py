"""bench.py's own multi-rank launcher on CPU: ``--gpus N`` outside torchrun
re-launches the script under torch.distributed.run (127.0.0.1), and the
reference arm runs P = min(nproc, N) concurrent CPU processes, one
environment each, and sums their throughput (BASELINE.md CPU-baseline plan).
The GPU arm's N > 1 path is the same launcher; its per-rank logic
(batched envs, max-over-ranks time) is covered by test_distributed.py."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
def test_reference_arm_two_ranks_via_own_launcher():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--workload", "cube", "--ref-budget", "1.5",
                          "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["processes"] == min(os.cpu_count() or 1, 2)
    assert d["value"] > 0 and d["unit"] == "particle-substeps/s"
    assert d["steps"] >= 1 and d["ms_per_step"] > 0
    # every timed step is one substep: steps x ms_per_step fits in the wall time
    assert d["steps"] * d["ms_per_step"] / 1e3 <= d["config"]["wall_s"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port"


def test_parse_defaults_to_the_north_star_workload():
    sys.path.insert(0, str(ROOT))
    import bench
    a = bench.parse([])
    assert a.workload == "sand1m" and a.gpus == 1 and a.warmup >= 3
    sc = bench.workload_scene("sand1m")
    assert sc["contact"]["eps_v"] == 1e-3
    # the pusher face starts at the sand face: contact-loaded from t = 0
    pusher = sc["bodies"][1]
    face = pusher["position"][0] + pusher["geoms"][0]["half_extents"][0]
    assert abs(face - (-sc["volumes"][0]["half"][0])) < 1e-12
