"""Host and device profile of the fused slab step at one rank (256k sand,
steps 1-2): cProfile of the host glue and torch.profiler's CUDA kernel table."""
import cProfile
import io
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_05046_b200 import scenes, slab  # noqa: E402

sc = bench.workload_scene(sys.argv[1] if len(sys.argv) > 1 else "sand", 0)
st = scenes.build_state(sc)
ss = slab.SlabState.from_state(st)
slab.slab_advance_step_fused(ss)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2):
    slab.slab_advance_step_fused(ss)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(30)
print(s.getvalue())
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        slab.slab_advance_step_fused(ss)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40))
