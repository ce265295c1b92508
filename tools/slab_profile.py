import cProfile, pstats, sys, io, torch
sys.path.insert(0, '.')
import bench
from paper_2503_05046_b200 import scenes, slab
sc = bench.workload_scene("sand", 0)
st = scenes.build_state(sc)
ss = slab.SlabState.from_state(st)
slab.slab_advance_step_fused(ss); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(2): slab.slab_advance_step_fused(ss)
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(35); print(s.getvalue())
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(40); print(s.getvalue())
