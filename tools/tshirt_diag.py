"""Why the T-shirt fold's pinch solves stop at max_iters: residual and
threshold traces of its unconverged substeps (op-by-op path), GPU and oracle."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import bench
    from paper_2503_05046_b200 import scenes
    from paper_2503_05046_b200.coupling import _advance_substep
    from paper_2503_05046_b200.transfer import build_sort_plan
    import paper_2503_05046_b200 as mp
    pinch = float(sys.argv[1]) if len(sys.argv) > 1 else None
    sc = bench.workload_scene("tshirt", 0)
    if pinch is not None:
        for b in sc["bodies"][1:]:
            p = b["trajectory"]["positions"]
            p[1][2] = p[0][2] - pinch
    st = scenes.build_state(sc)
    n = sc["substeps"]
    for step in range(20):
        plan = build_sort_plan(st.particles.x, st.h, st.step_index)
        st._bias_cache.clear()
        st._accum.reset()
        for k in range(n):
            info = _advance_substep(st, sc["dt"] / n, plan, st.step_index)
            rep = info["report"]
            if not rep.converged:
                res, thr = np.array(rep.residual_trace), np.array(rep.threshold_trace)
                print(f"step {step} sub {k}: contacts {info['n_contacts']} iters {rep.iterations} "
                      f"res {res[-1]:.3e} thr {thr[-1]:.3e} min res {res.min():.3e} "
                      f"res@50 {res[min(50, len(res) - 1)]:.3e} alpha_last {rep.alpha_trace[-5:]}",
                      flush=True)
        from paper_2503_05046_b200.coupling import _rigid_update
        _rigid_update(st, st.time + st.step.dt)
        st.time += st.step.dt
        st.step_index += 1


if __name__ == "__main__":
    main()
