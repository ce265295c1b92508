"""Time the device QN solve on a real pusher-loaded sand problem for several
forced CTA counts (MPMRB_SOLVER_CTAS), reporting us/iteration and (with
MPMRB_SOLVER_PROF=1) the in-kernel phase breakdown.

    python tools/solver_scaling.py [steps_to_advance] [half_x]
"""

import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2503_05046_b200 as mp  # noqa: E402
from paper_2503_05046_b200 import scenes  # noqa: E402
from paper_2503_05046_b200.collision import contact_velocities  # noqa: E402
from paper_2503_05046_b200.contact_model import normal_impulse  # noqa: E402


def build_problem(steps=16, hx=0.2):
    sc = scenes.sand_pile_scene(half=(hx, hx, hx / 2))
    st = scenes.build_state(sc)
    for _ in range(steps):
        mp.advance_step(st)
    dt_s = sc["dt"] / sc["substeps"]
    p = st.particles
    grid = mp.SparseGrid.allocate(p.x, st.h)
    stencil = mp.build_stencil(p.x, grid)
    plan = mp.build_sort_plan(p.x, st.h, 0)
    mp.particle_to_grid(p, grid, stencil, st.materials, dt_s, plan, 0)
    mp.grid_update(grid, st.step.gravity, dt_s)
    con = mp.detect_contacts(p, st.bodies, st.margin)
    vcs = contact_velocities(con, stencil, grid.v_k)
    con.gamma_lag = normal_impulse(vcs[:, 2], con.phi, st.contact_params, dt_s)
    prob, act = mp.build_contact_problem(grid, stencil, con, st.contact_params, dt_s, plan, 0)
    print(f"n={p.n} contacts={prob.n_contacts} active nodes={prob.m.shape[0]}", flush=True)
    return prob


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 14
    hx = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
    prob = build_problem(steps, hx)
    par = mp.SolverParams(eps_r=5e-2, max_iters=200)
    import ctypes as C
    from paper_2503_05046_b200 import _lib
    prof = (C.c_uint64 * 16)()
    if os.environ.get("ONE_SOLVE"):
        # single solve for ncu capture
        v, g, rep = mp.quasi_newton_solve(prob, mp.SolverParams(eps_r=5e-2, max_iters=20))
        torch.cuda.synchronize()
        print("one solve", rep.iterations, rep.ls_evals)
        return
    for ctas in (os.environ.get("CTAS_LIST") or "1,32,64,128,148,0").split(","):
        os.environ["MPMRB_SOLVER_CTAS"] = ctas
        mp.quasi_newton_solve(prob, par)  # warm
        torch.cuda.synchronize()
        _lib.lib().mpmrb_solver_profile(_lib.ctx(), prof, 1)
        t0 = time.perf_counter()
        v, g, rep = mp.quasi_newton_solve(prob, par)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        _lib.lib().mpmrb_solver_profile(_lib.ctx(), prof, 1)
        it = max(1, rep.iterations)
        ph = [prof[k] / 1e3 / it for k in range(6)]
        print(f"ctas={ctas:>4}: {dt * 1e3:8.2f} ms, iters={rep.iterations}, "
              f"ls_evals={rep.ls_evals}, us/iter={dt * 1e6 / it:7.1f} | per-iter us: "
              f"N={ph[1]:.1f} D={ph[2]:.1f} LS={ph[3]:.1f} U={ph[4]:.1f} "
              f"in-sync={prof[10] / 1e3 / it:.1f} "
              f"(LS/eval={prof[3] / 1e3 / max(1, rep.ls_evals):.2f}) "
              f"ctas={prof[8] & 0xffffffff} group={prof[8] >> 32} "
              f"light_nodes={prof[11] & 0xffffffff} heavy_nodes={prof[11] >> 32} N_loopA={prof[12] / 1e3 / it:.1f} N_loopB={prof[13] / 1e3 / it:.1f}",
              flush=True)


if __name__ == "__main__":
    main()
