"""Time the device QN solve on a real pusher-loaded sand problem for several
forced CTA counts (MPMRB_SOLVER_CTAS), reporting us/iteration and (with
MPMRB_SOLVER_PROF=1) the in-kernel phase breakdown.

    python tools/solver_scaling.py [steps_to_advance] [half_x] [half_z] [gap]

(10 0.4 0.1 0 is the profiled substep of the 1M bench window.)
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


def build_problem(steps=16, hx=0.2, hz=None, gap=None):
    kw = {} if gap is None else {"gap": gap}
    sc = scenes.sand_pile_scene(half=(hx, hx, hz if hz else hx / 2), **kw)
    st = scenes.build_state(sc)
    for _ in range(steps):
        mp.advance_step(st)
    dt_s = sc["dt"] / sc["substeps"]
    p = st.particles
    if not os.environ.get("NO_SORT"):
        # the fused path solves on (block, cell)-sorted particles; do the same
        import numpy as np
        x = p.x.cpu().numpy()
        cell = np.floor(x / st.h - 0.5).astype(np.int64)
        blk = cell >> 2
        order = np.lexsort((cell[:, 2] & 3, cell[:, 1] & 3, cell[:, 0] & 3,
                            blk[:, 2], blk[:, 1], blk[:, 0]))
        idx = torch.as_tensor(order, device=p.x.device)
        for k in ("x", "v", "f", "c", "mass", "volume0", "material_id", "plastic"):
            setattr(p, k, getattr(p, k)[idx].contiguous())
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
    import numpy as np
    nodes = prob.nodes.cpu().numpy() if hasattr(prob.nodes, "cpu") else np.asarray(prob.nodes)
    same = np.all(nodes[1:] == nodes[:-1], axis=1)
    runs = 1 + int((~same).sum())
    pc = con.particle.cpu().numpy() if hasattr(con.particle, "cpu") else np.asarray(con.particle)
    xc = p.x.cpu().numpy()[pc]
    cc = np.floor(xc / st.h - 0.5).astype(np.int64)
    samec = np.all(cc[1:] == cc[:-1], axis=1)
    print(f"   stencil runs={runs} base-cell runs={1 + int((~samec).sum())} "
          f"distinct cells={len(np.unique(cc, axis=0))}", flush=True)
    return prob


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 14
    hx = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
    hz = float(sys.argv[3]) if len(sys.argv) > 3 else None
    gap = float(sys.argv[4]) if len(sys.argv) > 4 else None
    prob = build_problem(steps, hx, hz, gap)
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
    for spec in (os.environ.get("CTAS_LIST") or "0").split(","):
        ctas, _, ls = spec.partition(":")
        os.environ["MPMRB_SOLVER_CTAS"] = ctas
        os.environ["MPMRB_SOLVER_LS_CTAS"] = ls or "0"
        mp.quasi_newton_solve(prob, par)  # warm
        torch.cuda.synchronize()
        _lib.lib().mpmrb_solver_profile(_lib.ctx(), prof, 1)
        reps = int(os.environ.get("REPS", "3"))
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            v, g, rep = mp.quasi_newton_solve(prob, par)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print("   solve ms:", " ".join(f"{1e3 * t:.2f}" for t in ts), flush=True)
        dt = sum(ts) / reps
        ctap = (C.c_uint64 * 800)()
        _lib.lib().mpmrb_solver_profile_cta(_lib.ctx(), ctap)
        _lib.lib().mpmrb_solver_profile(_lib.ctx(), prof, 1)
        it = max(1, rep.iterations) * reps
        import numpy as np
        cp = np.frombuffer(ctap, dtype=np.uint64).reshape(5, 160).astype(float) / 1e3 / it
        ncta = int(prof[8] & 0xffffffff)
        for ph, name in enumerate(["N", "D", "U", "N-reduce", "in-grid-sync (all)"]):
            v = cp[ph, :ncta]
            if os.environ.get("PER_CTA") == "2":
                print(f"   {name} all CTAs: " + " ".join(f"{x:.1f}" for x in v))
            elif os.environ.get("PER_CTA"):
                print(f"   {name} per CTA 0-7: " + " ".join(f"{x:.1f}" for x in v[:8])
                      + "  p10/50/90: " + " ".join(f"{x:.1f}" for x in np.percentile(v, [10, 50, 90])))
            print(f"   per-CTA {name} work us/iter: mean {v.mean():.2f} max {v.max():.2f} "
                  f"(cta {int(v.argmax())}) min {v.min():.2f}", flush=True)
        ph = [prof[k] / 1e3 / it for k in range(6)]
        nw, dw, uw = (prof[14] & 0xffffffff) / 1e3 / it, (prof[14] >> 32) / 1e3 / it, prof[15] / 1e3 / it
        print(f"ctas={spec:>7}: {dt * 1e3:8.2f} ms, iters={rep.iterations}, "
              f"ls_evals={rep.ls_evals}, us/iter={dt * 1e6 * reps / it:7.1f} | per-iter us: "
              f"N={ph[1]:.1f} (work {nw:.1f}) D={ph[2]:.1f} (work {dw:.1f}) LS={ph[3]:.1f} U={ph[4]:.1f} (work {uw:.1f}) "
              f"in-sync={prof[10] / 1e3 / it:.1f} kernel={sum(ph):.1f} (init {ph[0]:.1f} epi {ph[5]:.1f}) "
              f"(LS/eval={prof[3] / 1e3 / max(1, rep.ls_evals * reps):.2f}) "
              f"ctas={prof[8] & 0xffffffff} ls_group={prof[8] >> 32} "
              f"contact_nodes={prof[11] & 0xffffffff} groups={prof[11] >> 32} "
              f"ls_compute/eval={prof[12] / 1e3 / max(1, rep.ls_evals * reps):.2f} ls_reduce/eval={prof[13] / 1e3 / max(1, rep.ls_evals * reps):.2f}",
              flush=True)


if __name__ == "__main__":
    main()
