#!/usr/bin/env python
"""Benchmark of the fused MPM + convex-contact coupling step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sand1m|sand|cube|cloth|tshirt|multi4m]

A "step" is one rigid coupling step (N substeps of P2G -> grid update ->
contact detection -> device quasi-Newton solve -> G2P).  The default workload
is the scene BASELINE.json's north_star quotes its steps/s target on: a
1M-particle Drucker-Prager sand block on a floor, pushed by a kinematic box
whose face starts at the sand's face, so every timed step is contact-loaded
(SURVEY.md §8d C2 geometry at 0.8 x 0.8 x 0.2 m).  configs[1] (256k) is
``--workload sand``.  Inputs are synthetic (seeded jittered lattice), float64.

The timed window is the first K rigid steps of the scene from t = 0 (warm-up
steps run first and are rolled back), with L2 flushed between steps.

Metric: MPM particle-substeps/s including the convex contact solve (whole job,
all ranks), with ms per rigid step and rigid steps/s.  ``--gpus N`` without
torchrun re-launches itself under torch.distributed.run: N batched independent
environments, one per GPU (weak scaling, no data-path collective); timing is
device time (CUDA events) reduced as the MAX over ranks.

The cpu_baseline leg and ``--impl reference`` time the CPU oracle port
(oracle/, a float64 NumPy restatement of the reference, which is itself pure
NumPy and single-threaded) on this host on the contiguous prefix of the SAME
window: substeps 0, 1, 2, ... of the same scene from t = 0, until a time
budget is spent.  ``--impl reference --gpus N`` runs P = min(nproc, N)
environments as concurrent CPU processes and sums their throughput.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPM particle-substeps/sec incl. convex contact solve; ms per rigid step"
UNIT = "particle-substeps/s"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
WORKLOADS = ["sand1m", "sand", "cube", "cloth", "tshirt", "multi4m"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=WORKLOADS, default="sand1m")
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64",
                    help="f64: the reference's float64 throughout (default); f32: the fused "
                         "path's performance mode (float32 particle state and arithmetic, "
                         "float64 positions, grid and contact solve) -- narrower than the "
                         "reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=90.0,
                    help="seconds of timed CPU work per reference environment")
    ap.add_argument("--ncu-window", action="store_true",
                    help="only run to the profiled substep and bracket it with "
                         "cudaProfilerStart/Stop (ncu --profile-from-start off)")
    return ap.parse_args(argv)


def workload_scene(name: str, rank: int = 0) -> dict:
    from paper_2503_05046_b200 import scenes
    from paper_2503_05046_b200.distributed import env_scene
    if name == "sand":
        sc = scenes.sand_pile_scene(gap=0.0)
    elif name == "sand1m":
        sc = scenes.sand_pile_scene(half=(0.4, 0.4, 0.1), gap=0.0)
    elif name == "cloth":
        sc = scenes.cloth_sheet_scene()
        # start the sheet 3.5 mm above the sphere so the timed window is in contact
        sc["cloth"][0]["center"] = [0.0, 0.0, 0.2535]
        sc["cloth"][0]["velocity"] = [0.0, 0.0, -0.2]
    elif name == "tshirt":
        sc = scenes.tshirt_fold_scene()
    elif name == "multi4m":
        sc = scenes.multi_material_scene()
        # start the block on the floor and the pusher 1 mm clear (inside the
        # contact margin) so the timed window is contact-loaded from t = 0
        for vol in sc["volumes"]:
            vol["center"][2] = vol["half"][2]
        pusher = sc["bodies"][1]
        x0 = -sc["volumes"][1]["center"][0] * 2 - 0.05 - 0.001
        pusher["position"][0] = x0
        pusher["trajectory"]["positions"] = [[x0, 0, pusher["position"][2]],
                                             [x0 + 2.0, 0, pusher["position"][2]]]
    else:
        sc = scenes.elastic_cube_scene()
    return env_scene(sc, rank)  # independent environment per rank


def workload_name(name: str, n: int, N: int) -> str:
    return {
        "sand": f"sand pile (configs[1]): {n} particles/GPU, Drucker-Prager sand, floor + "
                f"kinematic pusher box (face at the sand face at t=0, +0.2 m/s), dt=2e-3, "
                f"N={N} substeps",
        "sand1m": f"sand pile 1M (north-star target scene): {n} particles/GPU, Drucker-Prager "
                  f"sand, floor + kinematic pusher box (face at the sand face at t=0, "
                  f"+0.2 m/s), dt=2e-3, N={N} substeps",
        "cube": f"elastic cube (configs[0]): {n} particles, dt=1e-3, N={N}",
        "cloth": f"cloth sheet over a sphere (configs[2]): {n} particles (vertices + faces), "
                 f"codimensional cloth, dt=2e-3, N={N}",
        "tshirt": f"cloth fold with two grippers (configs[3]): {n} particles, dt=2e-3, N={N}",
        "multi4m": f"multi-material block (configs[4], 1 GPU): {n} particles, elastic | "
                   f"Drucker-Prager sand split at x=0, h=5 mm, floor + kinematic pusher box, "
                   f"dt=2e-3, N={N} substeps",
    }[name]


def host_particles(scene: dict):
    from paper_2503_05046_b200.scenes import host_particles as hp
    return hp(scene)


def peaks():
    try:
        d = json.loads(PEAKS_FILE.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args, argv) -> int:
    """``--gpus N`` outside torchrun: re-run this script as N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1.  Rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ CPU oracle

def oracle_window(scene: dict, budget_s: float, max_substeps: int | None = None) -> dict:
    """Time the oracle port on the contiguous prefix of the workload's window:
    substeps 0, 1, 2, ... of the scene from t = 0 (rigid-step boundaries
    handled exactly as oracle.step.step does), one thread, until ``budget_s``
    of timed work is spent (at least one substep)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle import grid as og
    from oracle import step as ostep
    from scenes import oracle_state
    arr = host_particles(scene)
    s = oracle_state(scene, arr["x"], arr["v"], arr["f"], arr["c"], arr["mass"], arr["vol"],
                     arr["mid"])
    n = arr["x"].shape[0]
    N = scene["substeps"]
    dt_s = scene["dt"] / N
    secs, iters, ncs = [], [], []
    k = 0
    while True:
        t0 = time.perf_counter()
        if k % N == 0:  # rigid-step start (coupling.py:168-182)
            ostep.check_health(s)
            og.sort_plan(s.x, s.h, s.step_index)
            s.cache.clear()
            s.acc_lin[:] = 0.0
            s.acc_ang[:] = 0.0
        info = ostep.substep(s, dt_s)
        ostep.check_health(s)
        if k % N == N - 1:  # rigid update (coupling.py:192-219)
            t_new = s.time + s.dt
            for bi, body in enumerate(s.bodies):
                ostep.rigid_update(body, s.acc_lin[bi], s.acc_ang[bi], s.gravity, s.dt, t_new)
            s.time = t_new
            s.step_index += 1
        secs.append(time.perf_counter() - t0)
        iters.append(int(info["report"].iterations))
        ncs.append(int(info["contacts"].n))
        k += 1
        if sum(secs) + secs[-1] > budget_s or (max_substeps and k >= max_substeps):
            break
    t = sum(secs)
    return dict(n=n, substeps=k, seconds=t, value=n * k / t, iters=iters, contacts=ncs)


def oracle_loaded_substep(scene: dict, snap: dict) -> dict:
    """Time the oracle port on ONE contact-loaded substep of the window: the
    substep the GPU arm profiles (substep 0 of window step K/2), started from
    the GPU state at that point (particles, plastic strain, body poses and
    velocities, time), one thread.  A representative sample of the window's
    work, next to the window prefix (substeps 0, 1, ...; 1 solver iteration)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle import grid as og
    from oracle import step as ostep
    from scenes import oracle_state
    s = oracle_state(scene, snap["x"], snap["v"], snap["f"], snap["c"], snap["mass"],
                     snap["volume0"], snap["material_id"])
    s.plastic = snap["plastic"].copy()
    for b, (pos, quat, vel, om) in zip(s.bodies, snap["bodies"]):
        b.position, b.quat, b.v, b.omega = pos.copy(), quat.copy(), vel.copy(), om.copy()
    s.time, s.step_index = snap["time"], snap["step_index"]
    N = scene["substeps"]
    t0 = time.perf_counter()
    ostep.check_health(s)  # rigid-step start (coupling.py:168-182), then one substep
    og.sort_plan(s.x, s.h, s.step_index)
    s.cache.clear()
    s.acc_lin[:] = 0.0
    s.acc_ang[:] = 0.0
    info = ostep.substep(s, scene["dt"] / N)
    t = time.perf_counter() - t0
    n = snap["x"].shape[0]
    return dict(value=n / t, seconds=t, iterations=int(info["report"].iterations),
                contacts=int(info["contacts"].n), n=n)


def _window_sample_text(r: dict, N: int) -> str:
    return (f"substeps 0..{r['substeps'] - 1} of the timed window's scene from t=0 "
            f"(contiguous prefix of the GPU window; {r['n']} particles, "
            f"{np.mean(r['contacts']):.0f} contacts and {np.mean(r['iters']):.1f} solver "
            f"iterations per substep on average), {r['seconds']:.1f} s, one rigid step = "
            f"{N} substeps")


def _ref_worker(args_tuple):
    workload, env, budget = args_tuple
    os.environ["OMP_NUM_THREADS"] = "1"
    scene = workload_scene(workload, env)
    # untimed warm-up: one substep of a small sub-block (imports, allocators)
    small = json.loads(json.dumps(scene))
    for vol in small.get("volumes", []):
        vol["half"] = [a / 4 for a in vol["half"]]
    if small.get("volumes"):
        oracle_window(small, 0.0, max_substeps=1)
    r = oracle_window(scene, budget)
    r["N"] = scene["substeps"]
    return r


def run_reference(args):
    """The reference arm: the CPU oracle port of the pure-NumPy reference on
    this host's cores (see the module docstring)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    envs = max(args.gpus, world)
    P = max(1, min(os.cpu_count() or 1, envs))
    jobs = [(args.workload, e, args.ref_budget) for e in range(P)]
    t_wall = time.perf_counter()
    if P == 1:
        res = [_ref_worker(jobs[0])]
    else:
        import multiprocessing as mpr
        with mpr.get_context("spawn").Pool(P) as pool:
            res = pool.map(_ref_worker, jobs)
    t_wall = time.perf_counter() - t_wall
    value = float(sum(r["value"] for r in res))
    N = res[0]["N"]
    steps = min(r["substeps"] for r in res)
    ms_sub = 1e3 * float(np.mean([r["seconds"] / r["substeps"] for r in res]))
    sample = (f"{P} concurrent process(es), one environment each; per process: "
              + _window_sample_text(res[0], N))
    line = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=envs,
                steps=steps, warmup=1, ms_per_step=ms_sub,
                ms_per_rigid_step=ms_sub * N, rigid_steps_per_s=1e3 / (ms_sub * N),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic (seeded jittered lattice)",
                config=dict(workload=workload_name(args.workload, res[0]["n"], N),
                            step_unit=("one SUBSTEP of the window per timed step (a rigid "
                                       f"step is {N} substeps); steps = substeps timed per "
                                       "process"),
                            substeps=N, envs=P, processes=P, wall_s=t_wall,
                            solver_iters_per_substep=[r["iters"] for r in res],
                            contacts_per_substep=[r["contacts"] for r in res]),
                cpu_baseline=dict(value=value, unit=UNIT, cores=P, kind="port",
                                  sample=sample),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for ln in self.path.read_text().splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["no samples"])
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j] == "Active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return dict(sm_mhz=float(statistics.median(loaded)), sm_max_mhz=smax, reasons=reasons,
                    samples=len(rows))


# ------------------------------------------------------------------ ours

def algorithmic_bytes(stage: str, n: int, n_act: int, sand: bool, prof: dict | None = None,
                      precision: str = "f64") -> float:
    """Algorithmic HBM bytes per launch (float64):
    P2G reads x,v (24+24), C,F (72+72), m, V0, material id (8 each) = 216 B
    per particle and writes 7 channels x 8 B = 56 B per active node; G2P reads
    x, F (96) and writes x, v, C, F (192) = 288 B per particle (+16 B plastic
    read+write for sand) and reads v_next (24 B) per active node; the contact
    solve moves 80 B per active node + 128 B per contact per iteration and
    48 B per contact per line-search evaluation.  fp32 mode (float32 v, C, F,
    m, V0, plastic; float64 x and grid): P2G 24 + 12 + 36 + 36 + 4 + 4 + 8 =
    124 B per particle; G2P reads x, F (24 + 36) and writes x, v, C, F
    (24 + 12 + 36 + 36) = 168 B (+8 B plastic)."""
    if precision == "f32" and stage == "p2g":
        return 124.0 * n + 56.0 * n_act
    if precision == "f32" and stage == "g2p":
        return (168.0 + (8.0 if sand else 0.0)) * n + 24.0 * n_act
    if stage == "p2g":
        return 216.0 * n + 56.0 * n_act
    if stage == "g2p":
        return (288.0 + (16.0 if sand else 0.0)) * n + 24.0 * n_act
    if stage == "solve":
        nc = prof["n_contacts"]
        return (80.0 * n_act + 128.0 * nc) * prof["iterations"] + 48.0 * nc * prof["ls_evals"]
    raise ValueError(stage)


def run_ours(args):
    import copy

    import torch

    import paper_2503_05046_b200 as mp
    from paper_2503_05046_b200 import _lib, scenes
    from paper_2503_05046_b200 import distributed as D

    info = D.rank_info()
    world, rank, local = info.world, info.rank, info.local_rank
    torch.cuda.set_device(local)
    D.init("nccl")
    scene = workload_scene(args.workload, rank)
    state = scenes.build_state(scene, precision=args.precision)
    n = state.particles.n
    N = scene["substeps"]
    sand = any(m.get("model") == "sand" for m in scene["materials"])

    # The timed window is the first K steps from t = 0.  Warm-up runs on the
    # same scene and is rolled back (tensors restored in place, bodies re-copied).
    p_keys = ("x", "v", "f", "c", "plastic")
    snap = {k: getattr(state.particles, k).clone() for k in p_keys}
    d3_0 = state.cloth.d3.clone() if state.cloth is not None else None
    bodies0 = copy.deepcopy(state.bodies)

    def restore():
        for k in p_keys:
            getattr(state.particles, k).copy_(snap[k])
        if d3_0 is not None:
            state.cloth.d3.copy_(d3_0)
        state.bodies = copy.deepcopy(bodies0)
        state.time = 0.0
        state.step_index = 0
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        mp.advance_step(state)
    torch.cuda.synchronize()
    restore()
    stream = state._stream

    loaded_snap = {}

    def profiled_step(ncu: bool = False) -> dict:
        """Live per-stage timing of one substep in the middle of the window:
        restore, advance half the window, profile the next step's first
        substep (direct launches, CUDA events on the sim's stream).  The state
        at that substep's start is kept for the CPU oracle's loaded sample."""
        restore()
        for _ in range(args.steps // 2):
            mp.advance_step(state)
        if not ncu:
            loaded_snap.clear()
            loaded_snap.update(state.particles.numpy())
            loaded_snap["bodies"] = [(np.asarray(b.position, float), np.asarray(b.quat, float),
                                      np.asarray(b.v, float), np.asarray(b.omega, float))
                                     for b in state.bodies]
            loaded_snap["time"], loaded_snap["step_index"] = state.time, state.step_index
        prof = {"ncu": ncu}
        mp.advance_step(state, profile=prof)
        return prof

    if args.ncu_window:
        prof = profiled_step(ncu=True)
        if rank == 0:
            print(json.dumps(dict(ncu_window=args.workload, stage_ms=prof["stage_ms"],
                                  iterations=prof["iterations"], ls_evals=prof["ls_evals"],
                                  n_contacts=prof["n_contacts"], n_active=prof["n_active"])))
        D.shutdown()
        return 0

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # ---- timed region: K steps, L2 flushed between steps (outside timing)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    step_ms, sums = [], []
    D.barrier()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
        s = mp.advance_step(state)
        with torch.cuda.stream(stream):
            ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        sums.append(s)
    D.barrier()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    total_ms = D.max_over_ranks(sum(step_ms))  # device time of the job: slowest rank
    ms_per_step = total_ms / args.steps
    n_all = int(D.sum_over_ranks(n))       # every rank runs its own environment
    value = D.job_throughput(n_all * N * args.steps, total_ms * 1e-3)
    first_ms = D.max_over_ranks(step_ms[0])

    # solver work in the window (per rigid step: mean/max over its substeps)
    it_total = int(sum(round(x.iterations_mean * N) for x in sums))
    unconv = int(sum(x.substeps_unconverged for x in sums))
    it_unconv = int(sum(x.iterations_unconverged for x in sums))
    solver_window = dict(
        substeps=N * args.steps, iterations_total=it_total,
        iterations_per_substep_mean=it_total / (N * args.steps),
        iterations_max=int(max(x.iterations_max for x in sums)),
        iterations_mean_per_step=[round(x.iterations_mean, 2) for x in sums],
        iterations_max_per_step=[int(x.iterations_max) for x in sums],
        solves_at_max_iters=unconv, iterations_in_unconverged_solves=it_unconv,
        unconverged_share_of_iterations=(it_unconv / it_total if it_total else 0.0),
        max_iters=state.solver_params.max_iters,
        ls_evals_total=int(sum(x.ls_evals for x in sums)),
        contacts_mean=float(np.mean([x.n_contacts_mean for x in sums])),
        active_nodes_mean=float(np.mean([x.n_active_nodes for x in sums])))

    # ---- live per-stage timing (one profiled substep, direct launches)
    prof = profiled_step()
    st = prof["stage_ms"]
    substep_ms = sum(st.values())
    hbm, peak_src = peaks()
    tf = ROOT / "profiles" / "ncu_traffic.json"
    try:
        traffic_all = json.loads(tf.read_text()).get(args.workload, {}) if tf.exists() else {}
    except Exception:
        traffic_all = {}

    def kernel_roof(stage: str) -> dict:
        abytes = algorithmic_bytes(stage, n, prof["n_active"], sand, prof, args.precision)
        achieved = abytes / (st[stage] * 1e-3) / 1e9
        kname = {"solve": "k_qn_solve", "p2g": "k_p2g", "g2p": "k_g2p"}[stage]
        if stage != "solve":  # the transfer kernels are instantiated per precision
            kname += "<float>" if args.precision == "f32" else "<double>"
        tr = traffic_all.get(kname) or {}
        out = dict(bound="hbm", kernel=kname, achieved=achieved, peak=hbm, unit="GB/s",
                   frac=achieved / hbm, traffic=tr.get("dram_bytes"),
                   algorithmic_bytes=abytes, launch_ms=st[stage],
                   share_of_substep=st[stage] / substep_ms)
        if tr:
            out["ncu"] = {k: v for k, v in tr.items() if k != "dram_bytes"}
            if tr.get("fp64_flop") and tr.get("fp64_peak_tflops"):
                tfl = tr["fp64_flop"] / (st[stage] * 1e-3) / 1e12
                out["fp64"] = dict(achieved_tflops=tfl, peak_tflops=tr["fp64_peak_tflops"],
                                   frac=tfl / tr["fp64_peak_tflops"],
                                   flop_per_launch=tr["fp64_flop"],
                                   note="flops from the ncu capture of the same launch "
                                        "(sass dfma*2 + dmul + dadd), time from this run")
        return out

    dom = max(("solve", "p2g", "g2p"), key=lambda k: st[k])
    roofline = kernel_roof(dom)
    roofline["peak_source"] = peak_src
    if dom == "solve":
        roofline["note"] = ("latency-bound: per iteration two grid barriers and ~12 "
                            "line-search group reductions (DESIGN.md section 3) leave HBM "
                            "mostly idle")
    roofline["secondary"] = {k: kernel_roof(k) for k in ("solve", "p2g", "g2p") if k != dom}
    roofline["stages_ms"] = st
    roofline["profiled_substep"] = (f"substep 0 of window step {args.steps // 2} "
                                    "(direct launches, CUDA events on the sim stream)")
    roofline["solver"] = dict(iterations=prof["iterations"], ls_evals=prof["ls_evals"],
                              contacts=prof["n_contacts"], ms=st["solve"],
                              us_per_iter=(1e3 * st["solve"] / prof["iterations"]
                                           if prof["iterations"] else None))

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        p = state.particles
        keys = ("x", "v", "f", "c", "plastic", "mass", "volume0", "material_id")
        host = {k: torch.empty(getattr(p, k).shape, dtype=getattr(p, k).dtype,
                               pin_memory=True) for k in keys}
        restore()  # host buffers start from the initial state of the window
        for k in keys:
            host[k].copy_(getattr(p, k))
        # the step's inputs are the evolving state; mass, volume0 and
        # material_id never change, so they are uploaded once, before timing
        outs = ("x", "v", "f", "c", "plastic")
        ins = outs
        h2d = sum(host[k].numel() * host[k].element_size() for k in ins)
        d2h = sum(host[k].numel() * host[k].element_size() for k in outs) + 48 * len(state.bodies)
        ke = args.steps
        cur = torch.cuda.current_stream()
        e_ms = 0.0
        restore()
        for k in keys:
            if k not in ins:
                getattr(p, k).copy_(host[k])
        torch.cuda.synchronize()
        D.barrier()
        for _ in range(ke):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(cur)
            for k in ins:
                getattr(p, k).copy_(host[k], non_blocking=True)
            mp.advance_step(state)   # waits on `cur`, syncs its own stream at the end
            for k in outs:
                host[k].copy_(getattr(p, k), non_blocking=True)
            b.record(cur)
            b.synchronize()
            e_ms += a.elapsed_time(b)
        e_ms = D.max_over_ranks(e_ms)
        e2e = dict(value=D.job_throughput(n_all * N * ke, e_ms * 1e-3), unit=UNIT,
                   h2d_bytes_per_step=h2d,
                   d2h_bytes_per_step=d2h, steps=ke, ms_per_step=e_ms / ke,
                   rigid_steps_per_s=1e3 * ke / e_ms,
                   transfers=("each step: H2D of x, v, F, C, plastic from pinned host "
                              "buffers, advance_step, D2H of the same; mass, volume0 and "
                              "material_id (constant) uploaded once before timing"))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_window(scene, 30.0)
        cpu = dict(value=r["value"], unit=UNIT, cores=1, kind="port",
                   sample=_window_sample_text(r, N),
                   gpu_same_prefix=("the GPU arm's first rigid step of the same window: "
                                    f"{first_ms:.2f} ms device time"))
        if loaded_snap and args.workload not in ("cloth", "tshirt"):
            ld = oracle_loaded_substep(scene, loaded_snap)
            gpu_ms = substep_ms
            cpu["loaded_substep"] = dict(
                value=ld["value"], unit=UNIT, seconds=ld["seconds"],
                solver_iterations=ld["iterations"], contacts=ld["contacts"],
                gpu_ms_same_substep=gpu_ms, gpu_solver_iterations=prof["iterations"],
                ratio_gpu_over_cpu=(ld["seconds"] * 1e3) / gpu_ms,
                sample=(f"substep 0 of window step {args.steps // 2} from the GPU state at its "
                        "start (the substep roofline.stages_ms profiles), one thread"))

    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps,
            warmup=args.warmup, ms_per_step=ms_per_step,
            rigid_steps_per_s=1e3 / ms_per_step,
            higher_is_better=True, scaling="weak",
            vs_baseline=None,
            dtype=("f64" if args.precision == "f64" else
                   "f32 particle state/arithmetic; f64 positions, grid, contact solve"),
            data="synthetic (seeded jittered lattice)",
            config=dict(workload=workload_name(args.workload, n, N),
                        precision=args.precision,
                        particles_per_gpu=n, substeps=N, envs=world,
                        parallelism=f"{world} independent envs (1/GPU)",
                        window="the first K rigid steps from t=0 (warm-up rolled back)",
                        l2="flushed (256 MiB write) between timed steps",
                        first_step_ms=first_ms, solver=solver_window),
            roofline=roofline, cpu_baseline=cpu, e2e=e2e, gpu_launches=int(launches),
            clocks=clk)
        print(json.dumps(line), flush=True)
    D.shutdown()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args, argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
