"""Summarise the round's GPU evidence for profiles/:

    python tools/summarize_evidence.py LAUNCHES.csv NCU.ncu-rep TAG [WORKLOAD] [ROUND] [CMD]

* the ncu launch list (`--metrics gpu__time_duration.sum`) -> per-kernel
  launches, total device time, share and us/launch;
* the `ncu --set full` capture -> per-kernel duration, DRAM bytes, achieved
  DRAM GB/s, L2 hit rate, occupancy and registers, and profiles/ncu_traffic.json
  (dram bytes per launch, read by bench.py as roofline.traffic)."""

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^.*::", "", name)
    return name


def launches(path: Path, cmd: str) -> str:
    rows = [r for r in csv.reader(ln for ln in path.read_text().splitlines() if ln.startswith('"'))]
    hdr, unit, data = rows[0], rows[1], rows[2:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit[iv] or "nsecond", 1e-6)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in data:
        k = short(r[ik])
        tot[k] += float(r[iv].replace(",", "")) * scale
        cnt[k] += 1
    total = sum(tot.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
           f"command: {cmd}",
           f"{sum(cnt.values())} launches, {total:.3f} ms total device time",
           f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'us/launch':>10s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{k[:40]:40s} {cnt[k]:8d} {tot[k]:10.3f} {100 * tot[k] / total:6.2f}% "
                   f"{1e3 * tot[k] / cnt[k]:10.2f}")
    return "\n".join(out) + "\n"


def full(path: Path):
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name, default=None):
        i = col.get(name)
        if i is None or r[i] == "":
            return default
        try:
            return float(r[i].replace(",", ""))
        except ValueError:
            return r[i]

    def bytes_of(r, name):
        v = get(r, name, 0.0)
        u = unit[col[name]] if name in col else "byte"
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    def dur_us(r):
        v = get(r, "gpu__time_duration.sum", 0.0)
        u = unit[col["gpu__time_duration.sum"]]
        return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)

    lines = [f"{'kernel':14s} {'grid':>10s} {'dur us':>9s} {'DRAM MB':>9s} {'DRAM GB/s':>10s} "
             f"{'L2 hit%':>8s} {'occup%':>7s} {'regs':>5s}"]
    traffic = {}
    for r in data:
        k = short(r[col["Kernel Name"]])
        d = dur_us(r)
        b = bytes_of(r, "dram__bytes_read.sum") + bytes_of(r, "dram__bytes_write.sum")
        l2 = get(r, "lts__t_sector_hit_rate.pct", 0.0)
        occ = get(r, "sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)
        regs = get(r, "launch__registers_per_thread", 0.0)
        grid = r[col["Grid Size"]]
        lines.append(f"{k:14s} {grid:>10s} {d:9.2f} {b / 1e6:9.2f} {b / d / 1e3 if d else 0:10.1f} "
                     f"{l2:8.2f} {occ:7.2f} {regs:5.0f}")
        # FP64 work: thread instructions per elapsed cycle (summed over SMSPs)
        # x elapsed cycles; flops count a DFMA as 2.  The pipe fraction is the
        # FP64 compute roofline (DFMA, DMUL and DADD each take an issue slot).
        cyc = get(r, "sm__cycles_elapsed.avg", 0.0) or get(r, "gpc__cycles_elapsed.max", 0.0)
        rate = {op: get(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed", 0.0)
                for op in ("dfma", "dmul", "dadd")}
        fl = (2.0 * rate["dfma"] + rate["dmul"] + rate["dadd"]) * cyc
        pipe = get(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", None)
        traffic[k] = dict(dram_bytes=b, fp64_flop=fl or None, fp64_pipe_pct_of_peak=pipe,
                          cold_duration_us=d, l2_hit_pct=l2, occupancy_pct=occ, registers=regs)
        lines[-1] += f"  fp64 GFLOP {fl / 1e9:8.3f}  fp64 pipe {pipe or 0:5.1f}% of peak"
    return "\n".join(lines) + "\n", traffic


def main(launch_csv, ncu_rep, tag, workload="sand1m", rnd="r02",
         cmd="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"):
    prof = ROOT / "profiles"
    if launch_csv != "-":
        (prof / f"{rnd}_launches_{tag}_summary.txt").write_text(
            launches(Path(launch_csv), f"{cmd}  (workload {workload})"))
    if ncu_rep != "-":
        txt, traffic = full(Path(ncu_rep))
        (prof / f"{rnd}_ncu_{tag}_summary.txt").write_text(
            f"ncu --set full --clock-control none ({Path(ncu_rep).name}; one launch each, "
            "the profiled substep of bench.py --ncu-window)\n" + txt)
        peak = None
        pf = prof / "fp_peak.json"
        if pf.exists():
            peak = json.loads(pf.read_text()).get("fp64_fma_tflops")
        tf = prof / "ncu_traffic.json"
        d = json.loads(tf.read_text()) if tf.exists() else {}
        d["_note"] = ("per launch, from ncu --set full of the SAME profiled substep bench.py "
                      "times (bench.py --ncu-window, ncu --profile-from-start off): dram_bytes = "
                      "dram__bytes_read.sum + dram__bytes_write.sum (roofline.traffic); fp64_flop "
                      "= 2 dfma + dmul + dadd thread instructions; fp64_peak_tflops from "
                      "profiles/fp_peak.json (tools/fp_peak.cu)")
        d[workload] = {k: dict(v, fp64_peak_tflops=peak) for k, v in traffic.items()}
        tf.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
