"""Phase-level warp-stall breakdown of one k_qn_solve launch from an ncu
source-level capture (tools/gpu_ncu_solver_src.sh):

    python tools/solver_stalls.py REPORT.ncu-rep SOLVER_CUBIN_SASS

SOLVER_CUBIN_SASS is `nvdisasm --print-line-info` of the solver cubin taken
from the same library build (cuobjdump -xelf all libmpmrb_b200.so).  Every
sampled SASS address is mapped to its solver.cu line and the line to a phase
by the source's own markers."""

import collections
import csv
import re
import subprocess
import sys
from pathlib import Path

SRC = Path(__file__).resolve().parents[1] / "paper_2503_05046_b200" / "csrc" / "solver.cu"


def phases():
    lines = SRC.read_text().split("\n")

    def find(pat, start=0):
        for i in range(start, len(lines)):
            if re.search(pat, lines[i]):
                return i + 1
        raise KeyError(pat)

    k = find(r"k_qn_solve\(SolverArgs a\)")
    marks = [
        ("slot all-reduce polls (slot_poll_sum)", find(r"void slot_poll_sum\("), find(r"^// ---+ grid reductions")),
        ("grid barrier (Sync)", find(r"^struct Sync"), find(r"void block_reduce\(") - 2),
        ("block reductions", find(r"void block_reduce\("), find(r"void reduce_all\(") - 2),
        ("N reduction (reduce_all)", find(r"void reduce_all\("), find(r"void group_reduce\(") - 2),
        ("line-search group reduction", find(r"void group_reduce\("), find(r"void load_frame\(") - 1),
        ("D gather of dv (gather_contact)", find(r"void gather_contact_t\("), find(r"void stage_weights\(")),
        ("weight staging", find(r"void stage_weights\("), find(r"double contact_terms\(")),
        ("contact terms (U)", find(r"double contact_terms\("), find(r"void ls_terms\(")),
        ("line-search contact terms", find(r"void ls_terms\("), find(r"^struct NodeIn")),
        ("node finish (N: Cholesky, dv)", find(r"^struct NodeIn"), find(r"^struct ChunkGroups")),
        ("U chunk: contacts + cellsum", find(r"^struct ChunkGroups"), k),
        ("init", k, find(r"// ---- N:")),
        ("N: gathers of cellsum", find(r"// ---- N:"), find(r"// ---- D:")),
        ("D: direction phase + handoff", find(r"// ---- D:"), find(r"// ---- LS:")),
        ("LS loop (group CTAs)", find(r"// ---- LS:"), find(r"if \(!in_group\) \{")),
        ("alpha broadcast wait (non-group CTAs)", find(r"if \(!in_group\) \{") - 12, find(r"// ---- U:")),
        ("U loop + barrier", find(r"// ---- U:"), find(r"// ---- epilogue")),
        ("epilogue", find(r"// ---- epilogue"), find(r"bool same_stencil\(")),
    ]
    return marks


def main(rep, sass):
    lines = open(sass).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and "k_qn_solve" in l)
    line_of, cur = {}, None
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//---------------------"):
            break
        if "//##" in l:
            m = re.search(r'File "([^"]+)", line (\d+)', l)
            if m:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()[1:]))
    hdr, data = rows[0], rows[1:]
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    marks = phases()
    by = collections.Counter()
    tot = 0
    for r in data:
        s = int(r[isamp] or 0)
        tot += s
        f, ln = line_of.get(int(r[ia], 16) - base, ("?", 0))
        name = "inlined library code (shuffles, rsqrt, ...)" if f != "solver.cu" else "other"
        if f == "solver.cu":
            for nm, a, b in marks:
                if a <= ln < b:
                    name = nm
                    break
        by[name] += s
    print(f"k_qn_solve warp-stall samples by phase ({tot} samples, {Path(rep).name})")
    for nm, s in by.most_common():
        print(f"{100 * s / tot:6.1f}%  {nm}")


if __name__ == "__main__":
    main(*sys.argv[1:])
