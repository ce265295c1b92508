"""Committed SASS evidence for the sm_100a kernels (north_star: "each kernel is
justified by ... a committed SASS listing").

    python tools/sass_listing.py [out_dir]     # default profiles/sass

Disassembles the built C-ABI library with cuobjdump, writes the listing of
each hot kernel (encodings stripped) and a summary with register / shared
memory use and the instruction mix that matters for this path: float64 math
(DFMA/DADD/DMUL), global loads/stores and reductions (LDG/STG/REDG/ATOMG),
shared memory (LDS/STS), shuffles, barriers and local-memory traffic
(LDL/STL: stack frame and spills)."""

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2503_05046_b200" / "_native" / "libmpmrb_b200.so"
HOT = ("k_p2g", "k_g2p", "k_qn_solve", "k_grid_update", "k_contact_emit", "k_sort_keys",
       "k_reactions", "k_cloth_forces", "k_contact_prepare")
CLASSES = ("DFMA", "DADD", "DMUL", "MUFU", "LDG", "STG", "REDG", "ATOMG", "ATOMS", "LDS", "STS",
           "SHFL", "BAR", "LDL", "STL", "BRA")


def short(mangled: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+?)(?:I|E|$)", mangled.split("_cu_")[-1] if "_cu_" in mangled
                  else mangled)
    name = m.group(1) if m else mangled
    name = re.sub(r"^\d+", "", name)
    tail = mangled.split(name, 1)[-1] if name in mangled else ""
    if tail.startswith("IdE"):
        name += "<double>"
    elif tail.startswith("IfE"):
        name += "<float>"
    return name


def main(out_dir: str = "profiles/sass") -> None:
    out = ROOT / out_dir
    out.mkdir(parents=True, exist_ok=True)
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                          check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True,
                         text=True, check=True).stdout
    usage = {}
    cur = None
    for ln in res.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", ln)
        if m and cur:
            usage[cur] = tuple(int(x) for x in m.groups())
    funcs = re.split(r"\n\s*Function : ", sass)
    rows = []
    for blk in funcs[1:]:
        mangled = blk.split("\n", 1)[0].strip()
        name = short(re.sub(r"^_ZN5mpmrb\d+_GLOBAL__N__[0-9a-f]+_\d+_", "", mangled))
        body = []
        mix = collections.Counter()
        for ln in blk.split("\n")[1:]:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if not m:
                continue
            ins = m.group(2).strip()
            body.append(f"/*{m.group(1)}*/ {ins}")
            op = re.sub(r"^@!?U?P\w+\s+", "", ins).split()[0]
            base = op.split(".")[0]
            for c in CLASSES:
                if base == c:
                    mix[c] += 1
            mix["total"] += 1
        reg, stack, shared = usage.get(mangled, (None, None, None))
        rows.append((name, mangled, reg, stack, shared, mix))
        if any(name == h or name.startswith(h + "I") or name.startswith(h + "<") for h in HOT):
            fname = name.replace("<", "_").replace(">", "")
            (out / f"{fname}.sass").write_text(
                f"// {mangled}\n// sm_100a, from {LIB.name} (cuobjdump -sass, encodings stripped)\n"
                + "\n".join(body) + "\n")
    lines = ["# SASS summary (sm_100a): registers, stack / shared bytes, instruction mix",
             f"# source: cuobjdump -sass / -res-usage of {LIB.name}", "",
             "kernel | REG | STACK | SHARED | total | " + " | ".join(CLASSES)]
    for name, _, reg, stack, shared, mix in sorted(rows, key=lambda r: -r[5]["total"]):
        lines.append(f"{name} | {reg} | {stack} | {shared} | {mix['total']} | "
                     + " | ".join(str(mix[c]) for c in CLASSES))
    (out / "summary.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


if __name__ == "__main__":
    main(*sys.argv[1:])
