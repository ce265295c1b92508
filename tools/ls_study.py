"""Line-search round counting on real contact problems (CPU oracle).

    python tools/ls_study.py [half_x] [steps]

Runs the oracle on a sand pile pushed by the kinematic box, records every line
search's sequence of steps (Newton / bisection / expansion, solver.py:276-298)
and prints the evaluations per search and the number of group-reduction rounds
the device solver needs when each round also evaluates the two possible
non-Newton successors of its point (csrc/solver.cu, line search): a point
reached by bisection or expansion from a round's point is already summed.
Test/analysis infrastructure only (imports the oracle)."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import solver as osv, step as ostep  # noqa: E402
from paper_2503_05046_b200 import scenes as S  # noqa: E402
from scenes import oracle_state  # noqa: E402

stats = dict(calls=0, evals=0, newton=0, bisect=0, expand=0, rounds_plain=0, rounds_spec=0)


def traced_line_search(deriv, max_evals=50, tol=1e-8):
    d0, _ = deriv(0.0)
    lo, hi, a, d = 0.0, np.inf, 1.0, d0
    kinds = []
    stats["calls"] += 1
    for ev in range(1, max_evals + 1):
        d, dd = deriv(a)
        stats["evals"] += 1
        if abs(d) <= tol * abs(d0):
            break
        if d > 0.0:
            hi = a
        else:
            lo = a
        nxt = a - d / dd if (np.isfinite(dd) and dd > 0.0) else np.nan
        if np.isfinite(hi):
            if not np.isfinite(nxt) or not (lo < nxt < hi):
                nxt, k = 0.5 * (lo + hi), "b"
            else:
                k = "n"
        elif not np.isfinite(nxt) or nxt <= lo:
            nxt, k = 2.0 * max(a, 1e-8), "e"
        else:
            k = "n"
        kinds.append(k)
        a = nxt
    for k in kinds:
        stats[{"n": "newton", "b": "bisect", "e": "expand"}[k]] += 1
    # rounds after the first point (which the direction phase sums)
    stats["rounds_plain"] += len(kinds)
    main, rounds = True, 0
    for k in kinds:
        if main and k in "be":
            main = False  # summed speculatively with the previous point
        else:
            main, rounds = True, rounds + 1
    stats["rounds_spec"] += rounds
    if abs(d) <= tol * abs(d0):
        return a, len(kinds) + 1, d
    return (lo if lo > 0.0 else a), max_evals, d


def main(hx=0.1, steps=14):
    osv.exact_line_search = traced_line_search
    sc = S.sand_pile_scene(half=(hx, hx, hx / 2))
    a = S.host_particles(sc)
    st = oracle_state(sc, a["x"], a["v"], a["f"], a["c"], a["mass"], a["vol"], a["mid"])
    for _ in range(steps):
        ostep.step(st)
    c = max(stats["calls"], 1)
    print(f"{a['x'].shape[0]} particles, {stats['calls']} line searches: "
          f"{stats['evals'] / c:.2f} evaluations/search "
          f"(newton {stats['newton']}, bisection {stats['bisect']}, expansion {stats['expand']}); "
          f"reduction rounds/search: {stats['rounds_plain'] / c:.2f} plain, "
          f"{stats['rounds_spec'] / c:.2f} with speculative successors")


if __name__ == "__main__":
    main(*(float(x) if i == 0 else int(x) for i, x in enumerate(sys.argv[1:])))
