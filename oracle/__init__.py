"""CPU oracle for the convex MPM–rigid coupling substep (TEST INFRASTRUCTURE ONLY).

This package is a float64 NumPy restatement of the reference algorithm
(`/root/reference/pkg/src/mpmrb`), written from the reference's behaviour and
its tests, not copied from it.  Every function cites the reference file:line it
follows.  It exists for exactly three callers:

* ``tests/``                      — parity checker for the CUDA path,
* ``__graft_entry__.smoke()``      — checks one tiny CUDA substep,
* ``bench.py`` (``cpu_baseline`` leg and ``--impl reference``) — timed CPU port.

The product package ``paper_2503_05046_b200`` never imports this package and has
no CPU fallback; if its CUDA library is missing it raises.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``,
run in the build container where ``/root/reference`` is importable), and against
the reference tests' own known-answer values.  The Drucker–Prager return map in
``oracle.plasticity`` has no reference implementation: PARITY UNPINNED there
(pinned only by its own analytic KATs).
"""

from . import grid, mpm, sdf, contact, solver, step, plasticity  # noqa: F401
