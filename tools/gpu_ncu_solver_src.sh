#!/bin/bash
# Source-level ncu capture of one contact solve at 2M particles (stall sampling
# per CUDA source line; the library is built with -lineinfo).
mkdir -p gpurun_out
REPS=1 CTAS_LIST=0 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:k_qn_solve -s 140 -c 1 -o gpurun_out/prof_solver2m \
  python tools/solver_scaling.py 14 0.4 > gpurun_out/prof_solver2m.log 2>&1
