#!/bin/bash
mkdir -p gpurun_out
ONE_SOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qn_solve -c 1 -o gpurun_out/prof_solver python tools/solver_scaling.py 14 0.2 > gpurun_out/prof_solver.log 2>&1
