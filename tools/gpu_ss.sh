#!/bin/bash
mkdir -p gpurun_out
REPS=2 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/ss_chk256.txt 2>&1
REPS=2 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.05 > gpurun_out/ss_chk4k.txt 2>&1
