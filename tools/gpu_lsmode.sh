#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for m in 0 1 2; do
  MPMRB_LS_MODE=$m REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/lsm_2m_${m}_$rep.txt 2>&1
  MPMRB_LS_MODE=$m REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.28 > gpurun_out/lsm_1m_${m}_$rep.txt 2>&1
done
done
