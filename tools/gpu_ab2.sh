#!/bin/bash
# Interleaved A/B of the solver timing (tools/solver_scaling.py) between the
# default build and variants: main, v1, main, v1 ...
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "qn_solve or steps_match or fused" > gpurun_out/pytest_ab2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab2.log
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then lp=paper_2503_05046_b200/_native/libmpmrb_b200.so; else lp=paper_2503_05046_b200/_native/variants/$v.so; fi
  MPMRB_LIB_PATH=$lp REPS=5 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/ab2_ss256_${v}_$rep.txt 2>&1
  MPMRB_LIB_PATH=$lp REPS=5 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/ab2_ss2m_${v}_$rep.txt 2>&1
done
done
