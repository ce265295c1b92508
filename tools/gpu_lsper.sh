#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "qn_solve or steps_match or fused" > gpurun_out/pytest_lsper.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lsper.log
for rep in 1 2; do
for m in 4 6 8; do
  MPMRB_LS_PER_THREAD=$m REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/lsp_2m_${m}_$rep.txt 2>&1
  MPMRB_LS_PER_THREAD=$m REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.28 > gpurun_out/lsp_1m_${m}_$rep.txt 2>&1
  MPMRB_LS_PER_THREAD=$m REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/lsp_256_${m}_$rep.txt 2>&1
done
done
