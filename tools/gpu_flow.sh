#!/bin/bash
# NOTE: the dataflow variant this script A/B-tested was measured slower and removed;
# the results are in profiles/r01_solver_flow_ab_*.txt and DESIGN.md section 2.
# A/B of the dataflow solver iteration (MPMRB_SOLVER_FLOW=1, default) against
# the barrier iteration (=0): parity tests, solver timing, bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for F in 1 0; do
  MPMRB_SOLVER_FLOW=$F REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/ss256_f$F.txt 2>&1
  MPMRB_SOLVER_FLOW=$F REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/ss2m_f$F.txt 2>&1
  MPMRB_SOLVER_FLOW=$F timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_f$F.json 2> gpurun_out/bench_f$F.err
  MPMRB_SOLVER_FLOW=$F timeout 600 python bench.py --no-cpu-baseline --workload sand1m --steps 20 > gpurun_out/bench1m_f$F.json 2> gpurun_out/bench1m_f$F.err
done
