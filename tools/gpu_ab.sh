#!/bin/bash
# A/B of library variants (tools/build_variant.sh): solver timing at 256k / 2M
# and bench lines.  Usage: tools/gpu_ab.sh variant1 variant2 ...  ("main" = the
# default build)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "multi_material" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in "$@"; do
  if [ "$v" = main ]; then lp=paper_2503_05046_b200/_native/libmpmrb_b200.so; else lp=paper_2503_05046_b200/_native/variants/$v.so; fi
  MPMRB_LIB_PATH=$lp REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/ab_ss256_$v.txt 2>&1
  MPMRB_LIB_PATH=$lp REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/ab_ss2m_$v.txt 2>&1
  MPMRB_LIB_PATH=$lp timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
  MPMRB_LIB_PATH=$lp timeout 600 python bench.py --no-cpu-baseline --no-e2e --workload sand1m --steps 10 > gpurun_out/ab_bench1m_$v.json 2> gpurun_out/ab_bench1m_$v.err
done
