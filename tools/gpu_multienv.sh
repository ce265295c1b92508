#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/me_bench.json 2> /dev/null
for e in 1 2 4; do
  timeout 900 python tools/multi_env.py --envs $e > gpurun_out/me_$e.json 2> gpurun_out/me_$e.err
done
MPMRB_SOLVER_CTAS=74 timeout 900 python tools/multi_env.py --envs 1 > gpurun_out/me_1_74.json 2> gpurun_out/me_1_74.err
