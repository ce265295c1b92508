#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r_bench.json 2> /dev/null
timeout 600 python bench.py --no-cpu-baseline --workload sand1m > gpurun_out/r_bench1m.json 2> /dev/null
