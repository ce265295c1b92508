#!/bin/bash
# solver iteration: GPU tests, 1M bench (device line), in-kernel phase profile at 1M
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_1m.json 2> gpurun_out/r2e_bench_1m.err
MPMRB_SOLVER_PROF=1 timeout 600 python tools/solver_scaling.py 10 0.4 0.1 0 > gpurun_out/r2e_solver_prof_1m.txt 2>&1
tail -3 gpurun_out/r2e_pytest_gpu.log
