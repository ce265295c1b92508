#!/bin/bash
# P2G variants: parity tests of the transfer path + bench lines (256k, 1M)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p2g_bench.json 2> gpurun_out/p2g_bench.err
timeout 600 python bench.py --no-cpu-baseline --workload sand1m > gpurun_out/p2g_bench1m.json 2> gpurun_out/p2g_bench1m.err
