#!/bin/bash
# fp32 performance mode: GPU tests (fp32 + parity regression), 1M bench in both precisions
mkdir -p gpurun_out
rm -f gpurun_out/fp32_drift.jsonl gpurun_out/parity_configs.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2g_bench_1m.json 2> gpurun_out/r2g_bench_1m.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/r2g_bench_1m_f32.json 2> gpurun_out/r2g_bench_1m_f32.err
tail -3 gpurun_out/r2g_pytest_gpu.log
