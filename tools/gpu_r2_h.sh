#!/bin/bash
# transfer-kernel iteration: parity subset + 1M bench in both precisions
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_fp32.py -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_1m.json 2> gpurun_out/r2h_bench_1m.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_1m_f32.json 2> gpurun_out/r2h_bench_1m_f32.err
