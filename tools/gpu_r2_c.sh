#!/bin/bash
# round 2 re-entry check: GPU suite, smoke, default bench (1M), reference arm
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
tools/bin/fp_peak > gpurun_out/fp_peak.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench_1m.json 2> gpurun_out/r2_bench_1m.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
tail -3 gpurun_out/r2_pytest_gpu.log gpurun_out/r2_smoke.log
