#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_ab3.sh main shfl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_p2g -s 150 -c 1 -o gpurun_out/prof_p2g_slot python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_p2g_slot.log 2>&1
