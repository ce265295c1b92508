#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_p2g -s 40 -c 1 -o gpurun_out/prof_p2g python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_p2g.log 2>&1
timeout 600 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_durations.log 2>&1
