#!/bin/bash
# One GPU session: parity tests, smoke, bench, launch list and ncu captures.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload sand1m --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/launches_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_p2g|k_g2p|k_qn_solve' -s 30 -c 3 \
   -o gpurun_out/prof_sand python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/prof_sand.log 2>&1
ls -la gpurun_out
