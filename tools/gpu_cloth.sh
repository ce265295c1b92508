#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload cloth --no-cpu-baseline --steps 10 > gpurun_out/bench_cloth.json 2> gpurun_out/bench_cloth.err
timeout 900 python bench.py --workload tshirt --no-cpu-baseline --steps 10 > gpurun_out/bench_tshirt.json 2> gpurun_out/bench_tshirt.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_p2g|k_g2p|k_qn_solve' -s 100 -c 3 \
   -o gpurun_out/prof_sand_v5 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/prof_sand_v5.log 2>&1
