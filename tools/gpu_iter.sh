#!/bin/bash
# One build -> measure iteration: GPU tests, solver timing, bench lines and an
# ncu full capture of the three top kernels in the contact-loaded window.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.2 > gpurun_out/it_ss256.txt 2>&1
REPS=3 MPMRB_SOLVER_PROF=1 CTAS_LIST=0 timeout 300 python tools/solver_scaling.py 14 0.4 > gpurun_out/it_ss2m.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
timeout 600 python bench.py --no-cpu-baseline --workload sand1m > gpurun_out/it_bench1m.json 2> gpurun_out/it_bench1m.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_p2g|k_g2p|k_qn_solve' -s 450 -c 3 \
   -o gpurun_out/prof_it python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/prof_it.log 2>&1
