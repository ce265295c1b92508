#!/bin/bash
# quick solver perf iteration: in-kernel phase profile at 1M + 1M bench device line
mkdir -p gpurun_out
MPMRB_SOLVER_PROF=1 timeout 600 python tools/solver_scaling.py 10 0.4 0.1 0 > gpurun_out/r2f_solver_prof_1m.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2f_bench_1m.json 2> gpurun_out/r2f_bench_1m.err
