#!/bin/bash
mkdir -p gpurun_out tools/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/barrier_bench tools/barrier_bench.cu
timeout 120 tools/bin/barrier_bench > gpurun_out/barrier_bench.txt 2>&1
MPMRB_SOLVER_PROF=1 CTAS_LIST=148,0 timeout 600 python tools/solver_scaling.py 14 0.2 > gpurun_out/solver_scaling_256k.txt 2>&1
MPMRB_SOLVER_PROF=1 CTAS_LIST=148,0 timeout 600 python tools/solver_scaling.py 14 0.4 > gpurun_out/solver_scaling_1m.txt 2>&1
