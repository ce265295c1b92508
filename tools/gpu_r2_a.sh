#!/bin/bash
# round 2: parity at the measured configs + convergence of the bench scene variants
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x -s > gpurun_out/r2_pytest_configs.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_configs.log
timeout 600 python tools/diag_converge.py 30 0.2,0.2,0.1 touch3 inside3 > gpurun_out/r2_conv256b.txt 2>&1
timeout 600 python tools/diag_converge.py 30 0.4,0.4,0.1 touch3 > gpurun_out/r2_conv1mb.txt 2>&1
