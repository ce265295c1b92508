#!/bin/bash
# round 2: convergence study of the sand workload (256k and 1M) + GPU tests
mkdir -p gpurun_out
timeout 900 python tools/diag_converge.py 30 0.2,0.2,0.1 base epsv1e-3 pmu0 raised inside inside_raised slow k1e4 > gpurun_out/r2_conv256.txt 2>&1
timeout 600 python tools/diag_converge.py 25 0.4,0.4,0.1 base inside epsv1e-3 > gpurun_out/r2_conv1m.txt 2>&1
