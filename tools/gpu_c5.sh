#!/bin/bash
# configs[4] on one GPU: the multi-material parity test and a bench line.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "multi_material" > gpurun_out/pytest_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5.log
timeout 900 python bench.py --workload multi4m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_multi4m.json 2> gpurun_out/bench_multi4m.err
