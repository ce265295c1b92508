#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "p2g or g2p or steps_match or fused" > gpurun_out/pytest_q2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q2.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q2_bench.json 2> /dev/null
timeout 600 python bench.py --no-cpu-baseline --workload sand1m > gpurun_out/q2_bench1m.json 2> /dev/null
