#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "p2g or steps_match or fused or multi_material" > gpurun_out/pytest_p2g3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2g3.log
bash tools/gpu_ab3.sh main u1
