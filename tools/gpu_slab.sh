#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "slab or multi_material or qn_solve" > gpurun_out/pytest_slab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slab.log
