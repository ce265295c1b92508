#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "concurrent or smoke or steps_match" > gpurun_out/pytest_conc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conc.log
