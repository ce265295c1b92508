#!/bin/bash
mkdir -p gpurun_out
MPMRB_SOLVER_CTAS=50 timeout 900 python tools/multi_env.py --envs 2 > gpurun_out/me2_2_50.json 2> /dev/null
MPMRB_SOLVER_CTAS=49 timeout 900 python tools/multi_env.py --envs 3 > gpurun_out/me2_3_49.json 2> /dev/null
MPMRB_SOLVER_CTAS=30 timeout 900 python tools/multi_env.py --envs 4 > gpurun_out/me2_4_30.json 2> /dev/null
MPMRB_SOLVER_CTAS=37 timeout 900 python tools/multi_env.py --envs 4 > gpurun_out/me2_4_37.json 2> /dev/null
MPMRB_SOLVER_CTAS=18 timeout 900 python tools/multi_env.py --envs 8 > gpurun_out/me2_8_18.json 2> /dev/null
MPMRB_SOLVER_CTAS=24 timeout 900 python tools/multi_env.py --envs 6 > gpurun_out/me2_6_24.json 2> /dev/null
