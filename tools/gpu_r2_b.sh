#!/bin/bash
# round 2 evidence: fp peaks, parity at the measured configs, the default bench
# (1M sand), the reference arm, configs[1], launch list + ncu full capture of
# the profiled substep.
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
tools/bin/fp_peak > gpurun_out/fp_peak.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -s > gpurun_out/r2_pytest_configs.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_configs.log
timeout 900 python bench.py > gpurun_out/r2_bench_1m.json 2> gpurun_out/r2_bench_1m.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
timeout 900 python bench.py --workload sand --no-cpu-baseline > gpurun_out/r2_bench_256k.json 2> gpurun_out/r2_bench_256k.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 50000 --csv \
   --log-file gpurun_out/r2_launches_1m.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/r2_launches_1m.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:'k_p2g|k_g2p|k_qn_solve' -o gpurun_out/r2_prof_1m python bench.py --ncu-window --steps 20 \
   > gpurun_out/r2_prof_1m.log 2>&1
ls -la gpurun_out | tail -30
