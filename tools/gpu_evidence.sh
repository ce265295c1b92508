#!/bin/bash
# Round evidence: tests, smoke, full bench (with CPU baseline), reference arm,
# launch list of the bench command and ncu full captures of the top kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload sand1m --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err
timeout 900 python bench.py --workload cloth --no-cpu-baseline > gpurun_out/bench_cloth.json 2> gpurun_out/bench_cloth.err
timeout 900 python bench.py --workload tshirt --no-cpu-baseline > gpurun_out/bench_tshirt.json 2> gpurun_out/bench_tshirt.err
timeout 900 python bench.py --workload multi4m --steps 5 --no-cpu-baseline > gpurun_out/bench_multi4m.json 2> gpurun_out/bench_multi4m.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/launches_bench.log 2>&1
# skip into the contact-loaded window (the pusher reaches the pile after ~12 steps)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_p2g|k_g2p|k_qn_solve' -s 450 -c 3 \
   -o gpurun_out/prof_sand python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/prof_sand.log 2>&1
python tools/summarize_evidence.py gpurun_out/launches.csv gpurun_out/prof_sand.ncu-rep sand_final > gpurun_out/summarize.log 2>&1
ls -la gpurun_out
