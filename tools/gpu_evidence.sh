#!/bin/bash
# Evidence on the committed tree: full GPU suite, smoke, default bench
# (1M f64) + reference arm, f32 line, secondary workloads, launch list + ncu
# full capture of the profiled 1M substep, sanitizers, solver phase profile.
#   gpurun --timeout 5400 -- 'bash tools/gpu_evidence.sh'
# then, in this container:
#   python tools/summarize_evidence.py gpurun_out/ev_launches_1m.csv \
#       gpurun_out/ev_prof_1m.ncu-rep sand1m_final sand1m r02 "<bench command>"
# and copy gpurun_out/ev_* into profiles/r02_*.
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl gpurun_out/fp32_drift.jsonl
nvidia-smi > gpurun_out/ev_nvidia_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/ev_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench_1m.json 2> gpurun_out/ev_bench_1m.err
timeout 600 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/ev_bench_1m_f32.json 2> gpurun_out/ev_bench_1m_f32.err
timeout 900 python bench.py --workload sand --no-cpu-baseline > gpurun_out/ev_bench_256k.json 2> gpurun_out/ev_bench_256k.err
timeout 900 python bench.py --workload cloth --no-cpu-baseline > gpurun_out/ev_bench_cloth.json 2> gpurun_out/ev_bench_cloth.err
timeout 900 python bench.py --workload tshirt --no-cpu-baseline > gpurun_out/ev_bench_tshirt.json 2> gpurun_out/ev_bench_tshirt.err
timeout 900 python bench.py --workload multi4m --steps 5 --no-cpu-baseline > gpurun_out/ev_bench_multi4m.json 2> gpurun_out/ev_bench_multi4m.err
timeout 900 python bench.py --workload cube --no-cpu-baseline > gpurun_out/ev_bench_cube.json 2> gpurun_out/ev_bench_cube.err
MPMRB_SOLVER_PROF=1 timeout 600 python tools/solver_scaling.py 10 0.4 0.1 0 > gpurun_out/ev_solver_prof_1m.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 50000 --csv \
   --log-file gpurun_out/ev_launches_1m.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/ev_launches_1m.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:'k_p2g|k_g2p|k_qn_solve' -o gpurun_out/ev_prof_1m python bench.py --ncu-window --steps 20 \
   > gpurun_out/ev_prof_1m.log 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --launch-timeout 600 python -m pytest tests/test_gpu_parity.py -q -x \
     -k "qn_solve_matches_reference or steps_match_reference or p2g_grid_update" > gpurun_out/ev_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/ev_sanitizer_$tool.log
done
ls -la gpurun_out | tail -50
