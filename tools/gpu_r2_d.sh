#!/bin/bash
# round 2 evidence: launch list + ncu full capture of the profiled substep at
# 1M (roofline.traffic, fp64 flops), compute-sanitizer on the multi-CTA solve
# and the fused step, secondary workloads' bench lines.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 50000 --csv \
   --log-file gpurun_out/r2_launches_1m.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/r2_launches_1m.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:'k_p2g|k_g2p|k_qn_solve' -o gpurun_out/r2_prof_1m python bench.py --ncu-window --steps 20 \
   > gpurun_out/r2_prof_1m.log 2>&1
python tools/summarize_evidence.py gpurun_out/r2_launches_1m.csv gpurun_out/r2_prof_1m.ncu-rep sand1m_v1 sand1m r02 \
   "python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e" > gpurun_out/r2_summarize.log 2>&1
cp profiles/r02_* profiles/ncu_traffic.json gpurun_out/ 2>/dev/null
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --launch-timeout 600 python -m pytest tests/test_gpu_parity.py -q -x \
     -k "qn_solve_matches_reference and 3-1 or steps_match_reference" > gpurun_out/r2_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_sanitizer_$tool.log
done
timeout 900 python bench.py --workload sand --no-cpu-baseline > gpurun_out/r2_bench_256k.json 2> gpurun_out/r2_bench_256k.err
timeout 900 python bench.py --workload cloth --no-cpu-baseline > gpurun_out/r2_bench_cloth.json 2> gpurun_out/r2_bench_cloth.err
timeout 900 python bench.py --workload tshirt --no-cpu-baseline > gpurun_out/r2_bench_tshirt.json 2> gpurun_out/r2_bench_tshirt.err
timeout 900 python bench.py --workload multi4m --steps 5 --no-cpu-baseline > gpurun_out/r2_bench_multi4m.json 2> gpurun_out/r2_bench_multi4m.err
ls -la gpurun_out | tail -40
