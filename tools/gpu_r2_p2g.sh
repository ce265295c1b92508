#!/bin/bash
# P2G iteration: GPU suite, 1M bench (f64 twice, f32), ncu full capture of the
# profiled substep's k_p2g / k_g2p
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/p2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p2g_pytest.log
for r in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/p2g_bench_1m_$r.json 2> gpurun_out/p2g_bench_1m_$r.err
done
timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-e2e > gpurun_out/p2g_bench_1m_f32.json 2> gpurun_out/p2g_bench_1m_f32.err
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:'k_p2g|k_g2p' -o gpurun_out/p2g_prof_1m python bench.py --ncu-window --steps 20 \
   > gpurun_out/p2g_prof_1m.log 2>&1
