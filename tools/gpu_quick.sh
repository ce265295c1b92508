mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
for r in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench_$r.json 2>/dev/null; done
timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-e2e > gpurun_out/q_bench_f32.json 2>/dev/null
