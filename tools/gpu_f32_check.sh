# fp32 tests + the fp32 bench line (after an fp32 kernel change)
mkdir -p gpurun_out
rm -f gpurun_out/fp32_drift.jsonl
timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_tiles.py -q > gpurun_out/f32c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f32c_pytest.log
timeout 900 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/f32c_bench_1m_f32.json 2> gpurun_out/f32c_bench_1m_f32.err
