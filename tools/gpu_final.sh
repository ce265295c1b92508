# Re-check of the committed tree after a host-side change: full GPU suite,
# smoke, the default bench line, the reference arm and the fp32 line.
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl gpurun_out/fp32_drift.jsonl
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fin_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/fin_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench_1m.json 2> gpurun_out/fin_bench_1m.err
timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/fin_bench_1m_f32.json 2> gpurun_out/fin_bench_1m_f32.err
