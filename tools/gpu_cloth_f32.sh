# fp32 mode with cloth: the fp32 tests, the cloth parity tests, and the cloth
# and T-shirt bench lines in both precisions
mkdir -p gpurun_out
rm -f gpurun_out/fp32_drift.jsonl
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x > gpurun_out/cf_pytest_fp32.log 2>&1; echo "rc=$?" >> gpurun_out/cf_pytest_fp32.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k cloth > gpurun_out/cf_pytest_cloth.log 2>&1; echo "rc=$?" >> gpurun_out/cf_pytest_cloth.log
for prec in f64 f32; do
  timeout 600 python bench.py --workload cloth --precision $prec --no-cpu-baseline > gpurun_out/cf_bench_cloth_$prec.json 2> gpurun_out/cf_bench_cloth_$prec.err
  timeout 600 python bench.py --workload tshirt --precision $prec --no-cpu-baseline > gpurun_out/cf_bench_tshirt_$prec.json 2> gpurun_out/cf_bench_tshirt_$prec.err
done
