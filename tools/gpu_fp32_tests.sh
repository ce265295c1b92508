mkdir -p gpurun_out
rm -f gpurun_out/fp32_drift.jsonl
timeout 900 python -m pytest tests/test_gpu_fp32.py -q > gpurun_out/cf_pytest_fp32.log 2>&1; echo "rc=$?" >> gpurun_out/cf_pytest_fp32.log
