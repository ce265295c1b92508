# full GPU suite + smoke on the current tree
mkdir -p gpurun_out
rm -f gpurun_out/parity_configs.jsonl gpurun_out/fp32_drift.jsonl
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/suite_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/suite_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/suite_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/suite_smoke.log
