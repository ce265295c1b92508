# the all-reduce line search: its GPU slab tests and one timing at 256k
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "slab and allreduce" > gpurun_out/ar_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ar_pytest.log
timeout 300 python tools/slab_run.py --workload sand --steps 2 --warmup 1 --solve allreduce > gpurun_out/ar_w1.json 2>/dev/null
