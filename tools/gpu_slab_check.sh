mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k slab > gpurun_out/slab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/slab_pytest.log
rm -f gpurun_out/slab_w1_window.jsonl
bash tools/gpu_slab_w1.sh
