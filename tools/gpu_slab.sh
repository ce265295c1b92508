mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k slab > gpurun_out/slab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/slab_pytest.log
for s in gather0 allreduce; do
timeout 300 python tools/slab_run.py --workload sand --steps 2 --warmup 1 --solve $s > gpurun_out/slab_w1_$s.json 2> gpurun_out/slab_w1_$s.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/slab_run.py --workload sand --steps 2 --warmup 1 --backend gloo --solve $s > gpurun_out/slab_w2_$s.json 2> gpurun_out/slab_w2_$s.err
done
