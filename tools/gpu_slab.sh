# slab decomposition on one B200: GPU parity tests (ranks share cuda:0 over
# gloo) and slab_run timings of both substep paths and both solve modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k slab > gpurun_out/slab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/slab_pytest.log
for sub in "" "--ops"; do
for s in gather0 allreduce; do
tag=$s${sub:+_ops}
timeout 300 python tools/slab_run.py --workload sand --steps 2 --warmup 1 --solve $s $sub > gpurun_out/slab_w1_$tag.json 2> gpurun_out/slab_w1_$tag.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/slab_run.py --workload sand --steps 2 --warmup 1 --backend gloo --solve $s $sub > gpurun_out/slab_w2_$tag.json 2> gpurun_out/slab_w2_$tag.err
done
done
