#!/bin/bash
# slab decomposition with neighbour-only P2P exchanges: GPU parity (2, 3 ranks
# sharing one GPU over gloo), a functional 2-rank run, and the default bench
# with the contact-loaded CPU sample
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "slab" > gpurun_out/slab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/slab_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   tools/slab_run.py --workload sand --backend gloo --steps 2 --warmup 1 > gpurun_out/slab_run_w2.json 2> gpurun_out/slab_run_w2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
   tools/slab_run.py --workload sand --steps 2 --warmup 1 > gpurun_out/slab_run_w1.json 2> gpurun_out/slab_run_w1.err
timeout 1200 python bench.py > gpurun_out/slab_bench_1m.json 2> gpurun_out/slab_bench_1m.err
