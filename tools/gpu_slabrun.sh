#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/slab_run.py --workload sand --steps 2 --warmup 1 > gpurun_out/slab_w1.json 2> gpurun_out/slab_w1.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tools/slab_run.py --workload sand --steps 2 --warmup 1 --backend gloo > gpurun_out/slab_w2.json 2> gpurun_out/slab_w2.err
