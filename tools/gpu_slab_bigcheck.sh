# slab decomposition at bench size (256k sand) vs the undecomposed fused step
mkdir -p gpurun_out
rm -f gpurun_out/slab_check.jsonl
timeout 600 python tools/slab_check.py --steps 3 >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_w1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
   tools/slab_check.py --steps 3 >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_w2.err
