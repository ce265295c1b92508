# slab decomposition at bench size vs the undecomposed fused step (tools/slab_check.py):
# 256k at 1 and 2 ranks, 1M at 2 ranks, and the all-reduce line search at 256k
mkdir -p gpurun_out
rm -f gpurun_out/slab_check.jsonl
timeout 600 python tools/slab_check.py --steps 3 >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_w1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
   tools/slab_check.py --steps 3 >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_w2.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
   tools/slab_check.py --workload sand1m --steps 3 >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_1m.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 \
   tools/slab_check.py --steps 3 --solve allreduce >> gpurun_out/slab_check.jsonl 2> gpurun_out/slab_check_ar.err
