# slab decomposition at bench size, continued: 1M sand at 2 ranks (fused,
# gather0) and 256k at 2 ranks with the all-reduce line search
mkdir -p gpurun_out
rm -f gpurun_out/slab_check2.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
   tools/slab_check.py --workload sand1m --steps 3 >> gpurun_out/slab_check2.jsonl 2> gpurun_out/slab_check2_1m.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 \
   tools/slab_check.py --steps 3 --solve allreduce >> gpurun_out/slab_check2.jsonl 2> gpurun_out/slab_check2_ar.err
