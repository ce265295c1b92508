# slab decomposition at one rank against the undecomposed fused step, same window
mkdir -p gpurun_out
for m in "--single" "" "--ops"; do
timeout 300 python tools/slab_run.py --workload sand --steps 6 --warmup 1 $m >> gpurun_out/slab_w1_window.jsonl 2>/dev/null
timeout 300 python tools/slab_run.py --workload sand1m --steps 3 --warmup 1 $m >> gpurun_out/slab_w1_window.jsonl 2>/dev/null
done
