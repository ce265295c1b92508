# several independent environments on one GPU (tools/multi_env.py)
mkdir -p gpurun_out
rm -f gpurun_out/multi_env.jsonl
for e in 2 4; do timeout 900 python tools/multi_env.py --envs $e --workload sand >> gpurun_out/multi_env.jsonl 2>/dev/null; done
timeout 900 python tools/multi_env.py --envs 4 --workload cloth >> gpurun_out/multi_env.jsonl 2>/dev/null
