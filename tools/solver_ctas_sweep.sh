# Solver grid size sweep on the small and medium workloads (MPMRB_SOLVER_CTAS
# forces the persistent solve's CTA count; unset = one CTA per SM).
mkdir -p gpurun_out
for w in tshirt cloth sand; do
  for k in 0 16 24 32 48 64 96; do
    if [ $k = 0 ]; then unset MPMRB_SOLVER_CTAS; else export MPMRB_SOLVER_CTAS=$k; fi
    timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', $k, round(d['ms_per_step'],3), d['config']['solver']['iterations_per_substep_mean'])" >> gpurun_out/ctas_sweep.txt
  done
done
unset MPMRB_SOLVER_CTAS
for k in 0 16 32 64; do
  if [ $k = 0 ]; then unset MPMRB_SOLVER_CTAS; else export MPMRB_SOLVER_CTAS=$k; fi
  timeout 600 python bench.py --workload tshirt --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ctas', $k, round(d['ms_per_step'],3), d['config']['solver']['iterations_per_substep_mean'])" >> gpurun_out/ctas_sweep_tshirt.txt
done
unset MPMRB_SOLVER_CTAS
for g in 4 8 26; do
  MPMRB_SOLVER_LS_CTAS=$g timeout 600 python bench.py --workload tshirt --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ls_ctas', $g, round(d['ms_per_step'],3), d['config']['solver']['iterations_per_substep_mean'])" >> gpurun_out/ctas_sweep_tshirt.txt
done
