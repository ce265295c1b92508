# configs[3] T-shirt window (the default bench window: 170 solver iterations
# per substep): solver grid size and line-search group size sweeps
mkdir -p gpurun_out
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
