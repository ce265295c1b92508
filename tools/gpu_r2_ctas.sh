#!/bin/bash
# solver grid size vs problem size: bench lines with MPMRB_SOLVER_CTAS forced
mkdir -p gpurun_out
rm -f gpurun_out/ctas_*.json
for w in tshirt cloth sand; do
  for n in 0 16 32 64 96; do
    MPMRB_SOLVER_CTAS=$n timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ctas_${w}_$n.json 2> /dev/null
  done
done
