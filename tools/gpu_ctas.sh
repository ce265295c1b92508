#!/bin/bash
# solver CTA count sweep on the T-shirt workload (default window: contact-heavy)
mkdir -p gpurun_out
for n in 0 24 48 96; do
  MPMRB_SOLVER_CTAS=$n timeout 600 python bench.py --no-cpu-baseline --no-e2e --workload tshirt > gpurun_out/ctas_tshirt_$n.json 2> /dev/null
done
