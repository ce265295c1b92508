#!/bin/bash
# bench-level A/B of library variants (stage times of P2G / G2P in the JSON)
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then lp=paper_2503_05046_b200/_native/libmpmrb_b200.so; else lp=paper_2503_05046_b200/_native/variants/$v.so; fi
  MPMRB_LIB_PATH=$lp timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab3_256_${v}_$rep.json 2> /dev/null
  MPMRB_LIB_PATH=$lp timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workload sand1m > gpurun_out/ab3_1m_${v}_$rep.json 2> /dev/null
done
done
