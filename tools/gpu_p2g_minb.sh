# fp32 P2G occupancy A/B: the default build vs __launch_bounds__(128, 5)
mkdir -p gpurun_out
for r in 1 2; do
  timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-e2e > gpurun_out/pminb_default_$r.json 2>/dev/null
  MPMRB_LIB_PATH=paper_2503_05046_b200/_native/variants/p2g_f32_5.so timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-e2e > gpurun_out/pminb_5_$r.json 2>/dev/null
done
