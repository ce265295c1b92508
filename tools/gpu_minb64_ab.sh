# float64 P2G/G2P register-budget A/B (variants built by tools/build_variant.sh)
mkdir -p gpurun_out
rm -f gpurun_out/minb64_ab.txt
for r in 1 2; do
  for v in default g2p64_3 g2p64_5 p2g64_2; do
    if [ $v = default ]; then unset MPMRB_LIB_PATH; else export MPMRB_LIB_PATH=paper_2503_05046_b200/_native/variants/$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['roofline']['stages_ms']; print('$v', round(d['rigid_steps_per_s'],2), round(s['p2g'],4), round(s['g2p'],4))" >> gpurun_out/minb64_ab.txt
  done
done
unset MPMRB_LIB_PATH
