# ncu --set full of the fp32-mode P2G and G2P on the profiled 1M substep
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:'k_p2g|k_g2p' -o gpurun_out/ncu_f32_1m python bench.py --ncu-window --precision f32 --steps 20 \
   > gpurun_out/ncu_f32_1m.log 2>&1
echo rc=$? >> gpurun_out/ncu_f32_1m.log
