#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/scene_study.txt
for args in "" "eps_v=1e-3" "ctas=32" "ctas=64" "eps_v=1e-3 ctas=64"; do
  timeout 600 python tools/scene_study.py tshirt 20 $args >> gpurun_out/scene_study.txt 2>/dev/null
done
for args in "" "ctas=64" "ctas=96"; do
  timeout 600 python tools/scene_study.py cloth 20 $args >> gpurun_out/scene_study.txt 2>/dev/null
done
