#!/bin/bash
# ncu --set full of one K2 gate_up launch (Qwen-7B shape, M = 6) with SASS-level stall sampling
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 60 -c 1 \
  -o gpurun_out/k2_gu python tools/prof_gemv.py 6 > gpurun_out/ncu_gu.log 2>&1
ncu -i gpurun_out/k2_gu.ncu-rep --page source --csv --print-source sass > gpurun_out/k2_gu_sass.csv 2>&1
ncu -i gpurun_out/k2_gu.ncu-rep --page raw --csv > gpurun_out/k2_gu_raw.csv 2>&1
ls -la gpurun_out
