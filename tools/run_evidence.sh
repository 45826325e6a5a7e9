#!/bin/bash
# Round evidence: bench line, ncu launch list of the bench command, ncu --set full of K2 launches.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r1.jsonl 2> gpurun_out/bench_r1.err
tail -1 gpurun_out/bench_r1.jsonl
# launch list: skip the load/prefill/first (eager + capture) step; capture ~1 draft/verify worth
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 2200 -c 2500 --csv \
  --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_r1.log 2>&1
# full capture of dequant-GEMV launches at Qwen-7B shapes (M = 6): a gate_up and a qkv launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 60 -c 1 \
  -o gpurun_out/k2_gate_up_r1 python tools/prof_gemv.py 6 > gpurun_out/ncu_k2_r1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 4 -c 1 \
  -o gpurun_out/k2_qkv_r1 python tools/prof_gemv.py 6 >> gpurun_out/ncu_k2_r1.log 2>&1
ls -la gpurun_out
