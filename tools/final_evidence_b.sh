#!/bin/bash
# Round-end evidence, part B: the other BASELINE.json configurations and variants (one line each)
mkdir -p gpurun_out
T=${1:-r2}
free -g | head -2 > gpurun_out/configs_$T.log
run() { local name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/cfg_${name}_$T.jsonl 2>> gpurun_out/configs_$T.log; echo "$name rc=$?" >> gpurun_out/configs_$T.log; }
run planner4 --n-resident -1 --no-cpu-baseline --no-ar
run planner2 --n-resident -1 --sub-bits 2 --no-cpu-baseline --no-ar
run q2 --sub-bits 2 --no-cpu-baseline --no-ar --prompts 0
run q3 --sub-bits 3 --no-cpu-baseline --no-ar --prompts 0
run hqq --quant hqq --no-cpu-baseline --no-ar --prompts 0
run embedgpu --embed-gpu --no-cpu-baseline --no-ar --prompts 0
for B in 2 4 5; do run batch$B --batch $B --no-cpu-baseline --no-ar; done
run config4 --config qwen2.5-32b --cap-gib 24 --steps 3 --warmup 3 --no-cpu-baseline --no-ar --prompts 0 --no-e2e
SWEEP_D=8,16,32,48,96 SWEEP_K=1,2,4,6,8,16 SWEEP_STEPS=3 timeout 1800 python tools/sweep_config3.py > gpurun_out/sweep_config3_$T.jsonl 2>> gpurun_out/configs_$T.log
echo "sweep rc=$?" >> gpurun_out/configs_$T.log
