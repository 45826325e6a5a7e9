#!/bin/bash
# Round evidence (tag $1, default r2): GPU tests + smoke, the bench line, the ncu launch list of the
# bench's timed region, ncu --set full of the K2 substitute GEMV (gemv_q_kernel) launches and of the
# tcgen05 bf16 head GEMV (gemv_kernel) at Qwen2.5-7B shapes.
set -x
T=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$T.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests_$T.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/smoke_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_$T.err
tail -1 gpurun_out/bench_$T.jsonl | cut -c1-400
# launch list of exactly the timed steps (bench brackets them with cudaProfilerStart/Stop)
SS_PROFILE_TIMED=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ar --prompts 0 \
  > gpurun_out/ncu_launch_$T.log 2>&1
# full captures at M = 6 (see tools/prof_gemv.py for the launch order)
for spec in "gate_up 60" "qkv 4" "down 116"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_q_kernel -s $2 -c 1 \
    -o gpurun_out/k2_$1_$T python tools/prof_gemv.py 6 >> gpurun_out/ncu_k2_$T.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 \
  -o gpurun_out/head_$T python tools/prof_gemv.py 6 >> gpurun_out/ncu_k2_$T.log 2>&1
# K3 tree attention inside a draft pass (the 200th attention launch of tools/pass_time.py)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_node_kernel -s 200 -c 1 \
  -o gpurun_out/attn_$T python tools/pass_time.py 6 >> gpurun_out/ncu_k2_$T.log 2>&1
# copy/compute overlap of one step (events around every streamed group)
timeout 600 python tools/step_timeline.py gpurun_out/step_timeline_$T.json > gpurun_out/step_timeline_$T.log 2>&1
# K6 (tcgen05 verify GEMM) at M = 289 on a resident Qwen2.5-7B-width layer: gate_up and the head
# (launch order in tools/prof_k6.py with K6_ITERS=1: qkv 0-1, o 2-3, gate_up 4-5, down 6-7, head 8-9)
for spec in "gate_up 4" "head 8"; do
  set -- $spec
  K6_VARIANTS=0 K6_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s $2 -c 1 \
    -o gpurun_out/k6_$1_$T python tools/prof_k6.py 289 >> gpurun_out/ncu_k6_$T.log 2>&1
done
K6_VARIANTS=0,2,1 timeout 600 python tools/prof_k6.py 289 1025 > gpurun_out/k6_timing_$T.jsonl 2>> gpurun_out/ncu_k6_$T.log
ls -la gpurun_out | tail -30
