#!/bin/bash
# A/B: CTAs per SM of the cluster plan per matrix group (qkv 4608x3584, o 3584x3584, down 3584x18944)
mkdir -p gpurun_out
timeout 300 python tools/cta_trace.py 4 5 6 7 8 > gpurun_out/cta_trace_default.log 2>&1
for ovr in "" "3584:18944:1" "4608:3584:1" "3584:3584:1" "4608:3584:1,3584:3584:1,3584:18944:1" "4608:3584:1,3584:3584:1"; do
  echo "== SS_GEMV_PERSM_OVR=$ovr"
  SS_VERBOSE=1 SS_GEMV_PERSM_OVR=$ovr timeout 300 python tools/prof_pass.py 2>&1 | grep -E "plan|^full|^gemv only|^(qkv|attn|o|gate_up|down) " | sed -n '1,12p;19,26p'
done
