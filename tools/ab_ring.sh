#!/bin/bash
# A/B of the K2 ring depth (SS_GEMV_RING_KB: stages of 2 Q4 tile-chunks + activations, ~22.6 KB at M <= 8)
for r in 88 92 68; do
  echo "== ring_kb=$r"
  SS_VERBOSE=1 SS_GEMV_RING_KB=$r timeout 300 python tools/prof_gemv.py 6 2>&1 | grep -E "group|plan<1,1>"
  SS_GEMV_RING_KB=$r timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|attn|o|gate_up|down) " | sed -n '1,2p;13,18p'
done
