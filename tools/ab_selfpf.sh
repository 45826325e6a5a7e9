#!/bin/bash
# A/B: GEMV self-prefetch of each CTA's own weight range into L2 (bit g = matrix group g)
for v in 0 15 12 4 8; do
  echo "== SS_GEMV_SELF_PF=$v"
  SS_GEMV_SELF_PF=$v timeout 300 python tools/prof_gemv.py 6 2>&1 | grep group
  SS_GEMV_SELF_PF=$v timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|o|gate_up|down) " | sed -n '1,3p;8,12p'
done
