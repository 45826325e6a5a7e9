#!/bin/bash
# ring depth x CTAs/SM sweep of the K2 GEMV timing at Qwen-7B shapes
for ring in 44 88 176; do for per in 1 2; do
  echo "ring=${ring}KB per_sm=$per"
  SS_GEMV_RING_KB=$ring SS_GEMV_CTAS_PER_SM=$per python tools/prof_gemv.py 6 2>&1 | grep group
done; done
