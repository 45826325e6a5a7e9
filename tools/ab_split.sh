#!/bin/bash
# A/B of the cluster split-K factor cap and CTAs per SM for the narrow draft GEMVs (qkv, o, down)
for cfg in "8 2" "6 2" "5 2" "4 2" "8 1"; do set -- $cfg
  echo "== max_cluster=$1 ctas_per_sm=$2"
  SS_VERBOSE=1 SS_GEMV_MAX_CLUSTER=$1 SS_GEMV_CTAS_PER_SM=$2 timeout 300 python tools/prof_gemv.py 6 2>&1 | grep -E "group|plan<1,1>"
  SS_GEMV_MAX_CLUSTER=$1 SS_GEMV_CTAS_PER_SM=$2 timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|attn|o|gate_up|down) " | sed -n '1,2p;13,18p'
done
