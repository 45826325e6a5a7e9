#!/bin/bash
# A/B of draft-pass variants (multi-kernel with/without L2 prefetch, CTAs/SM, fused)
for cfg in "0 1 2" "0 0 2" "0 1 3" "1 1 2"; do set -- $cfg
  echo "== fused=$1 l2pf=$2 ctas/sm=$3"
  SS_FUSED_DRAFT=$1 SS_L2_PREFETCH=$2 SS_GEMV_CTAS_PER_SM=$3 SS_GEMV_RING_KB=$([ $3 = 3 ] && echo 60 || echo 88) timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|o|gate_up|down) " | sed -n '1,2p;7,10p'
done
