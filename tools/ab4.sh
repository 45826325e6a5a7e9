#!/bin/bash
for cfg in "88 2" "52 3" "40 3"; do set -- $cfg
  echo "== ring ${1}KB ctas/sm $2"
  SS_GEMV_RING_KB=$1 SS_GEMV_CTAS_PER_SM=$2 timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|o|gate_up|down) " | sed -n '1,2p;7,10p'
done
SS_GEMV_RING_KB=52 SS_GEMV_CTAS_PER_SM=3 timeout 300 python tools/prof_gemv.py 6
