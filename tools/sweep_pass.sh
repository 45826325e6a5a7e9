#!/bin/bash
for cfg in "88 1" "132 1" "176 1" "88 2"; do set -- $cfg
  echo "== ring=${1}KB ctas/sm=$2"
  SS_GEMV_RING_KB=$1 SS_GEMV_CTAS_PER_SM=$2 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|o|gate_up|down) " | sed -n '1,2p;7,10p'
done
