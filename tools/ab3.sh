#!/bin/bash
for cfg in "88 2" "66 2" "44 2" "66 3" "44 3"; do set -- $cfg
  echo "== ring ${1}KB ctas/sm $2: $(SS_GEMV_RING_KB=$1 SS_GEMV_CTAS_PER_SM=$2 timeout 300 python tools/prof_pass.py 2>&1 | grep -E '^full' )"
done
