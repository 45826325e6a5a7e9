#!/bin/bash
for r in 88 92 100; do
  echo "== ring $r KB"
  SS_GEMV_RING_KB=$r timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full"
  SS_GEMV_RING_KB=$r timeout 300 python tools/prof_gemv.py 6 2>&1 | tail -4
done
