#!/bin/bash
for mc in 16 8; do
  echo "== max cluster $mc"
  SS_GEMV_MAX_CLUSTER=$mc timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^gemv only|^(qkv|o|gate_up|down) " | sed -n '1,2p;7,10p'
done
