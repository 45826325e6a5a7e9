#!/bin/bash
for v in "SS_MLP_DBG=0" "SS_MLP_DBG=4" "SS_MLP_DBG=8"; do
  echo "== $v"; env $v timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^mlp|^o |mlp:" | sed -n '1p;5,7p'
done
