#!/bin/bash
for c in 8 9 10; do echo "== long-K cluster cap $c"; SS_VERBOSE=1 SS_GEMV_MAX_CLUSTER_LONGK=$c timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|K=18944" | head -3; done
