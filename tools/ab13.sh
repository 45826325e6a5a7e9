#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in 1 4; do echo "== attn cluster $s"; SS_ATTN_CLUSTER=$s timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^-attn|attn:" | head -4; done
