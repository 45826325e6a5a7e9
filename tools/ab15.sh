#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do echo "== xnorm $v"; SS_XNORM=$v timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full|^qkv|^down" | head -5; done
