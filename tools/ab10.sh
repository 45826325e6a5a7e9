#!/bin/bash
# fused MLP kernel: repro steps, GPU tests, pass attribution (fused vs not)
timeout 120 python tools/repro_q7b.py step3 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/prof_pass.py 2>&1 | head -30
SS_FUSE_MLP=0 timeout 300 python tools/prof_pass.py 2>&1 | head -3
