#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_qwen7b.py -x -q 2>&1 | grep -v "^$" | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/prof_pass.py 2>&1 | head -30
