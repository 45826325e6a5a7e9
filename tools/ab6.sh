#!/bin/bash
# token-split cluster epilogue + monotonic norm barrier: tests + pass attribution
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/prof_pass.py 2>&1 | head -30
