#!/bin/bash
timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full"
timeout 300 python tools/prof_gemv.py 6 2>&1 | tail -4
