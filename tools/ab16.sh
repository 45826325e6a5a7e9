#!/bin/bash
L3=paper_2509_18344_b200/_build/libsubspec_mb3.so
echo "== default"; timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full"; timeout 300 python tools/prof_gemv.py 6 2>&1 | tail -4
echo "== mb3 per_sm 3 ring 46"; SS_LIBSUBSPEC=$L3 SS_GEMV_CTAS_PER_SM=3 SS_GEMV_RING_KB=46 timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full"; SS_LIBSUBSPEC=$L3 SS_GEMV_CTAS_PER_SM=3 SS_GEMV_RING_KB=46 timeout 300 python tools/prof_gemv.py 6 2>&1 | tail -4
echo "== mb3 per_sm 2 ring 88"; SS_LIBSUBSPEC=$L3 timeout 300 python tools/prof_pass.py 2>&1 | grep -E "^full"
