#!/bin/bash
# Round-end evidence, part A: the round's evidence script (tests, smoke, bench, launch list, ncu full
# captures, step timeline, K6 timing) plus the draft-pass timeline and per-CTA trace of the K2 launches
bash tools/run_evidence.sh r2
timeout 400 python tools/prof_pass.py > gpurun_out/prof_pass_r2.log 2>&1
timeout 400 python tools/cta_trace.py 6 7 5 > gpurun_out/cta_trace_r2.log 2>&1
ls -la gpurun_out | tail -40
