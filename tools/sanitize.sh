#!/bin/bash
# compute-sanitizer over tools/sanitize.py (eager draft loop, no CUDA graph: the tools see each launch)
mkdir -p gpurun_out
tag=${1:-san}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize.py 0 \
    > gpurun_out/${tag}_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tag}_summary.log
  tail -3 gpurun_out/${tag}_${tool}.log >> gpurun_out/${tag}_summary.log
done
