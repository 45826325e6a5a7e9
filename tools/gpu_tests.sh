#!/bin/bash
# GPU test pass: pytest -m gpu (+ optional extra pytest args) and smoke; logs under gpurun_out/<tag>_*
tag=${1:-t}; shift
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
free -g > gpurun_out/${tag}_free.txt; nproc >> gpurun_out/${tag}_free.txt
