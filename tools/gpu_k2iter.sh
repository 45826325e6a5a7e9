#!/bin/bash
# K2 iteration: correctness (quickcheck tiny/small + kernel tests), group trace, perf sweep
mkdir -p gpurun_out
tag=${1:-k2}
timeout 300 python tools/gpu_quickcheck.py tiny > gpurun_out/${tag}_qc_tiny.log 2>&1; timeout 300 python tools/gpu_quickcheck.py small > gpurun_out/${tag}_qc_small.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_qc_small.log
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_q2.py -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
bash tools/gpu_perf.sh ${tag}
