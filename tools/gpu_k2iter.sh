#!/bin/bash
# K2 iteration: correctness (quickcheck tiny/small + kernel tests), group trace, perf sweep
mkdir -p gpurun_out
tag=${1:-k2}
timeout 300 python tools/gpu_quickcheck.py small > gpurun_out/${tag}_qc_small.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_qc_small.log
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_q2.py -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
SS_NVCC_FLAGS=-DSS_GTRACE SS_LIB_OUT=/tmp/libss_gt.so python -c "from paper_2509_18344_b200.build import build; build()" && SS_LIBSUBSPEC=/tmp/libss_gt.so timeout 300 python tools/gtrace.py > gpurun_out/${tag}_gt.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_gt.log
bash tools/gpu_perf.sh ${tag}
