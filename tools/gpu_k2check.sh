#!/bin/bash
# K2 bring-up: quickcheck (tiny, small) then the kernel parity tests, short timeouts
mkdir -p gpurun_out
tag=${1:-k2}
timeout 300 python tools/gpu_quickcheck.py tiny > gpurun_out/${tag}_qc_tiny.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_qc_tiny.log
timeout 300 python tools/gpu_quickcheck.py small > gpurun_out/${tag}_qc_small.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_qc_small.log
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_generator_quant.py tests/test_gpu_decode.py -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
