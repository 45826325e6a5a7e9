#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_host_weights.py tests/test_gpu_abi.py -m gpu -q -x > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
timeout 900 python bench.py > gpurun_out/r2d_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_bench.log
