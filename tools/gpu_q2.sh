mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_q2.py -x -q > gpurun_out/t_q2.log 2>&1; echo "rc=$?" >> gpurun_out/t_q2.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_generator_quant.py -x -q > gpurun_out/t_k.log 2>&1; echo "rc=$?" >> gpurun_out/t_k.log
timeout 600 python bench.py --sub-bits 2 --no-cpu-baseline > gpurun_out/bench_q2.jsonl 2> gpurun_out/bench_q2.err
