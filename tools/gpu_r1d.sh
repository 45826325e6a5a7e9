mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_generator_quant.py -x -q > gpurun_out/t_d.log 2>&1; echo "rc=$?" >> gpurun_out/t_d.log
bash tools/gpu_sweep3.sh
bash tools/gpu_configs.sh
