mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py tests/test_gpu_batch.py tests/test_gpu_q2.py tests/test_gpu_qwen7b.py -x -q > gpurun_out/t_k9.log 2>&1
tail -2 gpurun_out/t_k9.log > gpurun_out/ab9.log
bash tools/ab_rep.sh 2 "SS_GEMV_CW16=0" "SS_GEMV_CW16=1" >> gpurun_out/ab9.log 2>&1
timeout 300 python tools/prof_pass.py > gpurun_out/pass9.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
