mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py tests/test_gpu_batch.py tests/test_gpu_mlp.py tests/test_gpu_q2.py -x -q > gpurun_out/t_k8.log 2>&1
tail -2 gpurun_out/t_k8.log > gpurun_out/ab8.log
B=SS_LIBSUBSPEC=$PWD/paper_2509_18344_b200/libsubspec_base.so
bash tools/ab_rep.sh 2 "$B" "SS_X=1" >> gpurun_out/ab8.log 2>&1
timeout 300 python tools/prof_pass.py > gpurun_out/pass8.log 2>&1
