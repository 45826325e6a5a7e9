mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py -x -q > gpurun_out/t_kern.log 2>&1
tail -2 gpurun_out/t_kern.log > gpurun_out/ab4.log
B=SS_LIBSUBSPEC=$PWD/paper_2509_18344_b200/libsubspec_base.so
bash tools/ab_rep.sh 2 "$B" "SS_X=1" >> gpurun_out/ab4.log 2>&1
timeout 300 python tools/prof_pass.py > gpurun_out/pass2.log 2>&1
