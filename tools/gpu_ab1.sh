mkdir -p gpurun_out
B=SS_LIBSUBSPEC=$PWD/paper_2509_18344_b200/libsubspec_base.so
bash tools/ab_rep.sh 3 "$B" "SS_X=1" "SS_GEMV_PERSM_OVR=4608:3584:1" > gpurun_out/ab1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_mlp.py -x -q > gpurun_out/t_kern.log 2>&1
tail -3 gpurun_out/t_kern.log >> gpurun_out/ab1.log
