mkdir -p gpurun_out
bash tools/ab_rep.sh 2 "SS_X=1" "SS_GEMV_PERSM_OVR=3584:18944:1" "SS_GEMV_SPLIT_OVR=3584:18944:6" "SS_GEMV_SPLIT_OVR=3584:18944:7" > gpurun_out/ab7.log 2>&1
