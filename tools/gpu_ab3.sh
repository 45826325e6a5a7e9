mkdir -p gpurun_out
bash tools/ab_rep.sh 2 "SS_X=0" "SS_PF_DOWN=1" "SS_PF_DOWN=2" > gpurun_out/ab3.log 2>&1
SS_PF_DOWN=1 timeout 300 python tools/prof_pass.py > gpurun_out/pass_pfdown.log 2>&1
