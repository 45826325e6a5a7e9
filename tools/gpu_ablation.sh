mkdir -p gpurun_out
timeout 3000 python tools/ablation.py r1 > gpurun_out/ablation.log 2>&1
cp profiles/ablation_r1.json gpurun_out/ablation_r1.json
