mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 300 python tools/prof_pass.py > gpurun_out/pass1.log 2>&1
bash tools/ncu_gu.sh
