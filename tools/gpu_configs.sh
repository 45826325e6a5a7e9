mkdir -p gpurun_out
free -g | head -2 > gpurun_out/configs.log
timeout 900 python bench.py --n-resident -1 --no-cpu-baseline > gpurun_out/bench_planner4.jsonl 2>> gpurun_out/configs.log
timeout 900 python bench.py --n-resident -1 --sub-bits 2 --no-cpu-baseline > gpurun_out/bench_planner2.jsonl 2>> gpurun_out/configs.log
timeout 1500 python bench.py --config qwen2.5-32b --cap-gib 24 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_config4.jsonl 2>> gpurun_out/configs.log
tail -5 gpurun_out/configs.log
