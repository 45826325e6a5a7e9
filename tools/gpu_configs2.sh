mkdir -p gpurun_out
timeout 900 python bench.py --sub-bits 2 --no-cpu-baseline 2> gpurun_out/c2.err | tail -1 > gpurun_out/bench_q2.jsonl
timeout 900 python bench.py --n-resident -1 --no-cpu-baseline 2>> gpurun_out/c2.err | tail -1 > gpurun_out/bench_planner4.jsonl
timeout 900 python bench.py --n-resident -1 --sub-bits 2 --no-cpu-baseline 2>> gpurun_out/c2.err | tail -1 > gpurun_out/bench_planner2.jsonl
timeout 1500 python bench.py --config qwen2.5-32b --cap-gib 24 --steps 4 --warmup 3 --no-cpu-baseline 2>> gpurun_out/c2.err | tail -1 > gpurun_out/bench_config4.jsonl
