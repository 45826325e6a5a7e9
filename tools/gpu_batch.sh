mkdir -p gpurun_out
: > gpurun_out/bench_batch.jsonl
for B in 2 4 5; do
  timeout 900 python bench.py --batch $B --no-cpu-baseline 2>> gpurun_out/bench_batch.err | tail -1 >> gpurun_out/bench_batch.jsonl
done
