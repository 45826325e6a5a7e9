mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
