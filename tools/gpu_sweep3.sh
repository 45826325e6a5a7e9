mkdir -p gpurun_out
timeout 1500 python tools/sweep_config3.py > gpurun_out/sweep_config3.jsonl 2> gpurun_out/sweep_config3.err
tail -3 gpurun_out/sweep_config3.err
