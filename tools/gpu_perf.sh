#!/bin/bash
# perf check: per-group K2 sweep times + draft pass time + short bench (no cpu baseline)
mkdir -p gpurun_out
tag=${1:-perf}
cat > /tmp/k2sweep.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
from synth.prompts import mtbench_prompt
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes(4, 64)
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
def kb(N, K, M): return N*K//2 + N*K//64*4 + M*K*2 + M*N*2
res = {}
for M in (1, 6, 16, 24):
    for g, name in enumerate(("qkv", "o", "gate_up", "down")):
        N, K = ss.group_shape(g)
        t = ss.debug_time_matmul(-1, g, M, iters=3)
        res[f"{name}_M{M}"] = (round(t*1e3, 2), round(kb(N, K, M)/(t*1e-3)/1e9))
    t = ss.debug_time_matmul(-1, -2, M, iters=3)
    byt = sum(kb(*ss.group_shape(g), M) for g in range(4))
    res[f"sweep_M{M}"] = (round(t*1e3, 2), round(byt / (4*t*1e-3) / 1e9))
res["head_M6_us"] = ss.debug_time_matmul(0, -1, 6, iters=5) * 1e3
for M in (1, 6):
    res[f"pass_M{M}_us"] = ss.debug_time_pass(M, 5, 0) * 1e3
print(json.dumps(res, indent=0))
PY
timeout 600 python /tmp/k2sweep.py > gpurun_out/${tag}_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_sweep.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_bench.log
