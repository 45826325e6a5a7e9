#!/bin/bash
# End-of-round evidence: GPU tests, smoke, bench line, ncu launch list, K2 full captures (Q4 gate_up/qkv, Q2 gate_up)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/run_evidence.sh > gpurun_out/evidence.log 2>&1
cat > /tmp/q2gemv.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.set_substitute_bits(2); ss.load_weights(0x5EED, 0); ss.build_substitutes(2, 64)
for g in (0, 2, 3, 1):
    print("group", g, "us", ss.debug_time_matmul(-1, g, 6, iters=1) * 1e3, flush=True)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 60 -c 1 \
  -o gpurun_out/k2q2_gate_up_r1 python /tmp/q2gemv.py > gpurun_out/ncu_k2q2_r1.log 2>&1
ls -la gpurun_out
