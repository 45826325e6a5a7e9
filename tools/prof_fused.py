"""Time the fused persistent draft pass at the Qwen2.5-7B shape and break it down per phase."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_weights(0x5EED, 0); ss.build_substitutes()
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
for M in (1, 6):
    print(f"fused pass M={M}: {ss.debug_time_pass(M, 10, 0) * 1e3:9.1f} us", flush=True)
tr = ss.debug_trace_pass(6, cap=64).reshape(-1, 2).astype(np.float64)
names = ["embed"] + ["norm1", "qkv", "attn", "combine", "o", "norm2", "gate_up", "down"] * 28 + ["normf", "head", "topk1", "topk2"]
t0 = tr[0, 0]
agg = collections.defaultdict(float)
for i, nm in enumerate(names):
    if i >= len(tr): break
    s, e = tr[i]
    nxt = tr[i + 1, 0] if i + 1 < len(names) and i + 1 < len(tr) else e
    agg[nm] += (nxt - s) / 1e3      # phase time incl. the barrier into the next phase
tot = sum(agg.values())
for k, v in agg.items(): print(f"  {k:8s} {v:8.1f} us  ({v/tot:.1%})")
print("  first layer (us from start):", [round((tr[i, 0] - t0) / 1e3, 2) for i in range(1, 10)])
