"""Repro: Qwen-7B-shape SD generate (test_gpu_qwen7b flow) with optional debug_matmul first."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6, max_chunk=256)
ss.load_weights(0x5EED, n_resident=0)
ss.build_substitutes(4, 64)
prompt = mtbench_prompt(0x5EED, 0, QWEN7B.vocab)
if "mm" in sys.argv:
    for g in range(4):
        N, K = ss.group_shape(g)
        ss.debug_matmul(0, 3, g, np.zeros((6, K), np.uint16))
    print("matmul ok", flush=True)
t = time.time()
try:
    sd, hist = ss.generate(prompt, 24, 48, 6, 0.2)
    print("generate ok", time.time() - t, hist[:10], flush=True)
except Exception as e:
    print("FAIL after", time.time() - t, e, flush=True)
