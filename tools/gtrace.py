import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
from synth.prompts import mtbench_prompt
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes(4, 64)
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
np.set_printoptions(linewidth=200)
for g in range(4):
    print("plan", g, ss.debug_gemv_plan(g, 6))
for g in (2, 3, 0):
    t = ss.debug_group_trace(1, g, 6)
    n = int((t[:, 0] > 0).sum())
    v = t[:n]
    t0 = v[v > 0].min()
    d = np.where(v > 0, v - t0, -1)
    print("group", g, "n", n, "cols: 0 conv ready,1 A free,2 A written,3 MMA0 go,4 MMA1 go,5 MMA0 commit,6 acc ready,7 acc released,"
          "8 prod stage wait,9 prod stage free,10 conv full seen,11 MMA full seen,12 conv before full,13 MMA1 commit")
    print(d.astype(np.int64))
