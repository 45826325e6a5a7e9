import sys, os
sys.path.insert(0, os.getcwd())
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes(4, 64)
print(ss.debug_gemv_plan(2, 6))
