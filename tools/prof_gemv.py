"""Driver for ncu captures of the K2 dequant-GEMV at Qwen2.5-7B shapes (8 GiB cap, 0 resident)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
M = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0)
ss.build_substitutes()
for g in (0, 2, 3, 1):
    t = ss.debug_time_matmul(-1, g, M, iters=1)
    print("group", g, "us", t * 1e3, flush=True)
