"""Print the mean draft-pass time (Qwen-7B shape, 8 GiB, M = 6) over a few repeats."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
M = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes()
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
ss.debug_time_pass(M, 5, 0)
ts = [ss.debug_time_pass(M, 20, 0) * 1e3 for _ in range(5)]
gs = {g: ss.debug_time_matmul(-1, g, M, iters=3) * 1e3 for g in (0, 1, 2, 3)}
print("PASS_US", " ".join(f"{t:.1f}" for t in ts), "min %.1f" % min(ts),
      "| sweep us qkv %.2f o %.2f gate_up %.2f down %.2f" % (gs[0], gs[1], gs[2], gs[3]), flush=True)
