"""Draft-loop CUDA graph vs eager launches at config 2 (ss_options.cuda_graphs): draft and verify ms per
step over 6 steps after 3 warm-up steps, and the eager draft-pass timer, for graphs on / off / on.
Measured on B200: graphs 101.0 ms of draft per step, eager 103.3 ms."""
import sys, os, json
sys.path.insert(0, os.getcwd())
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
for graphs in (1, 0, 1):
    ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6, cuda_graphs=graphs)
    ss.load_synthetic(0x5EED, 0); ss.build_substitutes(4, 64)
    ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
    for _ in range(3): ss.step(48, 6, 0.2)
    ss.reset_stats() if hasattr(ss, "reset_stats") else None
    st0 = ss.stats()
    for _ in range(6): ss.step(48, 6, 0.2)
    st = ss.stats()
    print(json.dumps({"graphs": graphs, "draft_ms_per_step": (st["draft_ms"] - st0["draft_ms"]) / 6,
                      "verify_ms_per_step": (st["verify_ms"] - st0["verify_ms"]) / 6,
                      "pass_us_eager_timepass": ss.debug_time_pass(6, 5, 0) * 1e3}), flush=True)
    ss.close()
