"""A/B of K2 knobs on the Qwen2.5-7B shape: per-group sweep times and the draft pass, alternating."""
import sys, os, json
sys.path.insert(0, os.getcwd())
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
from synth.prompts import mtbench_prompt
knob = int(sys.argv[1]) if len(sys.argv) > 1 else 0
vals = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "0"])]
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes(4, 64)
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
def kb(N, K, M): return N*K//2 + N*K//64*4 + M*K*2 + M*N*2
for rep in range(2):
    for v in vals:
        ss.debug_set_knob(knob, v)
        res = {}
        for g, name in enumerate(("qkv", "o", "gate_up", "down")):
            t = ss.debug_time_matmul(-1, g, 6, iters=3)
            res[name] = round(t * 1e3, 2)
        t = ss.debug_time_matmul(-1, -2, 6, iters=3)
        byt = sum(kb(*ss.group_shape(g), 6) for g in range(4))
        res["sweep_gbs"] = round(byt / (4 * t * 1e-3) / 1e9)
        res["pass_us"] = round(ss.debug_time_pass(6, 5, 0) * 1e3, 1)
        print(f"knob{knob}={v}", json.dumps(res), flush=True)
