"""Attribute one Qwen-7B-shape draft pass (M = 6) to kernel classes by skipping them."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes()
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
for name, skip in (("full", 0), ("-attn", 1), ("-norm", 2), ("-gemv", 4), ("-head", 8), ("gemv+head only", 3), ("gemv only", 11), ("nothing", 15)):
    print(f"{name:16s} {ss.debug_time_pass(6, 5, skip) * 1e3:9.1f} us/pass", flush=True)
tr = ss.debug_trace_pass(6).astype("float64")
t0 = tr[:, 0].min()
names = ["qkv", "attn", "o", "gate_up", "down"]
print("launch  entry  pdep  cdep  first  loop0  loopmax  end   (us, rel. to first entry)")
prev_end = None
for i, r in enumerate(tr[:3 * len(names)]):
    rel = (r - t0) / 1e3
    gap = "" if prev_end is None else f" gap_from_prev_end={rel[0] - prev_end:6.2f}"
    print(f"{names[i % len(names)]:8s} " + " ".join(f"{v:6.2f}" for v in rel[[0, 1, 2, 3, 4, 7, 6]]) + gap)
    prev_end = rel[6]
    if names[i % len(names)] == "attn":
        print("         attn: entry %.2f dep %.2f q %.2f loop %.2f merge1 %.2f end %.2f" % tuple((r[0:6] - t0) / 1e3))
        prev_end = (r[5] - t0) / 1e3
        continue
    if names[i % len(names)] == "mlp":
        print("         mlp: A-done0 %.2f A-donemax %.2f B-first0 %.2f B-loopmax %.2f fin-epi %.2f end %.2f" % tuple((r[[4, 7, 3, 5, 8, 6]] - t0) / 1e3))
    if r[13]:
        print("         xnorm: r-ready %.2f built %.2f" % tuple((r[13:15] - t0) / 1e3))
    if r[8]:
        print("         epilogue: reduce %.2f resid %.2f barrier %.2f r %.2f done %.2f" % tuple((r[8:13] - t0) / 1e3))
