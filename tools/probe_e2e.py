"""Wall-clock per step: ss.step vs draft/verify/accept calls vs device events (Qwen-7B shape)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes()
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
for _ in range(3): ss.step(48, 6, 0.2)
torch.cuda.synchronize()
n = 6
t0 = time.perf_counter()
for _ in range(n): ss.step(48, 6, 0.2)
torch.cuda.synchronize(); print("ss.step wall ms/step", (time.perf_counter() - t0) / n * 1e3, flush=True)
root = int(ss.step(48, 6, 0.2)[-1]); torch.cuda.synchronize()
t0 = time.perf_counter()
tt = {"draft": 0, "verify": 0, "accept": 0}
for _ in range(n):
    a = time.perf_counter(); ss.draft_tree(48, 6, 0.2, root_token=root, want_tree=False); b = time.perf_counter()
    ss.verify_tree(want=False); c = time.perf_counter()
    toks, _ = ss.accept_and_commit(49); d = time.perf_counter()
    root = toks[-1]
    tt["draft"] += b - a; tt["verify"] += c - b; tt["accept"] += d - c
torch.cuda.synchronize(); print("3-call wall ms/step", (time.perf_counter() - t0) / n * 1e3, {k: v / n * 1e3 for k, v in tt.items()})
