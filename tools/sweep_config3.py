"""BASELINE.json config 3: Llama-3.1-8B shape, 12 GiB emulated cap, planner-max
residency, sweep of the draft tree depth D and width k (1 + kD <= 2048 - 512).  Per (D, k): step time
(CUDA events around K steps on the compute stream), draft / verify split, tau, the streamed bytes per
step, and the K2 GEMV time at M = k (layer sweep).  Random weights: tau is a property of the synthetic
model; the step-time columns are the systems result (how the verify compute stays hidden under the
host-link stream as the tree grows).  Writes one JSON line per point to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth.configs import LLAMA8B, GIB  # noqa: E402
from synth.prompts import mtbench_prompt  # noqa: E402
from paper_2509_18344_b200.binding import SubSpec  # noqa: E402

Ds = [int(x) for x in os.environ.get("SWEEP_D", "8,16,32,48,64,96").split(",")]
Ks = [int(x) for x in os.environ.get("SWEEP_K", "1,2,4,6,8,16,32").split(",")]
STEPS = int(os.environ.get("SWEEP_STEPS", "4"))
cfg = LLAMA8B
ss = SubSpec(cfg, 12 * GIB, max_depth=max(Ds), max_top_k=max(Ks), max_chunk=256)
ss.load_synthetic(0x5EED, -1)
ss.build_substitutes(4, 64)
st0 = ss.stats()
print(json.dumps({"config": "llama-3.1-8b, 12 GiB, planner max residency", "n_resident": st0["n_resident"],
                  "ring_bytes": st0["ring_bytes"], "substitute_bytes": st0["substitute_bytes"]}), flush=True)
cs = ss.compute_stream
for D in Ds:
    for k in Ks:
        if 1 + k * D > 2048 - 512:
            continue
        ss.prefill(mtbench_prompt(0x5EED, 0, cfg.vocab))
        ss.step(D, k, 0.2)                       # warm-up (graph capture for this shape)
        ss.reset_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cs)
        toks = 0
        for _ in range(STEPS):
            toks += len(ss.step(D, k, 0.2))
        ring_full = torch.cuda.Event()            # steady state, as bench.py: the ring is re-prefetched
        ring_full.record(ss.copy_stream)
        cs.wait_event(ring_full)
        e1.record(cs)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / STEPS
        st = ss.stats()
        k2 = ss.debug_time_matmul(-1, -2, k, iters=1) * 1e3   # us per GEMV launch, all layers x groups
        print(json.dumps({"D": D, "k": k, "nodes": 1 + k * D, "ms_per_step": ms, "tau": toks / STEPS,
                          "tokens_per_s": toks / STEPS / (ms / 1e3),
                          "draft_ms": st["draft_ms"] / STEPS if "draft_ms" in st else None,
                          "verify_ms": st["verify_ms"] / STEPS if "verify_ms" in st else None,
                          "stream_gb_per_step": st["stream_bytes"] / STEPS / 1e9,
                          "k2_us_per_launch": k2}), flush=True)
ss.close()
