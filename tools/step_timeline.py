"""Copy/compute overlap of one config-2 SubSpec step (A4 / K7; App. E): CUDA events
around every streamed layer group (ss_debug_step_timeline).  Writes the rows and a summary (copy-engine
busy fraction per phase, the verify's wait on copies, the per-group compute) as one JSON object.
Usage: python tools/step_timeline.py [out.json]"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec

D, K, T = 48, 6, 0.2
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=D, max_top_k=K)
ss.load_synthetic(0x5EED, 0)
ss.build_substitutes(4, 64)
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
for _ in range(3):                      # warm-up steps (graphs captured, ring in steady state)
    ss.step(D, K, T)
rows, ph = ss.debug_step_timeline(D, K, T)
t_draft, t_verify, t_accept = (float(x) for x in ph)
ok = rows[:, 4] > -1e8
cs, ce, ks, ke = rows[:, 4], rows[:, 5], rows[:, 6], rows[:, 7]


def busy(lo, hi):   # copy-engine busy ms inside [lo, hi)
    return float(sum(max(0.0, min(b, hi) - max(a, lo)) for a, b in zip(cs[ok], ce[ok])))


cons = (ks > -1e8) & (ke > -1e8)
summary = {
    "phases_ms": {"draft": t_draft, "verify": t_verify - t_draft, "accept": t_accept - t_verify, "step": t_accept},
    "copy_busy_ms": {"draft": busy(0.0, t_draft), "verify": busy(t_draft, t_verify)},
    "copy_busy_frac": {"draft": busy(0.0, t_draft) / max(t_draft, 1e-9),
                       "verify": busy(t_draft, t_verify) / max(t_verify - t_draft, 1e-9)},
    "groups_consumed": int(cons.sum()),
    "groups_copied_before_verify": int(((ce < t_draft) & cons & ok).sum()),
    "bytes_copied_during_draft": float(sum(b * max(0.0, min(e, t_draft) - max(st, 0.0)) / max(e - st, 1e-9)
                                          for b, st, e in zip(rows[ok, 3], cs[ok], ce[ok]))),
    "compute_ms_per_group_mean": float(np.mean(ke[cons] - ks[cons])) if cons.any() else None,
    "stream_bytes_step": float(rows[cons, 3].sum()),
    "verify_waiting_on_copies_ms": float(sum(max(0.0, s - max(prev, t_draft)) for s, prev in
                                            zip(ks[cons][1:], ke[cons][:-1]))),
}
res = {"config": "qwen2.5-7b, 8 GiB, n_resident=0, 4-bit g64, D=48 k=6 T=0.2, K7 codec on",
       "columns": ["item", "layer", "group", "host_bytes", "copy_start_ms", "copy_end_ms", "compute_start_ms",
                   "ring_release_ms"],
       "summary": summary, "rows": [[float(v) for v in r] for r in rows]}
out = sys.argv[1] if len(sys.argv) > 1 else None
txt = json.dumps(res)
if out:
    open(out, "w").write(txt)
print(json.dumps(summary, indent=1))
ss.close()
