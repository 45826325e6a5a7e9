"""Per-CTA timing of one draft-pass GEMV launch (layer 1: 4 qkv, 5 o, 6 gate_up, 7 down)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0); ss.build_substitutes()
ss.prefill(mtbench_prompt(0x5EED, 0, QWEN7B.vocab))
for launch in [int(a) for a in sys.argv[1:]] or [6, 7]:
    t = ss.debug_cta_trace(6, launch).astype(np.float64)
    sm = t[:, 0].astype(int)
    t0 = t[:, 1].min()
    ent, fst, lend, end = [(t[:, i] - t0) / 1e3 for i in (1, 2, 3, 4)]
    q = lambda v: " ".join(f"{x:6.2f}" for x in np.percentile(v, [0, 10, 50, 90, 100]))
    print(f"launch {launch}: {len(t)} CTAs on {len(set(sm))} SMs")
    print("  entry    p0/10/50/90/100:", q(ent))
    print("  first    ", q(fst))
    print("  loop end ", q(lend))
    print("  end      ", q(end))
    print("  loop dur ", q(lend - fst))
    cnt = np.bincount(sm, minlength=148)
    print("  CTAs per SM histogram:", np.bincount(cnt))
    # slowest 10 CTAs
    order = np.argsort(lend)[::-1][:10]
    for i in order:
        print(f"   cta {i:4d} sm {sm[i]:3d} (sm has {cnt[sm[i]]}) entry {ent[i]:6.2f} first {fst[i]:6.2f} loopend {lend[i]:6.2f}")
    # loop duration vs SM parity / half
    lo = sm < 74
    print("  loop dur  sm<74:", q((lend - fst)[lo]), " sm>=74:", q((lend - fst)[~lo]))
