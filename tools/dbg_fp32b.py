import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from synth.configs import TINY
from oracle.decode import Session
from oracle.tree import Tree
from paper_2509_18344_b200.binding import SubSpec, SS_FP32
SEED = 0x5EED
for nl in (1, 2):
    cfg = TINY.with_(n_layers=nl)
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, max_chunk=256, precision=SS_FP32)
    ss.load_synthetic(SEED, n_resident=nl)
    ss.build_substitutes(4, 64)
    ors = Session(cfg, SEED, n_resident=nl, mode="exact", max_nodes=256)
    for plen in (1, 3):
        prompt = [5, 77, 300][:plen]
        ors.kv.P = 0
        f = ss.prefill(prompt); of = ors.prefill(prompt)
        g, gh = ss.debug_forward(1, [f], [-1], hidden=True)
        o, oh = ors.forward_tree("target", Tree([f], [-1], [0], [0.0]), return_hidden=True)
        print(f"layers {nl} prompt {plen}: first {f}/{of} logits maxdiff {np.abs(g - o).max():.3e} hidden maxdiff {np.abs(gh - oh).max():.3e} scale {np.abs(o).max():.2f}")
    ss.close()
