"""Debug the SS_FP32 path against the oracle's exact mode step by step (tiny config)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from synth.configs import TINY
from synth.prompts import mtbench_prompt
from oracle.decode import Session
from oracle.tree import Tree
from paper_2509_18344_b200.binding import SubSpec, SS_FP32
SEED = 0x5EED
cfg = TINY
NR = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, max_chunk=256, precision=SS_FP32)
ss.load_synthetic(SEED, n_resident=NR)
ss.build_substitutes(4, 64)
ors = Session(cfg, SEED, n_resident=NR, mode="exact", max_nodes=256)
prompt = mtbench_prompt(SEED, 1, cfg.vocab, 40)
f = ss.prefill(prompt); of = ors.prefill(prompt)
print("first", f, of)
P = ors.kv.P
for l in range(cfg.n_layers):
    gk, gv = ss.debug_read_kv(l, 0, P)
    ok = ors.kv.K[l, :P].transpose(1, 0, 2); ov = ors.kv.V[l, :P].transpose(1, 0, 2)
    print("layer", l, "K maxdiff", np.abs(gk - ok).max(), "V maxdiff", np.abs(gv - ov).max(), "K scale", np.abs(ok).max())
tr = Tree([f], [-1], [0], [0.0])
g1 = ss.debug_forward(1, [f], [-1])
o1 = ors.forward_tree("target", tr)
print("target root maxdiff", np.abs(g1 - o1).max(), "scale", np.abs(o1).max())
g0, gh = ss.debug_forward(0, [f], [-1], hidden=True)
o0, oh = ors.forward_tree("draft", tr, return_hidden=True)
print("draft root maxdiff", np.abs(g0 - o0).max(), "hidden maxdiff", np.abs(gh - oh).max())
