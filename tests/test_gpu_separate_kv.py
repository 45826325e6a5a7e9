"""NEXT-4: Table 2's draft WITHOUT the shared KV-cache (the shared
cache of PAPER.md:141-143 is the default).  With ss_options.separate_draft_kv = 1 the draft keeps its
own committed cache, filled with the draft's own K/V.

* lossless: the output equals the GPU's AR output bitwise and the oracle's greedy AR output;
* the draft's cache: after prefill and several steps, every committed position's draft K/V equals the
  oracle's draft forward of the committed sequence as a chain (oracle.model.draft_layers, the bf16
  rounding points of reading R3) within rel-RMS 2e-2 — a position's draft K/V depends only on the
  token prefix, so a chain forward is its plain definition;
* the variant is rejected where it is not built (batched slots, SS_FP32).
"""
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt
from oracle.decode import Session
from oracle.tree import Tree
from oracle.numerics import bf16_bits_to_f64
from gpu_util import TOL_BF16, rel_rms, assert_matches_oracle_ar

pytestmark = pytest.mark.gpu
SEED = 0x5EED


@pytest.mark.parametrize("cfg,n_res", [(TINY, 1), (SMALL, 1), (SMALL, 0)], ids=["tiny", "small", "small-allsub"])
def test_separate_draft_kv_lossless_and_cache(cuda_required, cfg, n_res):
    from paper_2509_18344_b200.binding import SubSpec
    prompt = [int(t) for t in mtbench_prompt(SEED, 11, cfg.vocab, 44)]
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, separate_draft_kv=1)
    ss.load_synthetic(SEED, n_resident=n_res)
    ss.build_substitutes(4, 64)
    first = ss.prefill(prompt, chunk=32)          # two chunks: the draft's chain forward spans both
    emitted = []
    for _ in range(4):
        emitted += ss.step(4, 6, 0.2)
    committed = prompt + [first] + emitted[:-1]
    P = len(committed)
    ors = Session(cfg, SEED, n_resident=n_res, mode="bf16", max_nodes=P + 8)
    ors.forward_tree("draft", Tree(committed, [i - 1 for i in range(P)], list(range(P)), [0.0] * P))
    for l in range(cfg.n_layers):
        gk, gv = ss.debug_read_draft_kv(l, 0, P)
        ok = ors.kv.tK[l, :P].transpose(1, 0, 2)
        ov = ors.kv.tV[l, :P].transpose(1, 0, 2)
        assert rel_rms(bf16_bits_to_f64(gk), ok) <= TOL_BF16, f"layer {l} draft K"
        assert rel_rms(bf16_bits_to_f64(gv), ov) <= TOL_BF16, f"layer {l} draft V"
    if n_res > 0:   # layer 0 is shared and has no earlier layer: the two caches agree there
        tk, _ = ss.debug_read_kv(0, 0, P)
        dk, _ = ss.debug_read_draft_kv(0, 0, P)
        assert rel_rms(bf16_bits_to_f64(dk), bf16_bits_to_f64(tk)) <= TOL_BF16
    ss.close()
    # lossless: the same prompt generated through the variant == GPU AR == the oracle's greedy AR
    a = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, separate_draft_kv=1)
    a.load_synthetic(SEED, n_resident=n_res)
    a.build_substitutes(4, 64)
    out, _ = a.generate(prompt, 32, 4, 6, 0.2)
    a.close()
    b = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6)
    b.load_synthetic(SEED, n_resident=n_res)
    b.build_substitutes(4, 64)
    ar, _ = b.generate(prompt, 32, 0, 1, 1.0)
    b.close()
    assert out == ar
    assert_matches_oracle_ar(cfg, prompt, out, SEED)


def test_separate_draft_kv_rejected_where_not_built(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec, SubSpecError, SS_FP32
    with pytest.raises(SubSpecError):
        SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6, max_batch=2, separate_draft_kv=1)
    with pytest.raises(SubSpecError):
        SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6, precision=SS_FP32, separate_draft_kv=1)
