"""SS_FP32 precision mode (SURVEY §8(b) `precision`; BASELINE.json north_star: "1e-4 in fp32 mode"):
the lockstep protocol of tests/test_gpu_decode.py against the oracle's exact fp64 mode, with the fp32
tolerance: draft logits within 1e-4 x logit scale, final hidden rows and committed K/V within rel-RMS
1e-4, argmax mismatches only at near-ties under 2e-4 x scale, accepted path and tokens bit-exact, and
the generated sequence equal to the oracle's greedy AR output (O.8) up to flagged near-ties."""
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt
from oracle.decode import Session
from oracle.tree import Tree, tempered_log_softmax, select_topk
from oracle.verify import accept, commit, argmax_and_gap
from gpu_util import scale_of, assert_close_scaled, rel_rms, assert_matches_oracle_ar
from test_gpu_decode import _check_selection

pytestmark = pytest.mark.gpu
SEED = 0x5EED
TOL = 1e-4


def _gpu(cfg, n_res, D, k, cap=512 << 20):
    from paper_2509_18344_b200.binding import SubSpec, SS_FP32
    ss = SubSpec(cfg, cap, max_depth=D, max_top_k=k, max_chunk=256, precision=SS_FP32)
    ss.load_synthetic(SEED, n_resident=n_res)
    ss.build_substitutes(4, 64)
    return ss


@pytest.mark.parametrize("cfg,n_res,D,k", [(TINY, 1, 4, 6), (SMALL, 1, 4, 6), (SMALL, 0, 3, 4)],
                         ids=["tiny", "small", "small-allsub"])
def test_fp32_lockstep(cuda_required, cfg, n_res, D, k):
    T = 0.2
    ss = _gpu(cfg, n_res, D, k)
    ors = Session(cfg, SEED, n_resident=n_res, mode="exact", max_nodes=max(256, 1 + k * D))
    prompt = mtbench_prompt(SEED, 1, cfg.vocab, 40)
    first = ss.prefill(prompt)
    assert first == ors.prefill(prompt)
    root = first
    for step in range(3):
        tr = ss.draft_tree(D, k, T)
        n = len(tr["tokens"])
        assert n == 1 + k * D and tr["tokens"][0] == root
        g_draft, g_hid = ss.debug_forward(0, tr["tokens"], tr["parents"], hidden=True)
        tree = Tree([int(t) for t in tr["tokens"]], [int(p) for p in tr["parents"]],
                    [int(d) for d in tr["depths"]], [float(s) for s in tr["scores"]])
        o_draft, o_hid = ors.forward_tree("draft", tree, return_hidden=True)
        assert_close_scaled(g_draft, o_draft, tol=TOL, what="fp32 draft logits")
        assert rel_rms(g_hid, o_hid) <= TOL
        _check_selection(tr["tokens"], tr["parents"], tr["scores"], g_draft, D, k, T)
        am, gap = ss.verify_tree(n)
        o_logits = ors.forward_tree("target", tree)
        o_am, o_gap = argmax_and_gap(o_logits)
        bad = np.nonzero(am != o_am)[0]
        assert np.all(o_gap[bad] <= 2 * TOL * scale_of(o_logits)), f"unflagged argmax mismatch at {bad}"
        toks, path = ss.accept_and_commit(D + 1)
        o_path, o_emit = accept(tree, am)
        assert o_emit == toks and [0] + o_path == path
        P = ors.kv.P
        commit(ors.kv, o_path)
        for l in range(cfg.n_layers):
            gk, gv = ss.debug_read_kv(l, P, len(path))
            assert rel_rms(gk, ors.kv.K[l, P:P + len(path)].transpose(1, 0, 2)) <= TOL
            assert rel_rms(gv, ors.kv.V[l, P:P + len(path)].transpose(1, 0, 2)) <= TOL
        root = toks[-1]
    ss.close()


@pytest.mark.parametrize("cfg,n_res", [(TINY, 1), (SMALL, 0)], ids=["tiny", "small-allsub"])
def test_fp32_generate_equals_oracle_ar(cuda_required, cfg, n_res):
    ss = _gpu(cfg, n_res, 4, 6)
    for p in range(2):
        prompt = mtbench_prompt(SEED, 10 + p, cfg.vocab, 24 + 13 * p)
        out, _ = ss.generate(prompt, 32, 4, 6, 0.2)
        assert_matches_oracle_ar(cfg, prompt, out, SEED, tol=TOL, mode="exact")
    ss.close()
