"""Full-width oracle lockstep (SURVEY §8(c) protocol) at the hidden / FFN / head / vocab widths of the
BASELINE.json shapes, with two decoder layers, both offloaded (n_resident = 0): every
K2 substitute GEMV and the streamed K6 verify run at their production widths, GQA 7:1 (Qwen2.5-7B),
4:1 (Llama-3.1-8B, no bias) and 5:1 (Qwen2.5-32B), top-k over V = 152064 / 128256, the head argmax
over all vocab tiles, D = 48 / k = 6 / T = 0.2 trees (289 nodes, 49-deep ancestor tables), a prompt of
MT-Bench length (>= 160 tokens) and one longer than the 256-token prefill chunk.

The oracle runs in its fp32-BLAS mode (oracle.model.forward_nodes_batched: the bf16 rounding points of
reading R3, fp32 weights, node-batched fp32 products; pinned in tests/test_oracle_batched.py) and
generates its own weights (synth/weights.py), never reading anything from the GPU.

Per step, from a shared state:
 1. draft: GPU draft logits and final hidden rows on its own tree (teacher-forced, ss_debug_forward)
    vs the oracle's, within 2e-2 x logit scale / rel-RMS 2e-2; the oracle's sharpened top-k run on the
    GPU's logits rebuilds the GPU's tree (up to flagged fp32 near-ties);
 2. verify: GPU target argmax vs the oracle's; a mismatch is allowed only at a flagged near-tie;
 3. accept: the oracle's walk on (GPU tree, GPU argmax) reproduces the GPU's path and tokens exactly;
 4. commit: committed K/V rows within rel-RMS 2e-2.
The batched variant (B = 4 requests sharing one weight stream, NEXT-2) runs the same protocol on every
request through the batched kernels (B*k = 24 frontier rows per draft pass, 4 x 289 verify rows).
"""
import numpy as np
import pytest

from synth.configs import QWEN7B, LLAMA8B, QWEN32B, GIB
from synth.prompts import mtbench_prompt
from oracle.decode import Session
from oracle.model import TargetWeights, draft_layers
from oracle.tree import Tree
from oracle.verify import accept, commit, argmax_and_gap
from oracle.numerics import bf16_bits_to_f64
from gpu_util import TOL_BF16, scale_of, assert_close_scaled, rel_rms
from test_gpu_decode import _check_selection

pytestmark = pytest.mark.gpu
SEED = 0x5EED
D, K_TOP, T_S = 48, 6, 0.2

WIDTHS = {
    "qwen7b": (QWEN7B.with_(name="qwen2.5-7b-2l", n_layers=2), 4),
    "llama8b": (LLAMA8B.with_(name="llama-3.1-8b-2l", n_layers=2), 4),
    "qwen32b": (QWEN32B.with_(name="qwen2.5-32b-2l", n_layers=2), 6),
}


def _prompt(cfg, idx, n):
    return [int(t) for t in mtbench_prompt(SEED, idx, cfg.vocab, n)]


def _first_token_ok(cfg, ors_logits_last, gpu_tok):
    lg = ors_logits_last
    return int(np.argmax(lg)) == gpu_tok or lg.max() - lg[gpu_tok] <= 2 * TOL_BF16 * scale_of(lg)


def _step_check(ss, ors, tr_tok, tr_par, tr_dep, tr_sc, g_draft, g_hid, am, gap, toks, path, cfg, slot=0):
    """One request's lockstep checks (steps 1-4).  Returns (selection flags, argmax flags)."""
    tree = Tree([int(t) for t in tr_tok], [int(p) for p in tr_par], [int(d) for d in tr_dep],
                [float(s) for s in tr_sc])
    o_draft, o_hid = ors.forward_tree("draft", tree, return_hidden=True)
    assert_close_scaled(g_draft, o_draft, what=f"slot {slot} draft logits")
    assert rel_rms(g_hid, o_hid) <= TOL_BF16, f"slot {slot} draft hidden"
    sel = _check_selection(tr_tok, tr_par, tr_sc, g_draft, D, K_TOP, T_S)
    o_logits = ors.forward_tree("target", tree)
    o_am, o_gap = argmax_and_gap(o_logits)
    eps = 2 * TOL_BF16 * scale_of(o_logits)
    bad = np.nonzero(np.asarray(am) != o_am)[0]
    assert np.all(o_gap[bad] <= eps), f"slot {slot}: unflagged argmax mismatch at nodes {bad}"
    o_path, o_emit = accept(tree, np.asarray(am))          # oracle walk on (GPU tree, GPU argmax)
    assert o_emit == toks and [0] + o_path == path, f"slot {slot}: accept"
    P = ors.kv.P
    commit(ors.kv, o_path)
    for l in range(cfg.n_layers):
        gk, gv = ss.debug_read_kv(l, slot * cfg.max_context + P, len(path))
        ok = ors.kv.K[l, P:P + len(path)].transpose(1, 0, 2)
        ov = ors.kv.V[l, P:P + len(path)].transpose(1, 0, 2)
        assert rel_rms(bf16_bits_to_f64(gk), ok) <= TOL_BF16 and rel_rms(bf16_bits_to_f64(gv), ov) <= TOL_BF16
    return sel, len(bad)


@pytest.mark.parametrize("width", list(WIDTHS), ids=list(WIDTHS))
def test_lockstep_full_width(cuda_required, width):
    from paper_2509_18344_b200.binding import SubSpec
    cfg, cap = WIDTHS[width]
    ss = SubSpec(cfg, cap * GIB, max_depth=D, max_top_k=K_TOP, max_chunk=256)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(4, 64)
    ors = Session(cfg, SEED, n_resident=0, mode="bf16-fp32", max_nodes=512)
    # a prompt longer than one prefill chunk (multi-chunk prefill), then MT-Bench-length decoding
    prompt = _prompt(cfg, 7, 300)
    first = ss.prefill(prompt, chunk=256)
    o_first = ors.prefill(prompt, chunk=256)
    if first != o_first:   # allowed only as a near-tie of the oracle's last prompt position
        lg = Session(cfg, SEED, n_resident=0, mode="bf16-fp32", max_nodes=512, target=ors.target,
                     dlayers=ors.dlayers).forward_tree("target", Tree(prompt, [i - 1 for i in range(len(prompt))],
                                                                      list(range(len(prompt))), [0.0] * len(prompt)))[-1]
        assert _first_token_ok(cfg, lg, first), "prefill first token"
    for l in range(cfg.n_layers):   # the prompt's committed K/V (both chunks)
        gk, gv = ss.debug_read_kv(l, 0, len(prompt))
        assert rel_rms(bf16_bits_to_f64(gk), ors.kv.K[l, :len(prompt)].transpose(1, 0, 2)) <= TOL_BF16
        assert rel_rms(bf16_bits_to_f64(gv), ors.kv.V[l, :len(prompt)].transpose(1, 0, 2)) <= TOL_BF16
    root = first
    flags = [0, 0]
    for step in range(2):
        tr = ss.draft_tree(D, K_TOP, T_S)
        n = len(tr["tokens"])
        assert n == 1 + K_TOP * D and tr["tokens"][0] == root
        g_draft, g_hid = ss.debug_forward(0, tr["tokens"], tr["parents"], hidden=True)
        am, gap = ss.verify_tree(n)
        toks, path = ss.accept_and_commit(D + 1)
        f = _step_check(ss, ors, tr["tokens"], tr["parents"], tr["depths"], tr["scores"], g_draft, g_hid, am, gap,
                        toks, path, cfg)
        flags = [flags[0] + f[0], flags[1] + f[1]]
        root = toks[-1]
    print(f"{width}: selection flags {flags[0]}, argmax flags {flags[1]}")
    ss.close()


def test_lockstep_full_width_batched(cuda_required):
    """B = 4 requests per GPU (NEXT-2) at the Qwen2.5-7B widths: every request's draft logits, hidden
    rows, tree, argmax, accepted path and committed KV against its own oracle session."""
    from paper_2509_18344_b200.binding import SubSpec
    cfg, cap = WIDTHS["qwen7b"]
    B = 4
    ss = SubSpec(cfg, 6 * GIB, max_depth=D, max_top_k=K_TOP, max_chunk=256, max_batch=B)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(4, 64)
    tw = TargetWeights(cfg, SEED, dtype=np.float32)
    dl = draft_layers(tw, 0)
    sess = [Session(cfg, SEED, n_resident=0, mode="bf16-fp32", max_nodes=512, target=tw, dlayers=dl) for _ in range(B)]
    ss.set_batch(B)
    roots = []
    for b in range(B):
        prompt = _prompt(cfg, 20 + b, 160 + 24 * b)   # ragged prompt lengths
        first = ss.prefill_slot(b, prompt)
        o_first = sess[b].prefill(prompt)
        assert first == o_first or _first_token_ok(cfg, sess[b].forward_tree(
            "target", Tree(prompt, [i - 1 for i in range(len(prompt))], list(range(len(prompt))),
                           [0.0] * len(prompt)))[-1], first)
        roots.append(first)
    for step in range(2):
        tr = ss.draft_tree(D, K_TOP, T_S, n_req=B)
        n = tr["tokens"].shape[1]
        assert all(tr["tokens"][b][0] == roots[b] for b in range(B))
        g_draft, g_hid = ss.debug_forward(0, tr["tokens"], tr["parents"], hidden=True)
        am, gap = ss.verify_tree(n, n_req=B)
        toks, paths = ss.accept_and_commit_batch(B, D + 1)
        for b in range(B):
            _step_check(ss, sess[b], tr["tokens"][b], tr["parents"][b], tr["depths"][b], tr["scores"][b], g_draft[b],
                        g_hid[b], am[b], gap[b], toks[b], paths[b], cfg, slot=b)
            roots[b] = toks[b][-1]
    ss.close()
