"""End-to-end GPU parity of the SubSpec step against the oracle (SURVEY.md §8(c) lockstep protocol).

Per step, starting from a shared state:
 1. draft: GPU draft logits on its own tree vs the oracle's (bf16-emulation mode, teacher-forced on
    the GPU tree) within 2e-2 x logit scale; the oracle's sharpened top-k run on the GPU's logits must
    reproduce the GPU's tree (exact up to flagged fp32 near-ties);
 2. verify: GPU target argmax vs the oracle's argmax on the GPU tree; disagreements are allowed only
    where the oracle's top-1/top-2 gap <= 2 x tol x scale (flagged);
 3. accept: the oracle's acceptance walk on (GPU tree, GPU argmax) reproduces the GPU's path and
    emitted tokens bit-exactly;
 4. commit: committed K/V rows agree within tolerance; both sides adopt the GPU's tokens.
Separately: GPU SubSpec output == GPU AR output bitwise (batch-invariant target path), and == the
oracle's greedy AR output up to flagged positions.
"""
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt
from oracle.decode import Session, ar_generate
from oracle.tree import Tree, tempered_log_softmax, select_topk
from oracle.verify import accept, commit, argmax_and_gap
from oracle.numerics import bf16_bits_to_f64
from gpu_util import TOL_BF16, scale_of, assert_close_scaled, rel_rms

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _gpu(cfg, n_resident, D, k, cap=512 << 20, max_chunk=256, quant="rtn"):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, cap, max_depth=D, max_top_k=k, max_chunk=max_chunk)
    ss.load_synthetic(SEED, n_resident=n_resident)
    ss.build_substitutes(4, 64, method=quant)
    return ss


def _check_selection(tree_tok, tree_par, tree_score, gpu_logits, D, k, T):
    """Oracle top-k on the GPU's draft logits must rebuild the GPU tree (flags: fp32 ties)."""
    flags = 0
    scores = {0: 0.0}
    for d in range(D):
        fr = [0] if d == 0 else list(range(1 + (d - 1) * k, 1 + d * k))
        lp = np.stack([tempered_log_softmax(gpu_logits[f].astype(np.float64), T) for f in fr])
        picked = select_topk(fr, [scores[f] for f in fr], lp, k)
        got = [(int(tree_par[c]), int(tree_tok[c])) for c in range(1 + d * k, 1 + (d + 1) * k)]
        want = [(p, t) for p, t, _ in picked]
        if got != want:
            # allowed only when the k-th and (k+1)-th candidate scores are within fp32 noise
            sc = (np.array([scores[f] for f in fr])[:, None] + lp).reshape(-1)
            srt = np.sort(sc)[::-1]
            assert srt[k - 1] - srt[k] <= 1e-4 * max(1.0, abs(srt[k])), f"depth {d}: {got} != {want}"
            flags += 1
        for c in range(1 + d * k, 1 + (d + 1) * k):   # continue on the GPU's tree
            scores[c] = float(tree_score[c])
    return flags


@pytest.mark.parametrize("cfg,n_res,D,k,quant", [(TINY, 1, 4, 6, "rtn"), (SMALL, 1, 4, 6, "rtn"),
                                                 (SMALL, 0, 3, 4, "rtn"), (SMALL, 0, 4, 6, "hqq")],
                         ids=["tiny-D4k6", "small-D4k6", "small-allsub-D3k4", "small-allsub-hqq-D4k6"])
def test_lockstep(cuda_required, cfg, n_res, D, k, quant):
    T = 0.2
    ss = _gpu(cfg, n_res, D, k, quant=quant)
    ors = Session(cfg, SEED, n_resident=n_res, mode="bf16", max_nodes=max(256, 1 + k * D), quant=quant)
    prompt = mtbench_prompt(SEED, 1, cfg.vocab, 40)
    first = ss.prefill(prompt)
    o_first = ors.prefill(prompt)
    assert first == o_first
    root = first
    sel_flags = arg_flags = 0
    for step in range(4):
        tr = ss.draft_tree(D, k, T)
        n = len(tr["tokens"])
        assert n == 1 + k * D and tr["tokens"][0] == root
        assert np.all(tr["depths"] == [0] + [1 + (i - 1) // k for i in range(1, n)])
        g_draft = ss.debug_forward(0, tr["tokens"], tr["parents"])
        tree = Tree([int(t) for t in tr["tokens"]], [int(p) for p in tr["parents"]],
                    [int(d) for d in tr["depths"]], [float(s) for s in tr["scores"]])
        o_draft = ors.forward_tree("draft", tree)
        assert_close_scaled(g_draft[:1 + k * (D - 1)], o_draft[:1 + k * (D - 1)], what="draft logits")
        sel_flags += _check_selection(tr["tokens"], tr["parents"], tr["scores"], g_draft, D, k, T)
        am, gap = ss.verify_tree(n)
        o_logits = ors.forward_tree("target", tree)
        o_am, o_gap = argmax_and_gap(o_logits)
        eps = 2 * TOL_BF16 * scale_of(o_logits)
        bad = np.nonzero(am != o_am)[0]
        assert np.all(o_gap[bad] <= eps), f"unflagged argmax mismatch at nodes {bad}"
        arg_flags += len(bad)
        toks, path = ss.accept_and_commit(D + 1)
        o_path, o_emit = accept(tree, am)          # oracle walk on (GPU tree, GPU argmax)
        assert o_emit == toks and [0] + o_path == path
        P = ors.kv.P
        commit(ors.kv, o_path)
        for l in range(cfg.n_layers):
            gk, gv = ss.debug_read_kv(l, P, len(path))
            ok = ors.kv.K[l, P:P + len(path)].transpose(1, 0, 2)
            ov = ors.kv.V[l, P:P + len(path)].transpose(1, 0, 2)
            assert rel_rms(bf16_bits_to_f64(gk), ok) <= TOL_BF16 and rel_rms(bf16_bits_to_f64(gv), ov) <= TOL_BF16
        root = toks[-1]
    print(f"selection flags {sel_flags}, argmax flags {arg_flags}")
    ss.close()


@pytest.mark.parametrize("cfg,n_res,D,k", [(TINY, 1, 4, 6), (SMALL, 1, 4, 6), (SMALL, 0, 6, 2)],
                         ids=["tiny", "small", "small-allsub"])
def test_sd_equals_gpu_ar_and_oracle_ar(cuda_required, cfg, n_res, D, k):
    ss = _gpu(cfg, n_res, D, k)
    for p in range(3):
        prompt = mtbench_prompt(SEED, p, cfg.vocab, 32 + 17 * p)
        sd, hist = ss.generate(prompt, 40, D, k, 0.2)
        ar, _ = ss.generate(prompt, 40, 0, 1, 0.2)
        assert sd == ar, f"prompt {p}: SubSpec output differs from the GPU AR output"
        ref, s = ar_generate(cfg, prompt, 40, seed=SEED, mode="bf16")
        if sd != ref:   # allowed only from a flagged near-tie on, judged on the oracle's teacher-forced logits
            j = next(i for i in range(40) if sd[i] != ref[i])
            o = Session(cfg, SEED, mode="bf16", max_nodes=512)
            seq = [int(t) for t in prompt] + sd[:j]
            lg = o.forward_tree("target", Tree(seq, [i - 1 for i in range(len(seq))], list(range(len(seq))),
                                               [0.0] * len(seq)))[-1]
            assert lg.max() - lg[sd[j]] <= 2 * TOL_BF16 * scale_of(lg), f"prompt {p}: unflagged divergence at {j}"
    ss.close()


def test_self_draft_full_acceptance(cuda_required):
    # all layers shared (draft == target weights) and T = 0.01: tau = D+1, up to the
    # bf16 GEMV-vs-GEMM rounding of the draft path flipping a rare near-tie
    D, k = 4, 2
    ss = _gpu(SMALL, SMALL.n_layers, D, k)
    prompt = mtbench_prompt(SEED, 2, SMALL.vocab, 32)
    out, hist = ss.generate(prompt, 1 + 8 * (D + 1), D, k, 0.01)
    assert hist[D + 1] >= 0.75 * hist.sum(), hist
    ss.close()


def test_capacity_clamp(cuda_required):
    cfg = TINY.with_(max_context=96)
    ss = _gpu(cfg, 1, 6, 4, max_chunk=128)
    prompt = mtbench_prompt(SEED, 3, cfg.vocab, 48)
    sd, _ = ss.generate(prompt, 49, 6, 4, 0.2, chunk=128)      # reaches P = 96 exactly
    ar, _ = ss.generate(prompt, 49, 0, 1, 0.2, chunk=128)
    assert sd == ar and len(sd) == 49
    st = ss.stats()
    assert st["committed_len"] <= cfg.max_context
    ss.close()


def test_config1_100_seeds(cuda_required):
    """BASELINE config 1 at SURVEY §8(d)'s breadth: 100 seeded 32-token prompts x 64 new tokens on the tiny
    model (layer 0 shared, layer 1 a 4-bit substitute, D = 4, k = 6): the GPU SubSpec output equals the GPU
    AR output bitwise and the oracle's greedy AR output (bf16 emulation) up to flagged near-ties."""
    from gpu_util import assert_matches_oracle_ar
    D, k = 4, 6
    ss = _gpu(TINY, 1, D, k)
    flags = 0
    for p in range(100):
        prompt = mtbench_prompt(SEED + p, p, TINY.vocab, 32)
        sd, _ = ss.generate(prompt, 64, D, k, 0.2)
        ar, _ = ss.generate(prompt, 64, 0, 1, 0.2)
        assert sd == ar, f"seed {p}: SubSpec output differs from the GPU AR output"
        flags += assert_matches_oracle_ar(TINY, prompt, sd, SEED)
    # every divergence from the oracle is a flagged near-tie (asserted per token above); bf16 rounding
    # flips such ties at a low rate (measured 39 of 6400 tokens on B200)
    print(f"near-tie flags over 100 x 64 tokens: {flags}")
    assert flags <= 0.02 * 100 * 64
    ss.close()
