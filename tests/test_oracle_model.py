"""Pins for oracle/model.py (O.3) and the decode loop (O.7-O.10).

* library special case: a chain forward equals an independent torch-CPU fp64 composition of
  scaled_dot_product_attention(is_causal=True), rms_norm, silu and complex-rotation RoPE;
* chain == sequential and path replay, bitwise in exact mode;
* mask isolation: perturbing a non-ancestor changes nothing;
* chunked prefill == unchunked, bitwise;
* committed KV after SD == AR replay KV, bitwise;
* greedy losslessness SD == AR and full acceptance for a
  self-draft with T = 0.01.
"""
import numpy as np
import pytest
import torch

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt, uniform_prompt
from oracle.model import draft_layers, TargetWeights
from oracle.tree import Tree
from oracle.decode import Session, ar_generate, sd_generate

SEED = 0x5EED


@pytest.fixture(scope="module")
def tiny_target():
    return TargetWeights(TINY, SEED)


def _chain(tokens):
    n = len(tokens)
    return Tree(list(tokens), [i - 1 for i in range(n)], list(range(n)), [0.0] * n)


def _torch_chain_logits(cfg, tw, tokens):
    """Independent fp64 implementation of a causal forward using torch library ops."""
    T = torch.float64
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(T)
    n, d, nh, nkv = len(tokens), cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    x = f(tw.embed)[torch.tensor(tokens)]
    pos = torch.arange(n, dtype=T)
    inv = cfg.rope_theta ** (-torch.arange(d // 2, dtype=T) * 2.0 / d)
    rot = torch.polar(torch.ones(n, d // 2, dtype=T), pos[:, None] * inv[None, :])

    def rope(t):                      # t: [heads, n, d], rotate-half as a complex product
        z = torch.complex(t[..., : d // 2], t[..., d // 2:]) * rot
        return torch.cat([z.real, z.imag], dim=-1)

    for lw in tw.layers:
        h = torch.nn.functional.rms_norm(x, (cfg.hidden,), f(lw["attn_norm"]), eps=cfg.rms_eps)
        q = torch.nn.functional.linear(h, f(lw["wq"]), f(lw["bq"]) if cfg.qkv_bias else None)
        k = torch.nn.functional.linear(h, f(lw["wk"]), f(lw["bk"]) if cfg.qkv_bias else None)
        v = torch.nn.functional.linear(h, f(lw["wv"]), f(lw["bv"]) if cfg.qkv_bias else None)
        q = rope(q.view(n, nh, d).transpose(0, 1))
        k = rope(k.view(n, nkv, d).transpose(0, 1)).repeat_interleave(nh // nkv, dim=0)
        v = v.view(n, nkv, d).transpose(0, 1).repeat_interleave(nh // nkv, dim=0)
        o = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True)[0]
        x = x + torch.nn.functional.linear(o.transpose(0, 1).reshape(n, -1), f(lw["wo"]))
        h2 = torch.nn.functional.rms_norm(x, (cfg.hidden,), f(lw["mlp_norm"]), eps=cfg.rms_eps)
        a = torch.nn.functional.silu(torch.nn.functional.linear(h2, f(lw["wg"]))) * \
            torch.nn.functional.linear(h2, f(lw["wu"]))
        x = x + torch.nn.functional.linear(a, f(lw["wd"]))
    hf = torch.nn.functional.rms_norm(x, (cfg.hidden,), f(tw.final_norm), eps=cfg.rms_eps)
    return torch.nn.functional.linear(hf, f(tw.head)).numpy()


@pytest.mark.parametrize("cfg", [TINY, SMALL], ids=["tiny", "small"])
def test_chain_forward_matches_torch_library(cfg):
    tw = TargetWeights(cfg, SEED)
    toks = [int(t) for t in uniform_prompt(3, 0, cfg.vocab, 12)]
    s = Session(cfg, SEED, n_resident=cfg.n_layers, target=tw, max_nodes=64)
    got = s.forward_tree("target", _chain(toks))
    ref = _torch_chain_logits(cfg, tw, toks)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)


def test_chain_equals_sequential_bitwise(tiny_target):
    toks = [int(t) for t in uniform_prompt(5, 1, TINY.vocab, 20)]
    a = Session(TINY, SEED, target=tiny_target, max_nodes=64)
    la = a.forward_tree("target", _chain(toks))
    b = Session(TINY, SEED, target=tiny_target, max_nodes=64)
    for i, t in enumerate(toks):
        lb = b.forward_tree("target", _chain([t]))
        b.accept_and_commit(_chain([t]), [-1])        # commit the single root
        assert np.array_equal(la[i], lb[0])
    a.accept_and_commit(_chain(toks), toks[1:] + [-1])
    assert a.kv.P == b.kv.P == len(toks)
    assert np.array_equal(a.kv.K[:, :a.kv.P], b.kv.K[:, :b.kv.P])
    assert np.array_equal(a.kv.V[:, :a.kv.P], b.kv.V[:, :b.kv.P])


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_path_replay_and_mask_isolation(tiny_target, mode):
    rng = np.random.default_rng(7)
    prompt = [int(t) for t in uniform_prompt(6, 2, TINY.vocab, 9)]
    parents = [-1, 0, 0, 1, 1, 2, 4]
    depths = [0, 1, 1, 2, 2, 2, 3]
    toks = [int(t) for t in rng.integers(0, TINY.vocab, 7)]
    tree = Tree(toks, parents, depths, [0.0] * 7)

    def fresh():
        s = Session(TINY, SEED, target=tiny_target, mode=mode, max_nodes=64)
        s.prefill(prompt)
        return s
    s = fresh()
    lt = s.forward_tree("target", tree)
    for i in range(7):
        r = fresh()
        anc = tree.ancestors(i)
        lr = r.forward_tree("target", _chain([toks[a] for a in anc]))
        assert np.array_equal(lt[i], lr[-1]), f"path replay node {i}"
    # perturb node 5 (not an ancestor of 3, 4, 6): their logits are unchanged
    t2 = Tree(list(toks), parents, depths, [0.0] * 7)
    t2.tokens[5] = (toks[5] + 1) % TINY.vocab
    l2 = fresh().forward_tree("target", t2)
    for i in (0, 1, 2, 3, 4, 6):
        assert np.array_equal(lt[i], l2[i])
    assert not np.array_equal(lt[5], l2[5])


@pytest.mark.parametrize("chunk", [1, 7, 256, 45])
def test_chunked_prefill_equals_unchunked(tiny_target, chunk):
    prompt = [int(t) for t in uniform_prompt(8, 3, TINY.vocab, 45)]
    ref = Session(TINY, SEED, target=tiny_target, max_nodes=256)
    t_ref = ref.prefill(prompt, chunk=len(prompt))
    s = Session(TINY, SEED, target=tiny_target, max_nodes=256)
    t = s.prefill(prompt, chunk=chunk)
    assert t == t_ref and s.kv.P == ref.kv.P == 45
    assert np.array_equal(s.kv.K[:, :45], ref.kv.K[:, :45]) and np.array_equal(s.kv.V[:, :45], ref.kv.V[:, :45])


@pytest.mark.parametrize("mode", ["exact", "bf16"])
@pytest.mark.parametrize("n_resident,bits", [(0, 4), (1, 4), (0, 8)])
def test_sd_lossless_and_cache_exact(tiny_target, mode, n_resident, bits):
    for p in range(3):
        prompt = mtbench_prompt(SEED, p, TINY.vocab, 32)
        ar, sa = ar_generate(TINY, prompt, 40, session=Session(TINY, SEED, target=tiny_target, mode=mode))
        for D, k in ((1, 1), (4, 6), (6, 2)):
            sd, taus, ss = sd_generate(TINY, prompt, 40, D, k, 0.2, session=Session(
                TINY, SEED, n_resident=n_resident, bits=bits, target=tiny_target, mode=mode,
                max_nodes=max(256, 1 + k * D)))
            assert sd == ar, (p, D, k)
            assert all(1 <= t <= D + 1 for t in taus)
            # committed cache == AR replay over the same tokens (compare the common prefix)
            P = min(ss.kv.P, sa.kv.P)
            assert np.array_equal(ss.kv.K[:, :P], sa.kv.K[:, :P]) and np.array_equal(ss.kv.V[:, :P], sa.kv.V[:, :P])


def test_self_draft_full_acceptance(tiny_target):
    # all layers shared (draft == target), sharpening T = 0.01: tau = D+1 every step
    D, k = 5, 3
    prompt = mtbench_prompt(SEED, 4, TINY.vocab, 32)
    sd, taus, _ = sd_generate(TINY, prompt, 1 + 6 * (D + 1), D, k, 0.01, session=Session(
        TINY, SEED, n_resident=TINY.n_layers, target=tiny_target, max_nodes=256))
    assert taus == [D + 1] * 6


def test_capacity_clamp_keeps_losslessness(tiny_target):
    cfg = TINY.with_(max_context=64)
    tw = TargetWeights(cfg, SEED)
    prompt = mtbench_prompt(SEED, 5, cfg.vocab, 32)
    ar, _ = ar_generate(cfg, prompt, 31, session=Session(cfg, SEED, target=tw))
    s = Session(cfg, SEED, target=tw, max_nodes=256)
    sd, taus, s = sd_generate(cfg, prompt, 31, 6, 4, 0.2, session=s)
    assert sd == ar and s.kv.P <= cfg.max_context
    with pytest.raises(ValueError):
        s2 = Session(cfg, SEED, target=tw, max_nodes=256)
        s2.prefill(list(range(65)))


def test_sd_lossless_many_prompts(tiny_target):
    """O.8 at breadth (>= 200 prompts, D <= 48): for 200 MT-Bench-shaped prompts, SubSpec's
    greedy output equals plain greedy AR ("lossless"), over trees from D = 48, k = 6 (the
    paper's setting) down to a chain, in the GPU's bf16-emulation mode."""
    combos = [(48, 6), (16, 2), (4, 6), (1, 1), (8, 3), (24, 4), (2, 2), (4, 6), (12, 1), (6, 6),
              (32, 2), (16, 2), (4, 6), (1, 1), (8, 3), (24, 4), (2, 2), (4, 6), (12, 1), (6, 6)]
    views = {nr: draft_layers(tiny_target, nr) for nr in (0, 1)}   # the draft views, built once
    for p in range(200):
        prompt = mtbench_prompt(SEED, 2000 + p, TINY.vocab, 24 + (p * 7) % 40)
        ar, _ = ar_generate(TINY, prompt, 8, session=Session(TINY, SEED, target=tiny_target, mode="bf16"))
        D, k = combos[p % len(combos)]
        sd, taus, _ = sd_generate(TINY, prompt, 8, D, k, 0.2, session=Session(
            TINY, SEED, target=tiny_target, dlayers=views[p % 2], mode="bf16", max_nodes=max(256, 1 + k * D)))
        assert sd == ar, (p, D, k)
        assert all(1 <= t <= D + 1 for t in taus)
