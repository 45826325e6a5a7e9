"""Pins for the oracle's full-width pieces: the node-batched forward (forward_nodes_batched, the
fp32-BLAS mode of SURVEY §8(c)) and the draft view (draft_layers).

* library special case: the batched forward of a chain (fp64 weights) equals an independent torch-CPU
  composition of scaled_dot_product_attention(is_causal=True), rms_norm, silu and complex RoPE;
* tree mask: perturbing a non-ancestor's token changes nothing, a sibling's own
  logits equal its path replay;
* the fp32 mode (fp32 weights, fp32 products) stays within fp32 rounding of the fp64 one;
* draft_layers: shared layers are the target's own; substituted layers replace exactly the seven
  linear matrices (norms and biases kept); every substituted 64-group lies on its
  own grid z + c*s, c in 0..15, within the bound of reading R5, and differs from W.
"""
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt
from oracle.model import TargetWeights, KVCache, draft_layers, forward_nodes, forward_nodes_batched, LAYER_MATS
from oracle.quant import quantize
from test_oracle_model import _torch_chain_logits

SEED = 0x5EED


def _run(fn, cfg, tw, layers, tokens, parents, mode, P_prefix=None):
    kv = KVCache(cfg, 64)
    n = len(tokens)
    depth = [0] * n
    anc = []
    for i in range(n):
        if parents[i] >= 0:
            depth[i] = depth[parents[i]] + 1
        a, c = [], i
        while c >= 0:
            a.append(c)
            c = parents[c]
        anc.append(a[::-1])
    return fn(cfg, layers, tw, kv, tokens, list(range(n)), depth, anc, mode)


def test_batched_chain_equals_torch_library():
    tw = TargetWeights(TINY, SEED)
    toks = [int(t) for t in mtbench_prompt(SEED, 5, TINY.vocab, 12)]
    got = _run(forward_nodes_batched, TINY, tw, tw.layers, toks, [i - 1 for i in range(len(toks))], "exact")
    ref = _torch_chain_logits(TINY, tw, toks)
    assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))


def test_batched_equals_per_node_exact_and_bf16():
    tw = TargetWeights(SMALL, SEED)
    toks = [3, 17, 99, 5, 41, 7, 8]
    par = [-1, 0, 0, 1, 1, 2, 5]
    for mode, tol in (("exact", 1e-11), ("bf16", 2e-2)):
        a = _run(forward_nodes_batched, SMALL, tw, tw.layers, toks, par, mode)
        b = _run(forward_nodes, SMALL, tw, tw.layers, toks, par, mode)
        assert np.max(np.abs(a - b)) <= tol * max(1.0, np.max(np.abs(b))), mode


def test_batched_tree_mask_and_path_replay():
    tw = TargetWeights(TINY, SEED)
    toks = [3, 17, 99, 5, 41, 7, 8]
    par = [-1, 0, 0, 1, 1, 2, 5]
    base = _run(forward_nodes_batched, TINY, tw, tw.layers, toks, par, "exact")
    pert = list(toks)
    pert[2] = 500                     # node 2 is not an ancestor of nodes 1, 3, 4
    out = _run(forward_nodes_batched, TINY, tw, tw.layers, pert, par, "exact")
    for i in (0, 1, 3, 4):
        assert np.allclose(out[i], base[i], rtol=0, atol=1e-12)
    # node 6's logits == the chain root -> 2 -> 5 -> 6 replayed alone
    chain = _run(forward_nodes_batched, TINY, tw, tw.layers, [3, 99, 7, 8], [-1, 0, 1, 2], "exact")
    assert np.allclose(chain[3], base[6], rtol=0, atol=1e-10 * np.max(np.abs(base[6])))


def test_fp32_mode_within_fp32_rounding_of_fp64():
    t64 = TargetWeights(SMALL, SEED)
    t32 = TargetWeights(SMALL, SEED, dtype=np.float32)
    for l in range(SMALL.n_layers):
        for k, v in t64.layers[l].items():
            assert np.array_equal(t32.layers[l][k].astype(np.float64), v)   # bf16 values: exact in fp32
    toks = [int(t) for t in mtbench_prompt(SEED, 6, SMALL.vocab, 9)]
    par = [i - 1 for i in range(len(toks))]
    a = _run(forward_nodes_batched, SMALL, t32, t32.layers, toks, par, "exact")
    b = _run(forward_nodes_batched, SMALL, t64, t64.layers, toks, par, "exact")
    assert np.max(np.abs(a - b)) <= 1e-4 * max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_draft_layers_substitute_exactly_the_offloaded_matrices(dtype):
    cfg = SMALL
    tw = TargetWeights(cfg, SEED, dtype=dtype)
    assert all(a is b for a, b in zip(draft_layers(tw, cfg.n_layers), tw.layers))   # all shared
    dl = draft_layers(tw, 1, bits=4, block_rows=100)   # odd block size: blocks split inside tiles
    assert dl[0] is tw.layers[0]
    for l in range(1, cfg.n_layers):
        tgt, sub = tw.layers[l], dl[l]
        assert set(sub) == set(tgt)
        for k in tgt:
            if k not in LAYER_MATS:
                assert np.array_equal(sub[k], tgt[k]), k          # norms, biases: the target's
        for k in LAYER_MATS:
            W = np.asarray(tgt[k], np.float64)
            Wh = np.asarray(sub[k], np.float64)
            assert not np.array_equal(W, Wh), k                    # really a substitute
            codes, s, z = quantize(W, 4, 64)
            N, K = W.shape
            c = (Wh.reshape(N, K // 64, 64) - z[..., None]) / s[..., None]
            assert np.array_equal(c, np.rint(c)) and c.min() >= 0 and c.max() <= 15, k   # on the group's grid
            err = np.abs(Wh - W).reshape(N, K // 64, 64)
            bound = s[..., None] / 2 + 2.0 ** -8 * np.abs(W.reshape(N, K // 64, 64)) + 1e-30
            clamp = np.abs(W.reshape(N, K // 64, 64) - (z[..., None] + 15 * s[..., None]))   # bf16 s below (M-m)/15
            assert np.all(err <= np.maximum(bound, clamp + 1e-12)), k
