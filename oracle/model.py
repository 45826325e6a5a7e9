"""O.3 — forward of a set of tree nodes.  Test infrastructure only.

Model: decoder-only, pre-RMSNorm, rotary positions, gated-SiLU MLP, untied
head ("pre-RMS-norm, rotary positions, gated-SiLU MLP, untied
output head"), optional Qwen QKV bias.

Tree decoding: "Multiple branching token paths are flattened and evaluated in
one forward pass.  Positional encodings and attention masks are modified to
preserve tree structure dependency" (§2.2).  Reading R9: a node's
position is P + depth; its keys are the committed prefix [0, P) followed by
its ancestors root..self in depth order (the ancestor-closure mask,
SPEC.md:70).  The committed prefix holds the *target's* K/V and is read by
both draft and target (shared KV-cache); every forwarded
node writes its own K/V into its tree slot — draft values during drafting,
which the target overwrites during verification (Fig. 3 right).

Layer math for each layer, processed over all nodes before the next layer:
    h  = rmsnorm(x) * g_attn
    q,k,v = W_q h (+b_q), W_k h (+b_k), W_v h (+b_v);  RoPE(q, k) at pos
    store k, v in the node's tree slot
    per head: a = softmax_{keys}(q.k / sqrt(d_h));  o = sum a v   (GQA: kv head = hq // (n_h/n_kv))
    x += W_o concat(o) ;  h2 = rmsnorm(x) * g_mlp ;  x += W_d (silu(W_g h2) * (W_u h2))
Final: logits = Head (rmsnorm(x) * g_final).

mode "exact": float64 throughout.  mode "bf16": additionally rounds to bf16
(RNE) at the GPU's named rounding points (reading R3): h, h2 and the final
normed vector; q, k, v after bias and RoPE; the attention output; the
SiLU-mul activation.  Logits, scores, softmax and the residual stream are
never rounded.  Every node's arithmetic is a per-row op sequence identical to
what an autoregressive forward would do at that position, so chain ==
sequential and path replay hold bitwise.

mode "bf16-fp32" (SURVEY §8(c) "fp32-BLAS mode", for the full-width shapes): the
same steps and rounding points, with the weights held in float32 (bf16 values and
the substitutes' code*s + z are exact in fp32) and each linear map one float32
matrix product over all forwarded nodes (forward_nodes_batched).  Only the
summation order and fp32 accumulation of the products differ from "bf16".
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from synth.configs import ModelConfig
from synth.weights import tensor_specs, gen_tensor_bits
from .numerics import bf16_bits_to_f64, round_bf16, rmsnorm, silu, rope_rotate_half
from .quant import substitute_matrix

LAYER_MATS = ("wq", "wk", "wv", "wo", "wg", "wu", "wd")


class TargetWeights:
    """The target's bf16 weights as float64 (or, for mode "bf16-fp32", float32) arrays; every value
    is exactly a bf16.  Matrices are generated in row blocks of `block_rows` (memory)."""

    def __init__(self, cfg: ModelConfig, seed: int, layers=None, dtype=np.float64, block_rows=4096):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.layers = [dict() for _ in range(cfg.n_layers)]
        want = set(range(cfg.n_layers)) if layers is None else set(layers)

        def gen(tid, shape, kind, sigma):
            if len(shape) == 1:
                return bf16_bits_to_f64(gen_tensor_bits(seed, tid, shape, kind, sigma)).astype(self.dtype)
            out = np.empty(shape, dtype=self.dtype)

            def block(r0):   # row blocks are independent (counter-based generator): threads
                r1 = min(shape[0], r0 + block_rows)
                out[r0:r1] = bf16_bits_to_f64(gen_tensor_bits(seed, tid, shape, kind, sigma, rows=slice(r0, r1)))
            with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
                list(ex.map(block, range(0, shape[0], block_rows)))
            return out

        for tid, name, shape, kind, sigma in tensor_specs(cfg):
            if name.startswith("l"):
                l = int(name[1:name.index(".")])
                if l not in want:
                    continue
                self.layers[l][name.split(".", 1)[1]] = gen(tid, shape, kind, sigma)
            else:
                setattr(self, name, gen(tid, shape, kind, sigma))


def draft_layers(target: TargetWeights, n_resident: int, bits=4, group=64, block_rows=2048, method="rtn"):
    """Draft model view (SPEC.md:214-222 build_draft_view):
    layers [0, n_resident) are Shared (the target's own dict); the rest are
    Substitute: every linear matrix replaced by its dequantized low-bit copy,
    norms and biases kept (reading R6).  Groups are rows' 64
    consecutive inputs, so the substitute is computed row block by row block."""
    out = []
    dt = getattr(target, "dtype", np.dtype(np.float64))
    for l, lw in enumerate(target.layers):
        if l < n_resident:
            out.append(lw)
        else:
            sub = dict(lw)
            for m in LAYER_MATS:
                w = lw[m]
                q = np.empty(w.shape, dtype=dt)

                def block(r0, w=w, q=q):   # groups lie inside rows: row blocks are independent
                    blk = substitute_matrix(np.asarray(w[r0:r0 + block_rows], dtype=np.float64), bits, group, method)
                    q[r0:r0 + block_rows] = blk
                    if dt != np.float64:   # code*s + z must be exact in the storage type
                        assert np.array_equal(q[r0:r0 + block_rows].astype(np.float64), blk), "substitute not exact in fp32"
                with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
                    list(ex.map(block, range(0, w.shape[0], block_rows)))
                sub[m] = q
            out.append(sub)
    return out


class KVCache:
    """Shared KV-cache: committed region [0, P) plus per-node tree slots."""

    def __init__(self, cfg: ModelConfig, max_nodes: int):
        L, C, nkv, d = cfg.n_layers, cfg.max_context, cfg.n_kv_heads, cfg.head_dim
        self.cfg = cfg
        self.K = np.zeros((L, C, nkv, d))
        self.V = np.zeros((L, C, nkv, d))
        self.tK = np.zeros((L, max_nodes, nkv, d))
        self.tV = np.zeros((L, max_nodes, nkv, d))
        self.P = 0


def forward_nodes(cfg: ModelConfig, layers, target: TargetWeights, kv: KVCache,
                  tokens, slots, positions, ancestors, mode="exact", return_hidden=False):
    """Forward the given nodes through `layers` (a list of per-layer weight dicts).

    tokens[i], slots[i] (tree slot written), positions[i], ancestors[i] (tree
    slots root..self).  Returns logits [n, V] (and the final normed hidden)."""
    R = round_bf16 if mode == "bf16" else (lambda a: a)
    n = len(tokens)
    H, nh, nkv, d = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    grp = nh // nkv
    P = kv.P
    x = [target.embed[int(t)].copy() for t in tokens]
    inv_sqrt_d = 1.0 / np.sqrt(d)
    for l, lw in enumerate(layers):
        qs = []
        for i in range(n):
            h = R(rmsnorm(x[i], lw["attn_norm"], cfg.rms_eps))
            q = lw["wq"] @ h
            k = lw["wk"] @ h
            v = lw["wv"] @ h
            if cfg.qkv_bias:
                q = q + lw["bq"]
                k = k + lw["bk"]
                v = v + lw["bv"]
            q = q.reshape(nh, d)
            k = k.reshape(nkv, d)
            q = np.stack([rope_rotate_half(q[j], positions[i], cfg.rope_theta, d) for j in range(nh)])
            k = np.stack([rope_rotate_half(k[j], positions[i], cfg.rope_theta, d) for j in range(nkv)])
            qs.append(R(q))
            kv.tK[l, slots[i]] = R(k)
            kv.tV[l, slots[i]] = R(v.reshape(nkv, d))
        for i in range(n):
            anc = list(ancestors[i])
            o = np.empty((nh, d))
            for hq in range(nh):
                g = hq // grp
                Kall = np.concatenate([kv.K[l, :P, g], kv.tK[l, anc, g]])
                Vall = np.concatenate([kv.V[l, :P, g], kv.tV[l, anc, g]])
                s = (Kall @ qs[i][hq]) * inv_sqrt_d
                e = np.exp(s - s.max())
                p = e / e.sum()
                o[hq] = p @ Vall
            o = R(o.reshape(-1))
            x[i] = x[i] + lw["wo"] @ o
            h2 = R(rmsnorm(x[i], lw["mlp_norm"], cfg.rms_eps))
            a = R(silu(lw["wg"] @ h2) * (lw["wu"] @ h2))
            x[i] = x[i] + lw["wd"] @ a
    hf = [R(rmsnorm(x[i], target.final_norm, cfg.rms_eps)) for i in range(n)]
    logits = np.stack([target.head @ hf[i] for i in range(n)])
    if return_hidden:
        return logits, np.stack(hf)
    return logits


def _rmsnorm_rows(X, g, eps):
    """rmsnorm of every row of X (the per-row definition of numerics.rmsnorm)."""
    return X / np.sqrt(np.mean(X * X, axis=1, keepdims=True) + eps) * g


def _rope_rows(Q, positions, theta, d):
    """Rotate-half RoPE of every head vector: Q [n, heads, d], positions [n] (numerics.rope_rotate_half)."""
    half = d // 2
    j = np.arange(half, dtype=np.float64)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * theta ** (-2.0 * j / d)   # [n, half]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = Q[..., :half], Q[..., half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def forward_nodes_batched(cfg: ModelConfig, layers, target: TargetWeights, kv: KVCache,
                          tokens, slots, positions, ancestors, mode="bf16-fp32", return_hidden=False):
    """forward_nodes with each linear map applied to all nodes as one matrix product in the weights'
    storage type (float32 for mode "bf16-fp32").  Same steps, order and rounding points as
    forward_nodes; every node still attends only to its own key list (prefix ++ ancestors)."""
    R = round_bf16 if mode in ("bf16", "bf16-fp32") else (lambda a: a)
    n = len(tokens)
    H, nh, nkv, d = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    grp = nh // nkv
    P = kv.P
    wdt = getattr(target, "dtype", np.dtype(np.float64))

    def mm(A, W):   # A [n, K] (float64 values), W [N, K] -> [n, N] float64
        return (A.astype(wdt) @ W.T).astype(np.float64)

    X = np.stack([target.embed[int(t)].astype(np.float64) for t in tokens])
    inv_sqrt_d = 1.0 / np.sqrt(d)
    slots = list(slots)
    for l, lw in enumerate(layers):
        Hn = R(_rmsnorm_rows(X, lw["attn_norm"].astype(np.float64), cfg.rms_eps))
        Q, Kx, Vx = mm(Hn, lw["wq"]), mm(Hn, lw["wk"]), mm(Hn, lw["wv"])
        if cfg.qkv_bias:
            Q = Q + lw["bq"].astype(np.float64)
            Kx = Kx + lw["bk"].astype(np.float64)
            Vx = Vx + lw["bv"].astype(np.float64)
        Q = R(_rope_rows(Q.reshape(n, nh, d), positions, cfg.rope_theta, d))
        Kx = R(_rope_rows(Kx.reshape(n, nkv, d), positions, cfg.rope_theta, d))
        kv.tK[l, slots] = Kx
        kv.tV[l, slots] = R(Vx.reshape(n, nkv, d))
        O = np.empty((n, nh, d))
        for i in range(n):
            anc = list(ancestors[i])
            for g in range(nkv):
                Kall = np.concatenate([kv.K[l, :P, g], kv.tK[l, anc, g]])
                Vall = np.concatenate([kv.V[l, :P, g], kv.tV[l, anc, g]])
                S = (Q[i, g * grp:(g + 1) * grp] @ Kall.T) * inv_sqrt_d      # [grp, keys]
                E = np.exp(S - S.max(axis=1, keepdims=True))
                O[i, g * grp:(g + 1) * grp] = (E / E.sum(axis=1, keepdims=True)) @ Vall
        O = R(O.reshape(n, nh * d))
        X = X + mm(O, lw["wo"])
        H2 = R(_rmsnorm_rows(X, lw["mlp_norm"].astype(np.float64), cfg.rms_eps))
        A = R(silu(mm(H2, lw["wg"])) * mm(H2, lw["wu"]))
        X = X + mm(A, lw["wd"])
    HF = R(_rmsnorm_rows(X, target.final_norm.astype(np.float64), cfg.rms_eps))
    logits = mm(HF, target.head)
    if return_hidden:
        return logits, HF
    return logits
