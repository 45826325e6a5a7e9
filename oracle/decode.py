"""O.8-O.10 — AR reference, chunked prefill and the SubSpec loop.  Test infrastructure only.

O.8  Plain greedy autoregressive decoding of the target:
     x_{t+1} = argmax_v logits(x_1..x_t)[v], ties -> smallest id.  This is the
     result the method must reproduce exactly ("lossless").
O.9  Chunked prefill (§4.3): the prompt is
     processed in chunks of <= `chunk` tokens, each as a chain through the
     target, then committed.  The first generated token is the argmax at the
     last prompt position.
O.10 Capacity (reading R19): D_eff = min(D, floor((max_context - P - 1)/k));
     D_eff = 0 gives an AR step (tree = root only).  Generation stops after
     max_new tokens; the last step's tokens are truncated.
The SD step is Eq. 2's "D draft passes then one verification pass"
(PAPER.md:86): build_tree (draft weights) -> forward all nodes (target) ->
accept -> commit.
"""
import numpy as np

from synth.configs import ModelConfig
from .model import TargetWeights, KVCache, draft_layers, forward_nodes, forward_nodes_batched
from .tree import build_tree, Tree
from .verify import argmax_and_gap, accept, commit


class Session:
    """One generation session over a shared KV-cache."""

    def __init__(self, cfg: ModelConfig, seed: int, n_resident: int = 0, bits: int = 4,
                 group: int = 64, mode: str = "exact", max_nodes: int | None = None,
                 target: TargetWeights | None = None, dlayers=None, quant: str = "rtn"):
        """mode: "exact" (fp64), "bf16" (fp64 + the GPU's bf16 rounding points) or "bf16-fp32" (the
        rounding points with fp32 weights and node-batched fp32 matrix products: full-width shapes)."""
        self.cfg, self.mode = cfg, mode
        wdt = np.float32 if mode == "bf16-fp32" else np.float64
        self.target = target if target is not None else TargetWeights(cfg, seed, dtype=wdt)
        self.tlayers = self.target.layers
        # dlayers: a draft view built once and shared by several sessions (batched requests)
        self.dlayers = dlayers if dlayers is not None else draft_layers(self.target, n_resident, bits, group, method=quant)
        self.kv = KVCache(cfg, max_nodes or 512)
        self.n_forward_nodes = 0

    # -- forward helpers ------------------------------------------------
    def _forward(self, which, tokens, slots, positions, ancestors, **kw):
        layers = self.tlayers if which == "target" else self.dlayers
        self.n_forward_nodes += len(tokens)
        fwd = forward_nodes_batched if self.mode == "bf16-fp32" else forward_nodes
        return fwd(self.cfg, layers, self.target, self.kv, tokens, slots, positions, ancestors, self.mode, **kw)

    def forward_tree(self, which, tree: Tree, slots=None, **kw):
        """Teacher-forced forward of tree nodes (all nodes if slots is None); kw: return_hidden."""
        slots = list(range(len(tree))) if slots is None else list(slots)
        P = self.kv.P
        return self._forward(which, [tree.tokens[s] for s in slots], slots,
                             [P + tree.depths[s] for s in slots],
                             [tree.ancestors(s) for s in slots], **kw)

    # -- O.9 -------------------------------------------------------------
    def prefill(self, prompt, chunk=256):
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("empty prompt")
        if len(prompt) > self.cfg.max_context:
            raise ValueError("capacity")
        last = None
        for c0 in range(0, len(prompt), chunk):
            toks = prompt[c0:c0 + chunk]
            n = len(toks)
            tree = Tree(toks, [i - 1 for i in range(n)], list(range(n)), [0.0] * n)
            last = self.forward_tree("target", tree)[-1]
            commit(self.kv, list(range(1, n)))
        return int(np.argmax(last))

    # -- one SD step (O.4-O.7) -------------------------------------------
    def d_eff(self, D, k):
        return max(0, min(D, (self.cfg.max_context - self.kv.P - 1) // k))

    def draft_tree(self, root, D, k, T):
        if self.kv.P + 1 > self.cfg.max_context:
            raise ValueError("capacity")
        De = self.d_eff(D, k)
        return build_tree(root, De, k, T, lambda tree, fr: self.forward_tree("draft", tree, fr))

    def verify_tree(self, tree):
        logits = self.forward_tree("target", tree)
        am, gap = argmax_and_gap(logits)
        return am, gap, logits

    def accept_and_commit(self, tree, am):
        path, emitted = accept(tree, am)
        commit(self.kv, path)
        return path, emitted

    def step(self, root, D, k, T):
        tree = self.draft_tree(root, D, k, T)
        am, gap, _ = self.verify_tree(tree)
        path, emitted = self.accept_and_commit(tree, am)
        return tree, path, emitted


def ar_generate(cfg, prompt, max_new, seed=None, session=None, chunk=256, mode="exact"):
    """O.8: greedy AR decoding; returns max_new tokens (the first from prefill)."""
    s = session or Session(cfg, seed, mode=mode)
    out = [s.prefill(prompt, chunk)]
    while len(out) < max_new:
        root = out[-1]
        P = s.kv.P
        logits = s._forward("target", [root], [0], [P], [[0]])
        commit(s.kv, [])
        out.append(int(np.argmax(logits[0])))
    return out, s


def sd_generate(cfg, prompt, max_new, D, k, T, seed=None, session=None, n_resident=0,
                bits=4, chunk=256, mode="exact"):
    """SubSpec greedy generation; returns (tokens, per-step tau list, session)."""
    s = session or Session(cfg, seed, n_resident=n_resident, bits=bits, mode=mode,
                           max_nodes=max(1 + k * D, chunk))
    out = [s.prefill(prompt, chunk)]
    taus = []
    while len(out) < max_new:
        tree, path, emitted = s.step(out[-1], D, k, T)
        taus.append(len(emitted))
        out.extend(emitted)
    return out[:max_new], taus, s
