"""O.5-O.7 — verification, greedy acceptance, KV commit.  Test infrastructure only.

O.5  argmax per node of the target logits over the whole tree (ties -> the
     smallest id), and the top-1/top-2 gap used for near-tie flags.
O.6  Greedy branch of SPEC.md:391 ("draw token X from the target distribution
     (temperature 0 = argmax); if X equals one of the node's children, accept
     that child and descend; otherwise emit X as the final token and stop").
     tau_step = |path| + 1 in [1, D+1] (Eq. 2).
O.7  The committed KV at P + j becomes the target KV of (root, path...)[j];
     P <- P + |path| + 1, root <- the bonus token (reading R15).
"""
import numpy as np


def argmax_and_gap(logits):
    logits = np.asarray(logits, dtype=np.float64)
    am = np.argmax(logits, axis=1)                 # first occurrence = smallest id
    top = np.take_along_axis(logits, am[:, None], axis=1)[:, 0]
    masked = logits.copy()
    masked[np.arange(len(am)), am] = -np.inf
    second = masked.max(axis=1)
    return am.astype(np.int64), top - second


def accept(tree, argmax):
    """Returns (path slots, emitted tokens)."""
    path, cur = [], 0
    while True:
        y = int(argmax[cur])
        nxt = [c for c in tree.children(cur) if tree.tokens[c] == y]
        if not nxt:
            break
        cur = nxt[0]                    # children carry distinct tokens
        path.append(cur)
    emitted = [tree.tokens[c] for c in path] + [int(argmax[cur])]
    return path, emitted


def commit(kv, path):
    P = kv.P
    rows = [0] + list(path)
    for j, s in enumerate(rows):
        kv.K[:, P + j] = kv.tK[:, s]
        kv.V[:, P + j] = kv.tV[:, s]
    kv.P = P + len(rows)
