"""O.4 — context-aware dynamic draft tree with sharpening.
Test infrastructure only.

PAPER.md:148-152 §4.2: "In each of these D forward passes, all leaf nodes are
input to the draft model, each yielding probability distributions for the
potential next tokens.  The score for each potential next token is the
cumulative product of its conditional generation probability (from the draft
model) and its parent path score.  The top-k tokens with the highest scores
are selected to form the new k leaf nodes ... k x D draft tokens ... (not
including the root token)."
PAPER.md:157-159: sharpening applies temperature 0.2 to the draft
distribution "before calculating cumulative probabilities".

Log domain: lp_i = (l_i - max l_i)/T - log sum_v exp((l_i[v] - max l_i)/T);
candidate score = score(parent) + lp_parent[v].
Selection: global top-k over all (frontier node, token) by (score desc, token
asc, parent slot asc).  Storage: each depth in canonical order
(parent slot asc, token asc) (reading R12); depth-major slots: root = 0,
depth-d nodes at 1+(d-1)k .. dk.
"""
from dataclasses import dataclass, field
import numpy as np


def tempered_log_softmax(l, T):
    l = np.asarray(l, dtype=np.float64)
    t = (l - l.max()) / T
    return t - np.log(np.sum(np.exp(t)))


def tempered_softmax(l, T):
    """softmax(l/T); T = 0 -> one-hot of the first argmax."""
    l = np.asarray(l, dtype=np.float64)
    if T == 0:
        out = np.zeros_like(l)
        out[int(np.argmax(l))] = 1.0
        return out
    return np.exp(tempered_log_softmax(l, T))


@dataclass
class Tree:
    tokens: list = field(default_factory=list)
    parents: list = field(default_factory=list)
    depths: list = field(default_factory=list)
    scores: list = field(default_factory=list)

    def __len__(self):
        return len(self.tokens)

    def ancestors(self, i):
        path = []
        while i >= 0:
            path.append(i)
            i = self.parents[i]
        return path[::-1]

    def children(self, i):
        return [c for c in range(len(self.tokens)) if self.parents[c] == i]


def select_topk(frontier, frontier_scores, logp, k):
    """Global top-k over candidates (frontier[i], v) with score frontier_scores[i] + logp[i, v].
    Returns [(parent_slot, token, score)] in canonical order (parent asc, token asc)."""
    F, V = logp.shape
    sc = (np.asarray(frontier_scores, dtype=np.float64)[:, None] + logp).reshape(-1)
    tok = np.tile(np.arange(V), F)
    par = np.repeat(np.asarray(frontier), V)
    order = np.lexsort((par, tok, -sc))          # primary: -score, then token, then parent
    chosen = order[:k]
    picked = sorted((int(par[c]), int(tok[c]), float(sc[c])) for c in chosen)
    return picked


def build_tree(root_token, D, k, T, logits_fn):
    """Grow the draft tree.  logits_fn(tree, frontier_slots) -> logits [len(frontier), V]
    (one draft forward pass of the frontier, which may write KV for those slots)."""
    tree = Tree([int(root_token)], [-1], [0], [0.0])
    frontier = [0]
    for d in range(D):
        logits = np.asarray(logits_fn(tree, frontier), dtype=np.float64)
        logp = np.stack([tempered_log_softmax(logits[i], T) for i in range(len(frontier))])
        picked = select_topk(frontier, [tree.scores[f] for f in frontier], logp, k)
        frontier = []
        for par, tok, s in picked:
            frontier.append(len(tree.tokens))
            tree.tokens.append(tok)
            tree.parents.append(par)
            tree.depths.append(d + 1)
            tree.scores.append(s)
    return tree
