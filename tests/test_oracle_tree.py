"""Pins for oracle/tree.py (O.4) and oracle/verify.py (O.5-O.7):
SPEC/PAPER worked examples and brute-force enumeration on tiny vocabularies."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle.tree import tempered_softmax, tempered_log_softmax, build_tree, select_topk, Tree
from oracle.verify import accept, argmax_and_gap

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---- tempered softmax ------------------------------------------
def test_tempered_softmax_examples():
    np.testing.assert_allclose(tempered_softmax([0, 0, 0], 1.0), [1 / 3] * 3, rtol=1e-15)
    np.testing.assert_allclose(tempered_softmax([math.log(2), 0], 1.0), [2 / 3, 1 / 3], rtol=1e-15)
    assert tempered_softmax([1.0, 0.9, -3], 0).tolist() == [1, 0, 0]
    assert tempered_softmax([1.0, 1.0, -3], 0).tolist() == [1, 0, 0]        # tie -> smallest id
    p = tempered_softmax(np.log([0.45, 0.55]), 0.2)
    np.testing.assert_allclose(p, [0.45**5 / (0.45**5 + 0.55**5), 0.55**5 / (0.45**5 + 0.55**5)], rtol=1e-13)
    assert abs(p[0] - 0.2683) < 5e-5 and abs(p[1] - 0.7317) < 5e-5


def test_argmax_invariant_under_temperature_and_entropy_drops():
    rng = np.random.default_rng(0)
    for _ in range(50):
        l = rng.standard_normal(40) * 3
        base = tempered_softmax(l, 1.0)
        for T in (0.05, 0.2, 0.6, 2.0):
            p = tempered_softmax(l, T)
            assert np.argmax(p) == np.argmax(l)
            if T < 1:
                assert -(p * np.log(p + 1e-300)).sum() <= -(base * np.log(base)).sum() + 1e-12


# ---- Fig. 4 worked example -----------------------
def _fig4_logits_fn(g):
    X, Y, A, B = 0, 1, 2, 3
    tiny = 1e-30
    dist = {(): [g["root_probs"]["x"], g["root_probs"]["y"], tiny, tiny],
            (X,): [tiny, tiny, g["after_x"]["a"], g["after_x"]["b"]],
            (Y,): [tiny, tiny, g["after_y"]["a"], g["after_y"]["b"]]}

    def fn(tree, frontier):
        out = []
        for f in frontier:
            path = tuple(tree.tokens[a] for a in tree.ancestors(f)[1:])
            out.append(np.log(dist[path]))
        return np.array(out)
    return fn


@pytest.mark.parametrize("sharpen", [False, True])
def test_fig4_false_positive_path(sharpen):
    g = json.load(open(os.path.join(GOLD, "fig4_false_positive.json")))
    T = g["sharpened_T"] if sharpen else 1.0
    tree = build_tree(9, 2, g["k"], T, _fig4_logits_fn(g))
    depth2 = [i for i in range(len(tree)) if tree.depths[i] == 2]
    best = max(depth2, key=lambda i: tree.scores[i])
    through = "xy"[tree.tokens[tree.parents[best]]]
    want = g["sharpened_best"] if sharpen else g["unsharpened_best"]
    assert through == want["through"]
    assert abs(math.exp(tree.scores[best]) - want["score"]) < 5e-4
    other = [i for i in depth2 if tree.tokens[i] == 2 and i != best][0]
    assert abs(math.exp(tree.scores[other]) - want["other"]) < 5e-4


# ---- brute-force tree selection (SURVEY.md §8(c) O.4 pin) -------------------------
def _path_logits(path, V, seed):
    """A deterministic 'draft model': logits are a pure function of the token path."""
    h = hash((seed,) + tuple(path)) & 0xFFFFFFFF
    return np.random.default_rng(h).standard_normal(V) * 2.0


def _brute_force_tree(root, D, k, T, V, seed):
    """Independent replay: a node is identified by its token path; its score is recomputed
    from scratch by summing tempered log-probs along the path (no reuse of parent scores)."""
    def path_score(path):
        s = 0.0
        for j in range(1, len(path)):
            s += tempered_log_softmax(_path_logits(path[:j], V, seed), T)[path[j]]
        return s
    levels = [[(root,)]]
    for d in range(D):
        cands = []
        for pi, p in enumerate(levels[-1]):
            for v in range(V):
                cands.append((-path_score(p + (v,)), v, pi, p + (v,)))
        cands.sort(key=lambda c: (c[0], c[1], c[2]))
        chosen = cands[:k]
        chosen.sort(key=lambda c: (c[2], c[1]))              # canonical: parent asc, token asc
        levels.append([c[3] for c in chosen])
    return levels


@pytest.mark.parametrize("V,k,D,T", [(8, 1, 5, 0.2), (12, 2, 4, 0.2), (16, 3, 4, 1.0), (32, 4, 3, 0.2), (6, 4, 6, 0.6)])
def test_tree_matches_brute_force(V, k, D, T):
    for seed in range(3):
        def fn(tree, frontier):
            return np.array([_path_logits(tuple(tree.tokens[a] for a in tree.ancestors(f)), V, seed)
                             for f in frontier])
        tree = build_tree(1, D, k, T, fn)
        levels = _brute_force_tree(1, D, k, T, V, seed)
        assert len(tree) == 1 + k * D                                      # P:152 k x D + root
        for d in range(1, D + 1):
            got = [tuple(tree.tokens[a] for a in tree.ancestors(i)) for i in range(len(tree)) if tree.depths[i] == d]
            assert got == levels[d]
            assert [i for i in range(len(tree)) if tree.depths[i] == d] == list(range(1 + (d - 1) * k, 1 + d * k))
        for i in range(1, len(tree)):                                      # scores non-increasing along paths
            assert tree.scores[i] <= tree.scores[tree.parents[i]] + 1e-12


def test_k1_is_sharpened_greedy_chain():
    V = 20
    def fn(tree, frontier):
        return np.array([_path_logits(tuple(tree.tokens[a] for a in tree.ancestors(f)), V, 5) for f in frontier])
    tree = build_tree(3, 6, 1, 0.2, fn)
    path = [3]
    for _ in range(6):
        path.append(int(np.argmax(_path_logits(tuple(path), V, 5))))
    assert tree.tokens == path


def test_select_topk_tie_break():
    # equal scores: smaller token first, then smaller parent
    logp = np.zeros((2, 3))
    picked = select_topk([4, 7], [0.0, 0.0], logp, 3)
    assert picked == [(4, 0, 0.0), (4, 1, 0.0), (7, 0, 0.0)]


# ---- acceptance -------------------------------------------------
def test_accept_hand_examples():
    g = json.load(open(os.path.join(GOLD, "accept_examples.json")))
    for c in g["cases"]:
        t = Tree(c["tokens"], c["parents"], [0] * len(c["tokens"]), [0.0] * len(c["tokens"]))
        _, emitted = accept(t, c["argmax"])
        assert emitted == c["emitted"], c["name"]


def test_full_chain_gives_D_plus_1():
    D = 7
    toks = [5 + i for i in range(D + 1)]
    t = Tree(toks, [i - 1 for i in range(D + 1)], list(range(D + 1)), [0.0] * (D + 1))
    am = toks[1:] + [99]
    path, emitted = accept(t, am)
    assert len(emitted) == D + 1 and emitted[-1] == 99 and path == list(range(1, D + 1))


def test_accept_brute_force_longest_matching_path():
    rng = np.random.default_rng(11)
    for trial in range(200):
        V, k, D = 5, 3, 5
        n = 1 + k * D
        parents = [-1] + [int(rng.integers(max(0, 1 + (d - 2) * k) if d > 1 else 0, 1 + (d - 1) * k if d > 1 else 1))
                          for d in range(1, D + 1) for _ in range(k)]
        depths = [0] + [d for d in range(1, D + 1) for _ in range(k)]
        tokens = [0] + [int(x) for x in rng.integers(0, V, n - 1)]
        # siblings must carry distinct tokens (top-k picks distinct (parent, token) pairs)
        seen = set()
        for i in range(1, n):
            while (parents[i], tokens[i]) in seen:
                tokens[i] = (tokens[i] + 1) % V
            seen.add((parents[i], tokens[i]))
        t = Tree(tokens, parents, depths, [0.0] * n)
        am = [int(x) for x in rng.integers(0, V, n)]
        path, emitted = accept(t, am)
        # brute force: every node whose whole root path matches the target argmax chain
        best = [0]
        for i in range(n):
            anc = t.ancestors(i)
            if all(tokens[anc[j + 1]] == am[anc[j]] for j in range(len(anc) - 1)) and len(anc) > len(best):
                best = anc
        assert path == best[1:]
        assert emitted == [tokens[c] for c in best[1:]] + [am[best[-1]]]
        assert 1 <= len(emitted) <= D + 1


def test_argmax_and_gap():
    l = np.array([[1.0, 3.0, 3.0, 0.5], [2.0, -1.0, 0.0, 1.5]])
    am, gap = argmax_and_gap(l)
    assert am.tolist() == [1, 0] and gap.tolist() == [0.0, 0.5]
