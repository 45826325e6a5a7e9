"""Shared helpers for the GPU parity tests (no method arithmetic: comparisons only)."""
import numpy as np

TOL_BF16 = 2e-2     # BASELINE.json north_star: max-abs 2e-2 relative to logit scale (bf16)


def scale_of(ref):
    return max(1.0, float(np.max(np.abs(ref))))


def assert_close_scaled(got, ref, tol=TOL_BF16, what=""):
    s = scale_of(ref)
    err = float(np.max(np.abs(np.asarray(got, np.float64) - np.asarray(ref, np.float64))))
    assert err <= tol * s, f"{what}: max |diff| {err:.3e} > {tol} x scale {s:.3f}"
    return err / s


def rel_rms(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.sqrt(np.mean((got - ref) ** 2)) / max(1e-30, np.sqrt(np.mean(ref ** 2))))


def assert_matches_oracle_ar(cfg, prompt, got, seed, tol=TOL_BF16, mode="bf16"):
    """GPU output vs the oracle's greedy AR output (O.8): identical up to flagged near-ties.  At the
    first difference the oracle is teacher-forced on the GPU's tokens; the GPU token must be within
    2 x tol x scale of the oracle's top-1 logit there (a flag), and the comparison continues from
    the GPU's tokens.  Returns the number of flags."""
    from oracle.decode import Session
    from oracle.tree import Tree
    from oracle.verify import commit
    got = [int(t) for t in got]
    s = Session(cfg, seed, mode=mode, max_nodes=max(512, len(prompt) + len(got) + 1))
    nxt = s.prefill(prompt)
    flags = 0
    for i, g in enumerate(got):
        if g != nxt:
            # recompute the logits at this position (teacher-forced) to judge the near-tie
            o = Session(cfg, seed, mode=mode, max_nodes=max(512, len(prompt) + len(got) + 1), target=s.target)
            seq = [int(t) for t in prompt] + got[:i]
            lg = o.forward_tree("target", Tree(seq, [j - 1 for j in range(len(seq))], list(range(len(seq))),
                                               [0.0] * len(seq)))[-1]
            assert lg.max() - lg[g] <= 2 * tol * scale_of(lg), f"unflagged divergence at {i}: {g} vs {nxt}"
            flags += 1
        if i + 1 == len(got):
            break
        P = s.kv.P
        lg = s._forward("target", [g], [0], [P], [[0]])[0]
        commit(s.kv, [])
        nxt = int(np.argmax(lg))
    return flags
