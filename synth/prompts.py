"""MT-Bench-shaped synthetic prompts (SURVEY.md §8(d) "Prompts").

A fixed 24-token "template" prefix shared by all prompts, then a body of
U{40..232} tokens, so lengths lie in [64, 256] (mean ~160).  Token ids are
uniform over [0, V) from splitmix64 counters.  Input generator only.
"""
import numpy as np
from .weights import splitmix64, splitmix64_scalar, MASK64

TEMPLATE_LEN = 24
BODY_MIN, BODY_MAX = 40, 232


def _ids(key: int, n: int, vocab: int) -> np.ndarray:
    r = splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(key))
    return (r % np.uint64(vocab)).astype(np.int32)


def mtbench_prompt(seed: int, p: int, vocab: int, length: int | None = None) -> np.ndarray:
    tkey = splitmix64_scalar((seed ^ 0x7E4D_1A7E) & MASK64)
    pkey = splitmix64_scalar((seed * 0x100000001B3 + p + 1) & MASK64)
    if length is None:
        body = BODY_MIN + splitmix64_scalar(pkey ^ 0xB0D1) % (BODY_MAX - BODY_MIN + 1)
        length = TEMPLATE_LEN + body
    t = _ids(tkey, min(TEMPLATE_LEN, length), vocab)
    b = _ids(pkey, max(0, length - TEMPLATE_LEN), vocab)
    return np.concatenate([t, b]).astype(np.int32)


def uniform_prompt(seed: int, p: int, vocab: int, length: int) -> np.ndarray:
    key = splitmix64_scalar((seed * 0x9E37 + 17 * p + 3) & MASK64)
    return _ids(key, length, vocab)
