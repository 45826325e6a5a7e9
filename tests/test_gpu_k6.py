"""K6 (the target's verify GEMM; "verifies all drafted tokens in a
single forward pass") at the Qwen2.5-7B widths, on the tcgen05 kernel (gemm_tc_kernel).

* correctness: sampled output rows of every matrix group against fp64 products of the same bf16
  operands, within the fp32-accumulation bound, at M = 1 (an AR step), 128, 289 (a D = 48, k = 6 tree)
  and 300 (a ragged last token tile) — this spans cluster split-K S = 1 (gate_up), 4 (qkv, o) and 8
  (down) and several token tiles;
* batch invariance: a token's output row is bitwise the same whether it is computed
  alone (M = 1), in a 128-token launch or in a 289-token launch — the property that makes the GPU's
  SubSpec output equal its AR output bitwise;
* the legacy mma.sync kernel and the half-chunk tcgen05 variant (debug knob 2) agree within the same bound.
"""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import QWEN7B, GIB
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED


@pytest.fixture(scope="module")
def ctx(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    cfg = QWEN7B.with_(name="qwen2.5-7b-1l", n_layers=1)
    ss = SubSpec(cfg, 3 * GIB, max_depth=48, max_top_k=6)
    ss.load_synthetic(SEED, n_resident=1)
    ss.build_substitutes(4, 64)   # no offloaded layer: only moves the context to READY
    yield cfg, ss
    ss.close()


def _bound(xb, w):
    ax = np.abs(bf16_bits_to_f64(xb))
    return w.shape[1] * 2.0**-22 * (ax @ np.abs(w).T) + 1e-6


@pytest.mark.parametrize("g", [0, 1, 2, 3], ids=["qkv", "o", "gate_up", "down"])
def test_k6_full_width_and_batch_invariance(ctx, g):
    cfg, ss = ctx
    N, K = ss.group_shape(g)
    rng = np.random.default_rng(100 + g)
    w_all = ss.debug_read_group(0, g)
    rows = np.sort(rng.choice(N, size=384, replace=False))
    rows = np.unique(np.concatenate([rows, [0, 127, 128, N - 1]]))
    w = bf16_bits_to_f64(w_all[rows])
    x = W.f32_to_bf16_bits(rng.standard_normal((300, K)).astype(np.float32))
    ys = {}
    for M in (1, 128, 289, 300):
        y = ss.debug_matmul(1, 0, g, x[:M])
        assert y.shape == (M, N)
        ref = bf16_bits_to_f64(x[:M]) @ w.T
        err = np.abs(y[:, rows] - ref)
        assert np.all(err <= _bound(x[:M], w)), (g, M, float(err.max()))
        ys[M] = y
    # batch invariance: identical rows whatever the launch's M
    assert np.array_equal(ys[1][0], ys[289][0])
    assert np.array_equal(ys[128], ys[289][:128])
    assert np.array_equal(ys[289], ys[300][:289])
    for m in (150, 288):
        assert np.array_equal(ss.debug_matmul(1, 0, g, x[m:m + 1])[0], ys[289][m]), m


@pytest.mark.parametrize("variant", [1, 2], ids=["legacy", "half-chunk"])
def test_k6_variants_agree(ctx, variant):
    cfg, ss = ctx
    g = 3
    N, K = ss.group_shape(g)
    rng = np.random.default_rng(9)
    x = W.f32_to_bf16_bits(rng.standard_normal((289, K)).astype(np.float32))
    a = ss.debug_matmul(1, 0, g, x)
    ss.debug_set_knob(2, variant)
    try:
        b = ss.debug_matmul(1, 0, g, x)
    finally:
        ss.debug_set_knob(2, 0)
    rows = np.arange(0, N, 7)
    w = bf16_bits_to_f64(ss.debug_read_group(0, g)[rows])
    assert np.all(np.abs(a[:, rows] - b[:, rows]) <= 2 * _bound(x, w))


def test_k6_deterministic(ctx):
    cfg, ss = ctx
    rng = np.random.default_rng(4)
    N, K = ss.group_shape(1)
    x = W.f32_to_bf16_bits(rng.standard_normal((289, K)).astype(np.float32))
    assert np.array_equal(ss.debug_matmul(1, 0, 1, x), ss.debug_matmul(1, 0, 1, x))
