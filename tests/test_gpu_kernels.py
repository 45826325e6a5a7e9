"""GPU parity of the matrix kernels against the oracle.

K2 (draft dequant-GEMV): one-hot activations reproduce W_hat = code*s + z
bit-exactly (products by 1 and sums with 0 are exact in fp32); random activations agree with the
fp64 oracle within fp32 accumulation error.  NT = 1, 2, 4 token tiles (M = 1, 6, 13, 32).
K6 (target GEMM) and the bf16 GEMV on a resident layer: within fp32 accumulation error.
"""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import TINY, SMALL
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED


@pytest.fixture(scope="module", params=[TINY, SMALL], ids=["tiny", "small"])
def ctx(request, cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    cfg = request.param
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6)
    ss.load_synthetic(SEED, n_resident=1)     # layer 0 resident (bf16), others substituted
    ss.build_substitutes(4, 64)
    yield cfg, ss
    ss.close()


def _what(ss, layer, g):
    return dequantize(*quantize(bf16_bits_to_f64(ss.debug_read_group(layer, g))))


def test_k2_one_hot_exact(ctx):
    cfg, ss = ctx
    for g in range(4):
        N, K = ss.group_shape(g)
        what = _what(ss, 1, g)
        for k0 in range(0, K, 32):
            M = min(32, K - k0)
            x = np.zeros((M, K), np.uint16)
            x[np.arange(M), k0 + np.arange(M)] = 0x3F80
            y = ss.debug_matmul(0, 1, g, x).astype(np.float64)
            assert np.array_equal(y, what[:, k0:k0 + M].T), (g, k0)


@pytest.mark.parametrize("M", [1, 6, 13, 32])
def test_k2_random_activations(ctx, M):
    cfg, ss = ctx
    rng = np.random.default_rng(M)
    for g in range(4):
        N, K = ss.group_shape(g)
        what = _what(ss, 1, g)
        xb = W.f32_to_bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
        y = ss.debug_matmul(0, 1, g, xb)
        ref = bf16_bits_to_f64(xb) @ what.T
        # fp32 accumulation over K terms of |x w| ~ O(1): bound by K * 2^-22 * sum|x||w|
        bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(what).T) + 1e-6
        assert np.all(np.abs(y - ref) <= bound), (g, M, float(np.max(np.abs(y - ref))))


@pytest.mark.parametrize("which,M", [(0, 1), (0, 6), (0, 32), (1, 1), (1, 100), (1, 256)])
def test_bf16_gemv_and_gemm_resident(ctx, which, M):
    cfg, ss = ctx
    rng = np.random.default_rng(7 * M + which)
    for g in range(4):
        N, K = ss.group_shape(g)
        w = bf16_bits_to_f64(ss.debug_read_group(0, g))
        xb = W.f32_to_bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
        y = ss.debug_matmul(which, 0, g, xb)
        ref = bf16_bits_to_f64(xb) @ w.T
        bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(w).T) + 1e-6
        assert np.all(np.abs(y - ref) <= bound), (which, g, M)


def test_k2_deterministic(ctx):
    cfg, ss = ctx
    rng = np.random.default_rng(3)
    N, K = ss.group_shape(2)
    xb = W.f32_to_bf16_bits(rng.standard_normal((6, K)).astype(np.float32))
    a = ss.debug_matmul(0, 1, 2, xb)
    b = ss.debug_matmul(0, 1, 2, xb)
    assert np.array_equal(a, b)
