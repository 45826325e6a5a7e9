"""Pins for oracle/quant.py (O.2): SPEC.md quantize/dequantize examples, bounds, invariants."""
import json
import os

import numpy as np
import pytest

from oracle.quant import quantize, dequantize, substitute_matrix
from oracle.numerics import round_bf16

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_ramp_example_bf16_scale():
    g = json.load(open(os.path.join(GOLD, "quant_ramp_4bit.json")))
    x = np.arange(64, dtype=np.float64)[None, :]
    codes, s, z = quantize(x, 4, 64)
    assert s[0, 0] == g["scale"] and z[0, 0] == g["zero"]
    assert codes[0, 63] == g["code_of_63"]
    assert codes[0, :8].tolist() == g["first_codes"]
    xh = dequantize(codes, s, z)
    assert xh[0, 63] == g["dequant_of_63"]
    err = np.abs(xh - x)[0]
    assert err.max() == g["max_abs_error"] and int(np.argmax(err)) == g["argmax_error_x"]
    assert err.max() <= s[0, 0] / 2


def test_constant_group_exact():
    x = np.full((1, 64), 5.0)
    codes, s, z = quantize(x)
    assert np.all(codes == 0) and s[0, 0] == 1.0 and z[0, 0] == 5.0
    assert np.array_equal(dequantize(codes, s, z), x)


def test_zero_tensor():
    x = np.zeros((4, 128))
    assert np.array_equal(substitute_matrix(x), x)


def _bf16_random(shape, scale, seed):
    rng = np.random.default_rng(seed)
    return round_bf16(rng.standard_normal(shape) * scale)


def test_relaxed_error_bound():
    # reading R5: |W_hat - x| <= s/2 (1 + 2^-20) + 2^-8 |W_hat|  (bf16 unit roundoff u = 2^-8 for the rounding of W_hat)
    x = _bf16_random((64, 512), 0.05, 3)
    codes, s, z = quantize(x)
    xh = dequantize(codes, s, z)
    S = np.repeat(s, 64, axis=1)
    assert np.all(np.abs(xh - x) <= S / 2 * (1 + 2**-20) + 2**-8 * np.abs(xh))
    assert codes.max() <= 15 and codes.min() == 0


def test_dequant_is_single_rounding_of_exact_affine():
    x = _bf16_random((16, 256), 0.02, 4)
    codes, s, z = quantize(x)
    xh = dequantize(codes, s, z)
    exact = codes.reshape(16, 4, 64) * s[..., None] + z[..., None]
    # W_hat is the bf16 neighbour of the exact affine value (never more than half a bf16 ulp away)
    ulp = 2.0 ** (np.floor(np.log2(np.abs(xh.reshape(16, 4, 64)) + 1e-300)) - 7)
    assert np.all(np.abs(xh.reshape(16, 4, 64) - exact) <= ulp / 2 + 1e-300)


def test_more_bits_less_error():
    x = _bf16_random((32, 256), 0.05, 5)
    e4 = np.abs(substitute_matrix(x, 4) - x).mean()
    e8 = np.abs(substitute_matrix(x, 8) - x).mean()
    assert e8 < e4 / 8


def test_min_maps_to_code0_and_zero_point():
    x = _bf16_random((8, 128), 0.1, 6)
    codes, s, z = quantize(x)
    xg = x.reshape(8, 2, 64)
    assert np.array_equal(z, xg.min(axis=2))
    for n in range(8):
        for g in range(2):
            assert codes[n, 64 * g + int(np.argmin(xg[n, g]))] == 0


def test_nonfinite_rejected():
    x = np.zeros((1, 64)); x[0, 3] = np.nan
    with pytest.raises(ValueError):
        quantize(x)
