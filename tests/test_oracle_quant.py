"""Pins for oracle/quant.py (O.2): SPEC.md quantize/dequantize examples, bounds, invariants."""
import json
import os

import numpy as np
import pytest

from oracle.quant import quantize, dequantize, substitute_matrix
from oracle.numerics import round_bf16

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_ramp_example():
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


def test_error_bound():
    # SPEC.md:134 |x_hat - x| <= s/2, up to the fp32 rounding of (x - z)/s in the code decision
    # (reading R5) and the clamp when bf16 rounds s below (M - m)/15 (then the top code is 15)
    x = _bf16_random((64, 512), 0.05, 3)
    codes, s, z = quantize(x)
    xh = dequantize(codes, s, z)
    S = np.repeat(s, 64, axis=1)
    top = np.repeat(z + 15 * s, 64, axis=1)
    assert np.all((np.abs(xh - x) <= S / 2 * (1 + 2**-20)) | ((codes == 15) & (x >= top)))
    assert codes.max() <= 15 and codes.min() == 0


def test_dequant_is_exact_affine():
    # W_hat == code*s + z exactly: check against exact rational arithmetic
    from fractions import Fraction
    x = _bf16_random((4, 128), 0.02, 4)
    codes, s, z = quantize(x)
    xh = dequantize(codes, s, z)
    for n in range(4):
        for k in range(0, 128, 7):
            g = k // 64
            assert Fraction(xh[n, k]) == codes[n, k] * Fraction(s[n, g]) + Fraction(z[n, g])


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


# ---- 2-bit substitutes: the same rule with 3 levels ----------
def test_ramp_2bit_closed_form():
    # ramp 0..63: s = (63 - 0)/3 = 21 (exact in bf16), z = 0; no x/21 lands on a .5 tie, so the code
    # is plain integer rounding (2x + 21) // 42, and every error is |21 c - x| <= 10 < s/2
    x = np.arange(64, dtype=np.float64)[None, :]
    codes, s, z = quantize(x, 2, 64)
    assert s[0, 0] == 21.0 and z[0, 0] == 0.0
    want = (2 * np.arange(64) + 21) // 42
    assert codes[0].tolist() == want.tolist()
    assert codes[0, 10] == 0 and codes[0, 11] == 1 and codes[0, 31] == 1 and codes[0, 32] == 2 and codes[0, 63] == 3
    xh = dequantize(codes, s, z)
    assert np.array_equal(xh[0], 21.0 * want)
    assert np.abs(xh - x).max() == 10.0


def test_error_bound_2bit():
    x = _bf16_random((64, 512), 0.05, 13)
    codes, s, z = quantize(x, 2)
    xh = dequantize(codes, s, z)
    S = np.repeat(s, 64, axis=1)
    top = np.repeat(z + 3 * s, 64, axis=1)
    assert np.all((np.abs(xh - x) <= S / 2 * (1 + 2**-20)) | ((codes == 3) & (x >= top)))
    assert codes.max() == 3 and codes.min() == 0


def test_ramp_3bit_closed_form():
    # NEXT-3 3-bit: ramp 0..63, s = 63/7 = 9 exactly, z = 0; x/9 never lands on a .5
    # tie for integer x, so code = (2x + 9) // 18 and the largest error is 4 (x = 4: code 0)
    x = np.arange(64, dtype=np.float64)[None, :]
    codes, s, z = quantize(x, 3, 64)
    assert s[0, 0] == 9.0 and z[0, 0] == 0.0
    want = (2 * np.arange(64) + 9) // 18
    assert codes[0].tolist() == want.tolist() and codes.max() == 7
    xh = dequantize(codes, s, z)
    assert np.array_equal(xh[0], 9.0 * want) and np.abs(xh - x).max() == 4.0


def test_error_bound_3bit():
    x = _bf16_random((64, 512), 0.05, 17)
    codes, s, z = quantize(x, 3)
    xh = dequantize(codes, s, z)
    S = np.repeat(s, 64, axis=1)
    top = np.repeat(z + 7 * s, 64, axis=1)
    assert np.all((np.abs(xh - x) <= S / 2 * (1 + 2**-20)) | ((codes == 7) & (x >= top)))
    assert codes.max() == 7 and codes.min() == 0


def test_fewer_bits_more_error():
    # SPEC.md "monotone fidelity": mean abs error non-increasing in bits (2 -> 4 roughly / 5 here:
    # the step shrinks from range/3 to range/15)
    x = _bf16_random((32, 256), 0.05, 15)
    e2 = np.abs(substitute_matrix(x, 2) - x).mean()
    e3 = np.abs(substitute_matrix(x, 3) - x).mean()
    e4 = np.abs(substitute_matrix(x, 4) - x).mean()
    assert e2 > 3 * e4 and e2 > 1.5 * e3 > 1.5 * 1.5 * e4


# ---- HQQ refinement (NEXT-3, reading R28) ----------------------------------------------------
from oracle.quant import hqq_shrink, hqq_step, hqq_refine_zero, HQQ_P


def test_hqq_shrink_p1_is_soft_threshold_prox():
    # p = 1: W_e must be the proximal point argmin_w 1/2 (w - e)^2 + |w| / beta, found by brute force
    beta = 10.0
    grid = np.linspace(-1.0, 1.0, 400001)
    for e in [-0.7, -0.1, -0.05, 0.0, 0.03, 0.1, 0.2, 0.55]:
        obj = 0.5 * (grid - e) ** 2 + np.abs(grid) / beta
        w_bf = grid[np.argmin(obj)]
        assert abs(hqq_shrink(np.array([e]), beta, p=1.0)[0] - w_bf) <= 1e-5


def test_hqq_shrink_p07_threshold_and_shrinkage():
    # |e| - |e|^(p-1)/beta <= 0  <=>  |e| <= beta^(-1/(2-p)): zero inside, sign-preserving shrink outside
    beta = 10.0
    thr = beta ** (-1.0 / (2.0 - HQQ_P))
    e = np.array([-thr * 1.001, -thr * 0.999, thr * 0.999, thr * 1.001, 3 * thr, -5 * thr])
    we = hqq_shrink(e, beta)
    assert we[1] == 0 and we[2] == 0
    assert we[0] < 0 < we[3] and np.all(np.abs(we) <= np.abs(e))
    assert np.all(np.sign(we[[0, 3, 4, 5]]) == np.sign(e[[0, 3, 4, 5]]))


def test_hqq_zero_update_minimises_the_quadratic():
    # z_next = argmin_z sum (x - W_e - code*s - z)^2 for the step's own code and W_e (scipy minimiser)
    from scipy.optimize import minimize_scalar
    x = _bf16_random((3, 64), 0.02, 11)
    codes, s, z = quantize(x)
    for g in range(3):
        _, zn, code, we = hqq_step(x[g:g + 1], s[g:g + 1, 0], z[g:g + 1, 0], 10.0)
        f = lambda t: float(np.sum((x[g] - we[0] - code[0] * s[g, 0] - t) ** 2))
        r = minimize_scalar(f, bracket=(z[g, 0] - 0.01, z[g, 0] + 0.01), tol=1e-14)
        assert abs(zn[0] - r.x) <= 1e-9 * max(1.0, abs(r.x))
        # err is the mean absolute reconstruction error of the CURRENT zero, via the dequantiser
        err, _, _, _ = hqq_step(x[g:g + 1], s[g:g + 1, 0], z[g:g + 1, 0], 10.0)
        assert np.isclose(err[0], np.mean(np.abs(dequantize(codes[g:g + 1], s[g:g + 1], z[g:g + 1]) - x[g])),
                          rtol=1e-12)


def test_hqq_on_grid_group_is_fixed_point():
    # x exactly on z + c*s with c spanning 0..15: RTN is exact, HQQ keeps z and the codes
    rng = np.random.default_rng(5)
    c = rng.integers(0, 16, size=(4, 64))
    c[:, 0], c[:, 1] = 0, 15
    s, z = 0.00390625, -0.03125
    x = c * s + z
    for bits in (4,):
        cr, sr, zr = quantize(x, bits, 64, "rtn")
        ch, sh, zh = quantize(x, bits, 64, "hqq")
        assert np.array_equal(cr, ch) and np.array_equal(zr, zh) and np.array_equal(sr, sh)
        assert np.array_equal(dequantize(ch, sh, zh), x)


def test_hqq_constant_group_and_iters_limits():
    x = np.full((2, 64), 0.25)
    assert np.array_equal(quantize(x, 4, 64, "hqq")[2], quantize(x, 4, 64, "rtn")[2])
    y = _bf16_random((8, 256), 0.03, 12)
    # one iteration only evaluates the RTN zero: identical to RTN
    for a, b in zip(quantize(y, 4, 64, "hqq", hqq_iters=1), quantize(y, 4, 64, "rtn")):
        assert np.array_equal(a, b)


def test_hqq_error_trace_and_improvement():
    # the kept zero has the lowest mean |x - W_r| of the visited iterates (<= RTN's), and over many
    # Gaussian groups HQQ lowers the reconstruction error vs RTN in l1 and in HQQ's own l_0.7 (the
    # method's published purpose)
    x = _bf16_random((256, 1024), 0.02, 13)
    codes, s, z = quantize(x)
    xg = x.reshape(256, 16, 64)
    zb, errs = hqq_refine_zero(xg, s, z, trace=True)
    E = np.stack(errs)
    first = E[0]
    assert np.allclose(first, np.mean(np.abs(dequantize(codes, s, z) - x).reshape(256, 16, 64), axis=2), rtol=1e-12)
    assert len(errs) > 2
    best = np.min(E, axis=0)
    assert np.all(best <= first)
    assert np.mean(best < first) > 0.5                        # most groups improve
    ch, sh, zh = quantize(x, 4, 64, "hqq")
    assert np.array_equal(sh, s)                               # HQQ keeps the scale
    r, h = dequantize(codes, s, z) - x, dequantize(ch, sh, zh) - x
    assert np.mean(np.abs(h)) < 0.98 * np.mean(np.abs(r))
    assert np.mean(np.abs(h) ** HQQ_P) < 0.99 * np.mean(np.abs(r) ** HQQ_P)
    assert codes.max() <= 15 and ch.max() <= 15
