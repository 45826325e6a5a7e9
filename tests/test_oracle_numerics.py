"""Pins for oracle/numerics.py: bf16 rounding, RoPE, RMSNorm against library/closed forms."""
import numpy as np
import torch

from oracle.numerics import round_bf16, rope_rotate_half, rmsnorm, silu, bf16_bits_to_f64


def test_round_bf16_matches_torch_on_fp32_inputs():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(100_000) * np.exp(rng.uniform(-20, 20, 100_000))).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()   # torch: RNE
    assert np.array_equal(round_bf16(x.astype(np.float64)), ref)


def test_round_bf16_ties_and_no_double_rounding():
    one = 1.0
    assert round_bf16(np.array([one + 2**-8]))[0] == 1.0               # tie -> even (1.0)
    assert round_bf16(np.array([one + 3 * 2**-8]))[0] == one + 2**-6   # tie -> even (upper)
    # just above the tie: a float32 intermediate would drop 2^-40 and round to 1.0
    assert round_bf16(np.array([one + 2**-8 + 2**-40]))[0] == one + 2**-7
    assert round_bf16(np.array([-(one + 2**-8 + 2**-40)]))[0] == -(one + 2**-7)
    assert round_bf16(np.array([255.5 * 2**-7 * 2]))[0] == 4.0          # mantissa carry into exponent
    assert round_bf16(np.array([0.0]))[0] == 0.0
    assert round_bf16(np.array([4.2]))[0] == 4.1875


def test_bf16_bits_roundtrip():
    assert bf16_bits_to_f64(np.array([0x3F80, 0xC000, 0x4086], dtype=np.uint16)).tolist() == [1.0, -2.0, 4.1875]


def test_rope_against_complex_rotation():
    # rotate-half RoPE == multiplication of (v[j] + i v[j+d/2]) by exp(i pos theta^(-2j/d))
    rng = np.random.default_rng(1)
    d, theta = 128, 1e6
    v = rng.standard_normal(d)
    for pos in (0, 1, 17, 2047):
        z = (v[: d // 2] + 1j * v[d // 2:]) * np.exp(1j * pos * theta ** (-np.arange(d // 2) * 2.0 / d))
        out = rope_rotate_half(v, pos, theta, d)
        np.testing.assert_allclose(out, np.concatenate([z.real, z.imag]), rtol=0, atol=1e-12)
    np.testing.assert_array_equal(rope_rotate_half(v, 0, theta, d), v)


def test_rmsnorm_silu_match_torch():
    rng = np.random.default_rng(2)
    x, g = rng.standard_normal(256), rng.standard_normal(256)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (256,), torch.from_numpy(g), eps=1e-6).numpy()
    np.testing.assert_allclose(rmsnorm(x, g, 1e-6), ref, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(silu(x), torch.nn.functional.silu(torch.from_numpy(x)).numpy(), rtol=1e-14)
