"""Elementary numerics for the oracle (float64).  Test infrastructure only.

bf16 rounding points are the build's named reading of the paper's silent
precision (SURVEY.md §8(c) O.3 "bf16-emulation"; DESIGN.md "Readings" R3).
"""
import numpy as np


def bf16_bits_to_f64(b):
    b = np.asarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def round_bf16(x):
    """Round float64 values directly to the nearest bf16 (ties to even), returned as float64.

    Rounds once from the float64 value (no float32 intermediate, which would
    double-round).  Bits below bf16's 7 stored mantissa bits are the low 45
    bits of the float64 encoding.  Normal range only (|x| >= 2^-126) or zero;
    the forward never produces bf16 subnormals (checked)."""
    x = np.asarray(x, dtype=np.float64)
    u = x.view(np.uint64)
    lsb = (u >> np.uint64(45)) & np.uint64(1)
    with np.errstate(over="ignore"):
        r = (u + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)
    out = r.view(np.float64)
    a = np.abs(out)
    if np.any((a != 0) & (a < 2.0 ** -126)) or not np.all(np.isfinite(out)):
        raise ValueError("round_bf16: subnormal or non-finite value")
    return out


def to_bf16_bits(x):
    """float64 values that are already bf16-representable -> uint16 bit patterns."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    assert np.array_equal(f.astype(np.float64), np.asarray(x, dtype=np.float64)), "not bf16-exact"
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def rmsnorm(x, g, eps):
    """x * rsqrt(mean(x^2) + eps) * g   (SPEC.md:85 pre-RMS-norm)."""
    return x / np.sqrt(np.mean(x * x) + eps) * g


def silu(x):
    return x / (1.0 + np.exp(-x))


def rope_rotate_half(v, pos, theta, head_dim):
    """Rotate-half RoPE of one head vector at integer position `pos`:
    theta_j = theta^(-2j/d), angle = pos * theta_j,
    v'[j] = v[j] cos - v[j+d/2] sin ; v'[j+d/2] = v[j+d/2] cos + v[j] sin."""
    half = head_dim // 2
    j = np.arange(half, dtype=np.float64)
    ang = pos * theta ** (-2.0 * j / head_dim)
    c, s = np.cos(ang), np.sin(ang)
    a, b = v[:half], v[half:]
    return np.concatenate([a * c - b * s, b * c + a * s])
