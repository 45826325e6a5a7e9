"""O.2 — substitute-layer quantizer.  Test infrastructure only.

Paper: substitutes are data-free low-bit quantized copies of the offloaded
layers (§4.1), "quantized to 4 bits with a group size 64
using HQQ" (§5.1).  HQQ's half-quadratic refinement is not
described in the paper; SPEC.md:125 fixes its initialisation, asymmetric
min/max round-to-nearest (reading R1 in DESIGN.md).  Groups are 64
consecutive input (K) elements of one output row (R2); scale and zero are
bf16 (R3); constant groups use s = 1; rounding is half-to-even
(SPEC.md:125).

Per (row n, group g), with x the bf16 values (exact in fp32):
    m = min(x), M = max(x)
    s = 1.0                                   if M == m
      = RNE_bf16( fp32( fp32(M - m) / 15 ) )  otherwise
    z = m
    code = clamp( rint_half_even( fp32( fp32(x - z) / s ) ), 0, 2^bits - 1 )
    W_hat = code * s + z                      (exact; reading R3: the affine dequantisation is
                                               applied exactly, as fused low-bit GEMM kernels do
                                               when they scale per group in fp32)
"""
import numpy as np



def _f32_to_bf16_f32(x32):
    """Round fp32 -> bf16 (RNE), returned as fp32 values."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    bias = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return (((u + bias) >> np.uint32(16)) << np.uint32(16)).view(np.float32)


def quantize(w, bits=4, group=64):
    """w: float array [N, K] of bf16-representable values.
    Returns (codes uint8 [N, K], s float64 [N, K/group], z float64 [N, K/group]),
    s and z being bf16-representable."""
    w = np.asarray(w, dtype=np.float64)
    N, K = w.shape
    if K % group:
        raise ValueError("K must be a multiple of the group size")
    if not np.all(np.isfinite(w)):
        raise ValueError("non-finite input")            # SPEC.md:128 invalid-input
    qmax = (1 << bits) - 1
    x32 = w.astype(np.float32).reshape(N, K // group, group)
    assert np.array_equal(x32.astype(np.float64), w.reshape(N, K // group, group)), "input not fp32-exact"
    m = x32.min(axis=2)
    M = x32.max(axis=2)
    rng32 = (M - m).astype(np.float32)                          # fp32(M - m)
    s32 = _f32_to_bf16_f32((rng32 / np.float32(qmax)).astype(np.float32))
    s32 = np.where(M == m, np.float32(1.0), s32).astype(np.float32)
    z32 = m
    t = ((x32 - z32[..., None]).astype(np.float32) / s32[..., None]).astype(np.float32)
    codes = np.clip(np.rint(t), 0, qmax).astype(np.uint8)       # np.rint: half-to-even
    return codes.reshape(N, K), s32.astype(np.float64), z32.astype(np.float64)


def dequantize(codes, s, z, group=64):
    """W_hat[n,k] = code*s + z, exact in float64 (a <=8-bit x 8-bit significand product plus an
    8-bit-significand addend of nearby magnitude)."""
    N, K = codes.shape
    c = codes.astype(np.float64).reshape(N, K // group, group)
    return (c * s[..., None] + z[..., None]).reshape(N, K)


def substitute_matrix(w, bits=4, group=64):
    codes, s, z = quantize(w, bits, group)
    return dequantize(codes, s, z, group)
