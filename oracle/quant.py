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

method="hqq" (reading R28 in DESIGN.md): the paper names HQQ (PAPER.md:136
"HQQ", :278 "quantized to 4 bits with a group size 64 using HQQ") without describing it.  HQQ
(Badri & Shaji, 2023, "Half-Quadratic Quantization of Large Machine Learning Models") keeps the
min/max scale and refines the zero point by half-quadratic splitting of
    min_z  || x - W_r(z) ||_p^p ,   p = 0.7,   W_r(z) = code(z)*s + z,  code(z) = clamp(rint((x - z)/s)),
alternating, with beta growing by kappa each iteration:
    e    = x - W_r(z)
    W_e  = sign(e) * max(|e| - |e|^(p-1) / beta, 0)           (generalised soft-thresholding)
    z   <- mean(x - W_e - code*s)                             (closed-form least-squares zero)
for at most 20 iterations from the RTN zero, beta0 = 10, kappa = 1.01, stopping when the group's
mean |x - W_r| stops decreasing; the zero with the lowest error is kept (per 64-group: the groups
are independent problems).  The iteration runs in fp64 with sums in index order; the kept zero is
rounded once to bf16 and the codes are then taken with the same fp32 rule as RTN from the stored
(s, z).  Rewritten in (s, z) from HQQ's (scale' = 1/s, zero' = -z/s): the same iterates.
"""
import numpy as np

from .numerics import round_bf16

HQQ_P, HQQ_BETA0, HQQ_KAPPA, HQQ_ITERS = 0.7, 10.0, 1.01, 20



def _f32_to_bf16_f32(x32):
    """Round fp32 -> bf16 (RNE), returned as fp32 values."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    bias = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return (((u + bias) >> np.uint32(16)) << np.uint32(16)).view(np.float32)


def _seqsum(v):
    """sum over the last axis in index order (fp64): ((v0 + v1) + v2) + ..."""
    acc = np.zeros(v.shape[:-1], dtype=np.float64)
    for i in range(v.shape[-1]):
        acc = acc + v[..., i]
    return acc


def hqq_shrink(e, beta, p=HQQ_P):
    """W_e = sign(e) * max(|e| - |e|^(p-1)/beta, 0); e = 0 gives 0."""
    a = np.abs(e)
    with np.errstate(divide="ignore"):
        t = a - np.power(a, p - 1.0) / beta
    return np.sign(e) * np.maximum(t, 0.0)


def hqq_step(x, s, z, beta, bits=4, p=HQQ_P):
    """One half-quadratic iteration for zero z (x: [..., group], s and z: [...]).  Returns
    (err, z_next, code, W_e): err = mean |x - W_r(z)| of the current zero, W_e the shrunk residual
    and z_next = argmin_z' sum (x - W_e - code*s - z')^2 = mean(x - W_e - code*s)."""
    qmax = float((1 << bits) - 1)
    s = np.asarray(s, dtype=np.float64)[..., None]
    zz = np.asarray(z, dtype=np.float64)[..., None]
    n = x.shape[-1]
    code = np.clip(np.rint((x - zz) / s), 0.0, qmax)
    e = x - (code * s + zz)
    err = _seqsum(np.abs(e)) / n
    we = hqq_shrink(e, beta, p)
    z_next = _seqsum((x - we) - code * s) / n
    return err, z_next, code, we


def hqq_refine_zero(x, s, z0, bits=4, iters=HQQ_ITERS, p=HQQ_P, beta0=HQQ_BETA0, kappa=HQQ_KAPPA,
                    trace=False):
    """x: [..., group] bf16 values (fp64); s, z0: [...] the RTN scale and zero (bf16 values).
    Returns the kept zero (fp64, before bf16 rounding) and, with trace=True, also the list of the
    per-iteration mean |x - W_r| arrays (inf where a group had already stopped)."""
    x = np.asarray(x, dtype=np.float64)
    z = np.array(z0, dtype=np.float64)
    best_z = z.copy()
    best_err = np.full(z.shape, np.inf)
    active = np.ones(z.shape, dtype=bool)
    beta = beta0
    errs = []
    for _ in range(iters):
        err, z_next, _, _ = hqq_step(x, s, z, beta, bits, p)
        errs.append(np.where(active, err, np.inf))
        improve = active & (err < best_err)
        best_err = np.where(improve, err, best_err)
        best_z = np.where(improve, z, best_z)
        active = improve
        if not active.any():
            break
        z = np.where(active, z_next, z)
        beta = beta * kappa
    return (best_z, errs) if trace else best_z


def quantize(w, bits=4, group=64, method="rtn", hqq_iters=HQQ_ITERS):
    """w: float array [N, K] of bf16-representable values.
    Returns (codes uint8 [N, K], s float64 [N, K/group], z float64 [N, K/group]),
    s and z being bf16-representable.  method: "rtn" (min/max round-to-nearest) or "hqq" (the RTN
    scale with the half-quadratic zero, module docstring)."""
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
    if method == "hqq":
        zr = hqq_refine_zero(x32.astype(np.float64), s32.astype(np.float64), m.astype(np.float64), bits,
                             iters=hqq_iters)
        z32 = round_bf16(zr).astype(np.float32)
    elif method != "rtn":
        raise ValueError(f"unknown quantizer {method!r}")
    t = ((x32 - z32[..., None]).astype(np.float32) / s32[..., None]).astype(np.float32)
    codes = np.clip(np.rint(t), 0, qmax).astype(np.uint8)       # np.rint: half-to-even
    return codes.reshape(N, K), s32.astype(np.float64), z32.astype(np.float64)


def dequantize(codes, s, z, group=64):
    """W_hat[n,k] = code*s + z, exact in float64 (a <=8-bit x 8-bit significand product plus an
    8-bit-significand addend of nearby magnitude)."""
    N, K = codes.shape
    c = codes.astype(np.float64).reshape(N, K // group, group)
    return (c * s[..., None] + z[..., None]).reshape(N, K)


def substitute_matrix(w, bits=4, group=64, method="rtn"):
    codes, s, z = quantize(w, bits, group, method)
    return dequantize(codes, s, z, group)
