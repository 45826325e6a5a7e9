"""Counter-based weight generator — SURVEY.md §8(c) O.1 (SPEC.md:40-48 `init_random`
made bit-exact across CPU and GPU).

Every tensor has an id `tid`; element i (row-major) of tensor tid is

    key = splitmix64(seed ^ (tid * 0xD1B54A32D192ED03 mod 2^64))
    r   = splitmix64(key ^ i)
    S2  = 2 * sum_{j=0..3} ((r >> 16j) & 0xFFFF) - 4*65535        (Irwin-Hall(4), |S2| < 2^18)
    w32 = fp32(S2) * c32                                           (one IEEE fp32 multiply)
    w   = RNE_bf16(w32)

with c32 = fp32((sigma * sqrt(12)) / 262144) computed in fp64 and rounded once.
Norm gains are RNE_bf16(fp32(1.0f + w32)) with sigma = 0.05 (two separately
rounded fp32 ops, never an FMA).  sigma: matrices 1/sqrt(fan_in), embedding 1,
norm gains 0.05, biases 0.02.

This module is an input generator only.  csrc/gen.cu implements the same
generator independently for the GPU; tests/test_synth.py pins this copy to
published splitmix64 outputs and to its statistical moments, and
tests/test_gpu_weights.py checks both agree bitwise.
"""
import math
import numpy as np

from .configs import ModelConfig

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TID_MUL = 0xD1B54A32D192ED03

# per-layer tensor slots (tid = 1 + 16*layer + slot)
SLOTS = ("attn_norm", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "mlp_norm", "wg", "wu", "wd")
SLOT_ID = {s: i for i, s in enumerate(SLOTS)}


def splitmix64_scalar(x: int) -> int:
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def tensor_key(seed: int, tid: int) -> int:
    return splitmix64_scalar((seed ^ ((tid * TID_MUL) & MASK64)) & MASK64)


def irwin_hall_s2(key: int, start: int, count: int) -> np.ndarray:
    """Integer S2 values (int32) for element indices [start, start+count)."""
    i = np.arange(start, start + count, dtype=np.uint64)
    r = splitmix64(i ^ np.uint64(key))
    s = np.zeros(count, dtype=np.int64)
    for j in range(4):
        s += ((r >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64)
    return (2 * s - 4 * 65535).astype(np.int32)


def f32_to_bf16_bits(x32: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 (finite inputs)."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    bias = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + bias) >> np.uint32(16)).astype(np.uint16)


def scale_c32(sigma: float) -> np.float32:
    return np.float32((sigma * math.sqrt(12.0)) / 262144.0)


def tensor_specs(cfg: ModelConfig):
    """[(tid, name, shape, kind, sigma)] for every tensor of the model, in tid order.
    kind: 'mat' | 'gain' | 'bias'."""
    H, L = cfg.hidden, cfg.n_layers
    specs = [(0, "embed", (cfg.vocab, H), "mat", 1.0)]
    for l in range(L):
        base = 1 + 16 * l
        specs.append((base + 0, f"l{l}.attn_norm", (H,), "gain", 0.05))
        specs.append((base + 1, f"l{l}.wq", (cfg.q_dim, H), "mat", 1.0 / math.sqrt(H)))
        if cfg.qkv_bias:
            specs.append((base + 2, f"l{l}.bq", (cfg.q_dim,), "bias", 0.02))
        specs.append((base + 3, f"l{l}.wk", (cfg.kv_dim, H), "mat", 1.0 / math.sqrt(H)))
        if cfg.qkv_bias:
            specs.append((base + 4, f"l{l}.bk", (cfg.kv_dim,), "bias", 0.02))
        specs.append((base + 5, f"l{l}.wv", (cfg.kv_dim, H), "mat", 1.0 / math.sqrt(H)))
        if cfg.qkv_bias:
            specs.append((base + 6, f"l{l}.bv", (cfg.kv_dim,), "bias", 0.02))
        specs.append((base + 7, f"l{l}.wo", (H, cfg.q_dim), "mat", 1.0 / math.sqrt(cfg.q_dim)))
        specs.append((base + 8, f"l{l}.mlp_norm", (H,), "gain", 0.05))
        specs.append((base + 9, f"l{l}.wg", (cfg.ffn, H), "mat", 1.0 / math.sqrt(H)))
        specs.append((base + 10, f"l{l}.wu", (cfg.ffn, H), "mat", 1.0 / math.sqrt(H)))
        specs.append((base + 11, f"l{l}.wd", (H, cfg.ffn), "mat", 1.0 / math.sqrt(cfg.ffn)))
    specs.append((1 + 16 * L, "final_norm", (H,), "gain", 0.05))
    specs.append((2 + 16 * L, "head", (cfg.vocab, H), "mat", 1.0 / math.sqrt(H)))
    return specs


def gen_tensor_bits(seed: int, tid: int, shape, kind: str, sigma: float,
                    rows: slice | None = None) -> np.ndarray:
    """bf16 bit patterns (uint16) of one tensor (optionally only a row range of a matrix)."""
    key = tensor_key(seed, tid)
    if len(shape) == 2 and rows is not None:
        r0, r1, _ = rows.indices(shape[0])
        start, count, out_shape = r0 * shape[1], (r1 - r0) * shape[1], (r1 - r0, shape[1])
    else:
        start, count, out_shape = 0, int(np.prod(shape)), shape
    c = scale_c32(sigma)
    w32 = irwin_hall_s2(key, start, count).astype(np.float32) * c
    if kind == "gain":
        w32 = np.float32(1.0) + w32
    return f32_to_bf16_bits(w32).reshape(out_shape)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def generate_model(cfg: ModelConfig, seed: int):
    """dict name -> bf16 bit pattern array (uint16).  Intended for small configs."""
    return {name: gen_tensor_bits(seed, tid, shape, kind, sigma)
            for tid, name, shape, kind, sigma in tensor_specs(cfg)}


def checksum_bits(b: np.ndarray) -> int:
    """Order-sensitive 64-bit checksum of a bf16 bit array: sum_i (i+1) * bits[i] mod 2^64."""
    v = np.asarray(b, dtype=np.uint16).reshape(-1).astype(np.uint64)
    idx = np.arange(1, v.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum(v * idx, dtype=np.uint64))
