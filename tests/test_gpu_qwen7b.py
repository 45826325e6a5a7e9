"""Full-size GPU parity at BASELINE.json config 2 (Qwen2.5-7B shape, 8 GiB cap, all 28 layers
offloaded with 4-bit/g64 substitutes, D = 48, k = 6 - the configuration bench.py times).

* K1 on sampled rows of every matrix group: codes/s/z bit-exact vs the oracle quantizer run on the
  generator's rows;
* K2 (M = k = 6) on sampled output rows vs the fp64 oracle dot products;
* end to end: SubSpec steps emit exactly the GPU AR sequence (batch-invariant target path), tau in
  [1, D+1], committed length bookkeeping.
"""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import QWEN7B, GIB
from synth.prompts import mtbench_prompt
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED
D, K_TOP = 48, 6


@pytest.fixture(scope="module")
def q7(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(QWEN7B, 8 * GIB, max_depth=D, max_top_k=K_TOP, max_chunk=256)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(4, 64)
    yield ss
    ss.close()


def _fused_rows(layer, g, rows):
    """Generator rows of the fused (layer, group) matrix, fused row order (see subspec.h)."""
    cfg = QWEN7B
    b = 1 + 16 * layer
    H, F = cfg.hidden, cfg.ffn
    out = []
    for r in rows:
        if g == 0:
            if r < cfg.q_dim:
                tid, src, K, sig = b + 1, r, H, 1 / np.sqrt(H)
            elif r < cfg.q_dim + cfg.kv_dim:
                tid, src, K, sig = b + 3, r - cfg.q_dim, H, 1 / np.sqrt(H)
            else:
                tid, src, K, sig = b + 5, r - cfg.q_dim - cfg.kv_dim, H, 1 / np.sqrt(H)
            shape = (cfg.q_dim if tid == b + 1 else cfg.kv_dim, H)
        elif g == 1:
            tid, src, shape, sig = b + 7, r, (H, cfg.q_dim), 1 / np.sqrt(cfg.q_dim)
        elif g == 2:
            blk, i = divmod(r, 128)
            tid = b + 9 if i < 64 else b + 10
            src, shape, sig = 64 * blk + (i % 64), (F, H), 1 / np.sqrt(H)
        else:
            tid, src, shape, sig = b + 11, r, (H, F), 1 / np.sqrt(F)
        out.append(W.gen_tensor_bits(SEED, tid, shape, "mat", sig, rows=slice(src, src + 1))[0])
    return np.stack(out)


@pytest.mark.parametrize("layer", [0, 27])
def test_k1_sampled_rows_bit_exact(q7, layer):
    rng = np.random.default_rng(layer)
    for g in range(4):
        N, K = q7.group_shape(g)
        codes, s, z = q7.debug_get_substitute(layer, g)
        rows = sorted(set([0, 1, N - 1] + rng.integers(0, N, 13).tolist()))
        ref = _fused_rows(layer, g, rows)
        rc, rs, rz = quantize(bf16_bits_to_f64(ref))
        assert np.array_equal(codes[rows], rc), (layer, g)
        assert np.array_equal(bf16_bits_to_f64(s[rows]), rs) and np.array_equal(bf16_bits_to_f64(z[rows]), rz)


@pytest.mark.parametrize("layer", [3])
def test_k2_sampled_rows_at_full_shape(q7, layer):
    rng = np.random.default_rng(11)
    for g in range(4):
        N, K = q7.group_shape(g)
        xb = W.f32_to_bf16_bits(rng.standard_normal((K_TOP, K)).astype(np.float32))
        y = q7.debug_matmul(0, layer, g, xb)
        rows = sorted(set([0, N - 1] + rng.integers(0, N, 30).tolist()))
        what = dequantize(*quantize(bf16_bits_to_f64(_fused_rows(layer, g, rows))))
        ref = bf16_bits_to_f64(xb) @ what.T
        bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(what).T) + 1e-6
        assert np.all(np.abs(y[:, rows] - ref) <= bound), g


def test_sd_steps_equal_gpu_ar(q7):
    prompt = mtbench_prompt(SEED, 0, QWEN7B.vocab)
    sd, hist = q7.generate(prompt, 24, D, K_TOP, 0.2)
    st = q7.stats()
    assert st["committed_len"] == len(prompt) + sum(i * int(h) for i, h in enumerate(hist))
    assert hist[0] == 0 and hist.sum() >= 1
    ar, _ = q7.generate(prompt, 24, 0, 1, 0.2)
    assert sd == ar
