"""GPU parity: counter-based generator and K1 substitute quantizer (O.2), bit-exact."""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import TINY, SMALL, QWEN7B
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED


@pytest.fixture(scope="module")
def small_ctx(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(SMALL, 512 << 20, max_depth=6, max_top_k=6, max_chunk=256)
    yield ss
    ss.close()


def test_device_generator_matches_numpy(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6)
    for tid, name, shape, kind, sigma in W.tensor_specs(TINY):
        got = ss.debug_gen_tensor(SEED, tid, shape, kind, sigma)
        assert np.array_equal(got.reshape(shape), W.gen_tensor_bits(SEED, tid, shape, kind, sigma)), name
    # Qwen2.5-7B tensor ids / scales on row slices (the generator is counter-based: row slices are exact)
    for tid, name, shape, kind, sigma in W.tensor_specs(QWEN7B)[:14] + W.tensor_specs(QWEN7B)[-2:]:
        rows = min(shape[0], 64) if len(shape) == 2 else None
        sh = (rows, shape[1]) if rows else shape
        got = ss.debug_gen_tensor(SEED, tid, sh, kind, sigma)
        ref = W.gen_tensor_bits(SEED, tid, shape, kind, sigma, rows=slice(0, rows)) if rows else \
            W.gen_tensor_bits(SEED, tid, shape, kind, sigma)
        assert np.array_equal(got.reshape(ref.shape), ref), name
    ss.close()


@pytest.mark.parametrize("cfg", [TINY, SMALL], ids=["tiny", "small"])
def test_placed_weights_and_substitutes_bit_exact(cuda_required, cfg):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6)
    ss.load_synthetic(SEED, n_resident=1)
    ss.build_substitutes(4, 64)
    model = W.generate_model(cfg, SEED)
    for l in range(cfg.n_layers):
        qkv = np.concatenate([model[f"l{l}.wq"], model[f"l{l}.wk"], model[f"l{l}.wv"]])
        gu = np.zeros((2 * cfg.ffn, cfg.hidden), np.uint16)
        for b in range(cfg.ffn // 64):
            gu[128 * b:128 * b + 64] = model[f"l{l}.wg"][64 * b:64 * b + 64]
            gu[128 * b + 64:128 * b + 128] = model[f"l{l}.wu"][64 * b:64 * b + 64]
        refs = [qkv, model[f"l{l}.wo"], gu, model[f"l{l}.wd"]]
        for g in range(4):
            assert np.array_equal(ss.debug_read_group(l, g), refs[g]), (l, g)
            if l >= 1:   # offloaded: K1 codes, s, z bit-exact vs the oracle quantizer
                codes, s, z = ss.debug_get_substitute(l, g)
                rc, rs, rz = quantize(bf16_bits_to_f64(refs[g]))
                assert np.array_equal(codes, rc), (l, g)
                assert np.array_equal(bf16_bits_to_f64(s), rs) and np.array_equal(bf16_bits_to_f64(z), rz), (l, g)
    ss.close()
