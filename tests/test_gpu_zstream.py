"""K7 stream codec (zstream.cu, ss_options.compress_stream): the streamed target layers cross the host
link as lossless exponent-coded blobs and are decoded on the GPU before the verify GEMM (SURVEY §8(a)
A4).

* exactness: every offloaded group decoded by the GPU kernel equals the generator's bf16 weights
  bitwise (and the CPU decoder of the same blob), at tiny/small and at the Qwen2.5-7B widths where the
  7 most frequent exponents of each matrix leave ~0.3% exceptions;
* a matrix with no exponent structure (uniformly random exponents) falls back to a raw blob, still
  bit-exact;
* the method's output is unchanged: SubSpec with and without the codec emit the same tokens, equal
  to the oracle's greedy AR output;
* the bytes crossing the link: <= 0.72 of the bf16 bytes for the Gaussian-like synthetic weights.
"""
import numpy as np
import pytest

from synth.configs import TINY, SMALL, QWEN7B, GIB
from synth.weights import generate_model
from synth.prompts import mtbench_prompt
from gpu_util import assert_matches_oracle_ar

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _ctx(cfg, cap, compress, n_res):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, cap, max_depth=4, max_top_k=6, compress_stream=compress)
    ss.load_synthetic(SEED, n_resident=n_res)
    return ss


@pytest.mark.parametrize("cfg,cap,n_res", [(TINY, 256 << 20, 1), (SMALL, 512 << 20, 0),
                                           (QWEN7B.with_(name="qwen2.5-7b-2l", n_layers=2), 4 * GIB, 0)],
                         ids=["tiny", "small", "qwen7b-width"])
def test_codec_bit_exact_and_smaller(cuda_required, cfg, cap, n_res):
    ss = _ctx(cfg, cap, 1, n_res)
    raw = coded = 0
    for l in range(n_res, cfg.n_layers):
        for g in range(4):
            ref = ss.debug_read_group(l, g)                # CPU decoder of the host blob
            dec, mode, nbytes = ss.debug_decode_group(l, g)
            assert mode == 1, (l, g)
            assert np.array_equal(dec, ref), (l, g)
            raw += ref.size * 2
            coded += nbytes
    if cfg is not TINY:   # the generator's weights, independently (tiny: covered by the decode tests)
        plain = _ctx(cfg, cap, 0, n_res)
        for l in range(n_res, cfg.n_layers):
            for g in range(4):
                assert np.array_equal(plain.debug_read_group(l, g), ss.debug_decode_group(l, g)[0]), (l, g)
        plain.close()
    ss.close()
    assert coded <= 0.72 * raw, coded / raw


def test_codec_raw_fallback(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec
    w = generate_model(TINY, SEED)
    rng = np.random.default_rng(1)
    bad = rng.integers(0, 1 << 16, size=w["l1.wo"].shape, dtype=np.uint16)
    bad = (bad & ~np.uint16(0x4000)).astype(np.uint16)   # finite, every exponent < 128 used
    w["l1.wo"] = bad
    ss = SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6, compress_stream=1)
    ss.load_weights(w, n_resident=1)
    dec, mode, nbytes = ss.debug_decode_group(1, 1)
    assert mode == 0 and nbytes >= bad.size * 2
    assert np.array_equal(dec, bad)
    assert np.array_equal(ss.debug_read_group(1, 1), bad)
    ss.close()


@pytest.mark.parametrize("cfg,n_res", [(TINY, 1), (SMALL, 0)], ids=["tiny", "small-allsub"])
def test_codec_output_unchanged(cuda_required, cfg, n_res):
    prompt = [int(t) for t in mtbench_prompt(SEED, 9, cfg.vocab, 40)]
    outs = []
    for compress in (1, 0):
        ss = _ctx(cfg, 512 << 20, compress, n_res)
        ss.build_substitutes(4, 64)
        out, _ = ss.generate(prompt, 32, 4, 6, 0.2)
        st = ss.stats()
        if compress:
            assert st["stream_bytes"] < 0.75 * st["stream_raw_bytes"]
        else:
            assert st["stream_bytes"] == st["stream_raw_bytes"]
        ss.close()
        outs.append(out)
    assert outs[0] == outs[1]
    assert_matches_oracle_ar(cfg, prompt, outs[0], SEED)
