"""ss_load_weights from caller-owned host arrays (`const ss_host_weights*`, bf16,
out x in row-major; PAPER.md:133-139 — the substitutes are derived from the target's own weights).

The host arrays come from synth/weights.py (the host copy of the generator); the library tiles and
places them itself.  Checks: every matrix group reads back bitwise equal to the host arrays; the
substitutes built from them equal the oracle's quantizer bitwise; the decode output equals the
oracle's greedy AR output (and the device-generator context's output bitwise)."""
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.weights import generate_model
from synth.prompts import mtbench_prompt
from gpu_util import assert_matches_oracle_ar
from oracle.quant import quantize
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _group_natural(w, cfg, l, g):
    if g == 0:
        return np.concatenate([w[f"l{l}.wq"], w[f"l{l}.wk"], w[f"l{l}.wv"]])
    if g == 1:
        return w[f"l{l}.wo"]
    if g == 2:   # rows interleaved per 64: gate 64, up 64, ...
        gt, up = w[f"l{l}.wg"], w[f"l{l}.wu"]
        out = np.empty((2 * cfg.ffn, cfg.hidden), np.uint16)
        for b in range(cfg.ffn // 64):
            out[128 * b: 128 * b + 64] = gt[64 * b: 64 * b + 64]
            out[128 * b + 64: 128 * b + 128] = up[64 * b: 64 * b + 64]
        return out
    return w[f"l{l}.wd"]


@pytest.mark.parametrize("cfg,n_res,embed_on_host", [(TINY, 1, 1), (SMALL, 1, 0), (SMALL, 0, 1)],
                         ids=["tiny", "small-embed-gpu", "small-allsub"])
def test_host_weights_roundtrip_and_decode(cuda_required, cfg, n_res, embed_on_host):
    from paper_2509_18344_b200.binding import SubSpec
    w = generate_model(cfg, SEED)
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, embed_on_host=embed_on_host)
    ss.load_weights(w, n_resident=n_res)
    for l in range(cfg.n_layers):
        for g in range(4):
            assert np.array_equal(ss.debug_read_group(l, g), _group_natural(w, cfg, l, g)), (l, g)
    ss.build_substitutes(4, 64)
    for l in range(n_res, cfg.n_layers):
        codes, s, z = ss.debug_get_substitute(l, 1)
        oc, osz, oz = quantize(bf16_bits_to_f64(w[f"l{l}.wo"]), 4, 64)
        assert np.array_equal(codes, oc)
        assert np.array_equal(bf16_bits_to_f64(s), osz) and np.array_equal(bf16_bits_to_f64(z), oz)
    prompt = mtbench_prompt(SEED, 4, cfg.vocab, 40)
    out, _ = ss.generate(prompt, 24, 4, 6, 0.2)
    ss.close()
    gen = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, embed_on_host=embed_on_host)
    gen.load_synthetic(SEED, n_resident=n_res)
    gen.build_substitutes(4, 64)
    out2, _ = gen.generate(prompt, 24, 4, 6, 0.2)
    gen.close()
    assert out == out2
    assert_matches_oracle_ar(cfg, prompt, out, SEED)


def test_host_weights_errors(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec, SubSpecError
    w = generate_model(TINY, SEED)
    ss = SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6)
    bad = dict(w)
    bad["l0.wq"] = bad["l0.wq"][:-1]
    with pytest.raises(ValueError):
        ss.load_weights(bad, 1)
    ss.load_weights(w, 1)
    with pytest.raises(SubSpecError):   # already loaded
        ss.load_weights(w, 1)
    ss.close()
