"""Pins for the seeded input generators (synth/): SURVEY.md §8(c) O.1, §8(d) prompts."""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import TINY, SMALL, QWEN7B, PRESETS
from synth.prompts import mtbench_prompt, TEMPLATE_LEN


def test_splitmix64_published_sequence():
    # SplitMix64 (Steele/Lea/Flood; Vigna's reference) seeded with 0: the first three outputs.
    g = W.GOLDEN
    outs = [W.splitmix64_scalar((i * g) & W.MASK64) for i in range(3)]
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_vectorised_matches_scalar():
    xs = [0, 1, 2**63 + 5, 0xDEADBEEFCAFEBABE]
    v = W.splitmix64(np.array(xs, dtype=np.uint64))
    assert [int(a) for a in v] == [W.splitmix64_scalar(x) for x in xs]


def test_irwin_hall_range_and_parity():
    s = W.irwin_hall_s2(W.tensor_key(1, 1), 0, 200_000)
    assert s.min() >= -4 * 65535 and s.max() <= 4 * 65535
    assert np.all(s % 2 == 0)          # 2*sum - 4*65535 is even


@pytest.mark.parametrize("sigma", [1.0, 1 / 16, 0.02])
def test_moments(sigma):
    # Irwin-Hall(4) rescaled: mean 0, std sigma, excess kurtosis -6/(5*4) = -0.3, |w| <= sqrt(12) sigma
    b = W.gen_tensor_bits(0x5EED, 3, (400, 1000), "mat", sigma)
    x = W.bf16_bits_to_f32(b).astype(np.float64)
    assert abs(x.mean()) < 0.01 * sigma
    assert abs(x.std() / sigma - 1) < 0.01
    k = ((x - x.mean()) ** 4).mean() / x.var() ** 2 - 3
    assert abs(k + 0.3) < 0.05
    assert np.abs(x).max() <= np.sqrt(12) * sigma * 1.01


def test_gain_centred_on_one():
    b = W.gen_tensor_bits(7, 1, (100_000,), "gain", 0.05)
    x = W.bf16_bits_to_f32(b).astype(np.float64)
    assert abs(x.mean() - 1) < 1e-3 and abs(x.std() - 0.05) < 2e-3


def test_determinism_and_seed_sensitivity():
    a = W.generate_model(TINY, 7)
    b = W.generate_model(TINY, 7)
    c = W.generate_model(TINY, 8)
    assert all(np.array_equal(a[k], b[k]) for k in a)
    assert any(not np.array_equal(a[k], c[k]) for k in a)


def test_row_slice_consistent():
    full = W.gen_tensor_bits(3, 17, (64, 96), "mat", 0.1)
    part = W.gen_tensor_bits(3, 17, (64, 96), "mat", 0.1, rows=slice(10, 20))
    assert np.array_equal(full[10:20], part)


def test_tensor_ids_unique_and_shapes():
    for cfg in PRESETS.values():
        specs = W.tensor_specs(cfg)
        tids = [s[0] for s in specs]
        assert len(set(tids)) == len(tids)
        n = sum(int(np.prod(s[2])) for s in specs if s[1].startswith("l0."))
        extra = (cfg.qkv_rows if cfg.qkv_bias else 0) + 2 * cfg.hidden
        assert n == cfg.params_per_layer() + extra


def test_qwen7b_layer_bytes():
    # 233.05 M params / layer, 466.1 MB bf16, 131.1 MB at 4.5 bit/weight
    p = QWEN7B.params_per_layer()
    assert abs(p / 1e6 - 233.05) < 0.01
    assert abs(2 * p / 1e6 - 466.1) < 0.1
    assert abs(p * 0.5625 / 1e6 - 131.1) < 0.1


def test_prompt_recipe():
    ps = [mtbench_prompt(0x5EED, p, QWEN7B.vocab) for p in range(40)]
    lens = [len(p) for p in ps]
    assert min(lens) >= 64 and max(lens) <= 256
    assert all(np.array_equal(ps[0][:TEMPLATE_LEN], p[:TEMPLATE_LEN]) for p in ps)
    assert all(p.min() >= 0 and p.max() < QWEN7B.vocab for p in ps)
    assert np.array_equal(ps[3], mtbench_prompt(0x5EED, 3, QWEN7B.vocab))
