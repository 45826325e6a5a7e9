"""GPU parity of K1's HQQ zero refinement (reading R28; oracle/quant.py):
codes, scales and zeros bit-exact against oracle.quant.quantize(method="hqq") for 4- and 2-bit
substitutes at the tiny/small shapes and on sampled rows of a Qwen2.5-7B-width layer, and the HQQ
substitutes' reconstruction error below RTN's.  The decode lockstep with HQQ drafts is
tests/test_gpu_decode.py::test_lockstep[small-allsub-hqq-D4k6]."""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import TINY, SMALL, QWEN7B, GIB
from synth.prompts import mtbench_prompt
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _groups(model, cfg, l):
    qkv = np.concatenate([model[f"l{l}.wq"], model[f"l{l}.wk"], model[f"l{l}.wv"]])
    gu = np.zeros((2 * cfg.ffn, cfg.hidden), np.uint16)
    for b in range(cfg.ffn // 64):
        gu[128 * b:128 * b + 64] = model[f"l{l}.wg"][64 * b:64 * b + 64]
        gu[128 * b + 64:128 * b + 128] = model[f"l{l}.wu"][64 * b:64 * b + 64]
    return [qkv, model[f"l{l}.wo"], gu, model[f"l{l}.wd"]]


@pytest.mark.parametrize("cfg,bits", [(TINY, 4), (SMALL, 4), (SMALL, 2)], ids=["tiny-4", "small-4", "small-2"])
def test_hqq_substitutes_bit_exact(cuda_required, cfg, bits):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6)
    if bits != 4:
        ss.set_substitute_bits(bits)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(bits, 64, method="hqq")
    model = W.generate_model(cfg, SEED)
    improved = []
    for l in range(cfg.n_layers):
        refs = _groups(model, cfg, l)
        for g in range(4):
            codes, s, z = ss.debug_get_substitute(l, g)
            x = bf16_bits_to_f64(refs[g])
            rc, rs, rz = quantize(x, bits, 64, "hqq")
            assert np.array_equal(bf16_bits_to_f64(s), rs), (l, g, "scale")
            assert np.array_equal(bf16_bits_to_f64(z), rz), (l, g, "zero")
            assert np.array_equal(codes, rc), (l, g, "codes")
            qc, qs, qz = quantize(x, bits, 64, "rtn")
            improved.append(np.mean(np.abs(dequantize(rc, rs, rz) - x)) < np.mean(np.abs(dequantize(qc, qs, qz) - x)))
    assert all(improved)
    ss.close()


def test_hqq_qwen7b_sampled_rows(cuda_required):
    """Qwen2.5-7B-width layer 0 (all layers offloaded, the bench's placement): sampled row blocks of
    every matrix group bit-exact (the oracle quantizes only the sampled rows: groups lie in rows)."""
    from paper_2509_18344_b200.binding import SubSpec
    cfg = QWEN7B
    ss = SubSpec(cfg, 8 * GIB, max_depth=48, max_top_k=6)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(4, 64, method="hqq")
    spec = {name: (tid, shape, kind, sigma) for tid, name, shape, kind, sigma in W.tensor_specs(cfg)}
    rng = np.random.default_rng(7)

    def rows_of(name, r0, r1):
        tid, shape, kind, sigma = spec[name]
        return W.gen_tensor_bits(SEED, tid, shape, kind, sigma, rows=slice(r0, r1))

    for g in range(4):
        codes, s, z = ss.debug_get_substitute(0, g)
        N = codes.shape[0]
        for r0 in sorted(set([0, N - 64] + [int(v) * 64 for v in rng.integers(0, N // 64, 2)])):
            if g == 0:   # qkv rows: [q; k; v]
                parts, off = [], 0
                for nm in ("wq", "wk", "wv"):
                    n_nm = spec[f"l0.{nm}"][1][0]
                    lo, hi = max(r0, off), min(r0 + 64, off + n_nm)
                    if lo < hi:
                        parts.append(rows_of(f"l0.{nm}", lo - off, hi - off))
                    off += n_nm
                ref = np.concatenate(parts)
            elif g == 2:  # gate_up interleaved per 64 rows: block b = gate rows, then up rows
                b, half = r0 // 128, (r0 % 128) // 64
                ref = rows_of("l0.wg" if half == 0 else "l0.wu", 64 * b, 64 * b + 64)
            else:
                ref = rows_of("l0.wo" if g == 1 else "l0.wd", r0, r0 + 64)
            rc, rs, rz = quantize(bf16_bits_to_f64(ref), 4, 64, "hqq")
            assert np.array_equal(codes[r0:r0 + 64], rc), (g, r0)
            assert np.array_equal(bf16_bits_to_f64(s[r0:r0 + 64]), rs), (g, r0)
            assert np.array_equal(bf16_bits_to_f64(z[r0:r0 + 64]), rz), (g, r0)
    ss.close()


def test_hqq_decode_lossless(cuda_required):
    """HQQ drafts change only the tree, never the output: SubSpec == GPU AR bitwise == oracle AR."""
    from paper_2509_18344_b200.binding import SubSpec
    from gpu_util import assert_matches_oracle_ar
    cfg = SMALL
    prompt = mtbench_prompt(SEED, 2, cfg.vocab, 48)
    outs = {}
    for method, D in (("hqq", 4), ("hqq", 0)):
        ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6)
        ss.load_synthetic(SEED, n_resident=0)
        ss.build_substitutes(4, 64, method=method)
        outs[D], _ = ss.generate(prompt, 32, depth=D, top_k=6, sharpen_t=0.2)
        ss.close()
    assert outs[4] == outs[0]
    assert_matches_oracle_ar(cfg, prompt, outs[4], SEED)
