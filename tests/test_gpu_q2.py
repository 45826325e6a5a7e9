"""GPU parity of 2- and 3-bit substitutes ("more aggressive methods
(e.g., 2-bit or 3-bit quantization) could further reduce VRAM demands").

The rule is the 4-bit one with 2^bits - 1 levels (oracle/quant.py), packed in the Q2 / Q3 layouts
(common.cuh: Q3 = the Q2 plane of the low two bits + a plane of high bits).  Checks: K1 codes / s / z bit-exact vs the oracle quantizer; K2 one-hot activations
reproduce W_hat = code*s + z bit-exactly and random activations agree within fp32 accumulation
error; the lockstep draft logits vs the oracle's 2-bit draft; SubSpec output with a 2-bit draft ==
GPU AR output bitwise (lossless: the draft only proposes) and == the oracle's greedy AR output;
footprint: the substitutes take 0.3125 (0.4375) B/weight and the freed arena goes to the streaming ring.
"""
import numpy as np
import pytest

from synth import weights as W
from synth.configs import TINY, SMALL, QWEN7B, GIB
from synth.prompts import mtbench_prompt
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64
from oracle.decode import Session, ar_generate
from oracle.tree import Tree
from gpu_util import assert_close_scaled, assert_matches_oracle_ar

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _ctx(cfg, cap=512 << 20, n_resident=1, D=4, k=6, bits=2):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, cap, max_depth=D, max_top_k=k)
    ss.set_substitute_bits(bits)
    ss.load_synthetic(SEED, n_resident=n_resident)
    ss.build_substitutes(bits, 64)
    return ss


@pytest.fixture(scope="module", params=[(TINY, 2), (SMALL, 2), (TINY, 3), (SMALL, 3)],
                ids=["tiny-2", "small-2", "tiny-3", "small-3"])
def ctx(request, cuda_required):
    cfg, bits = request.param
    ss = _ctx(cfg, bits=bits)
    ss.bits = bits
    yield cfg, ss
    ss.close()


def test_q2_substitutes_bit_exact(ctx):
    cfg, ss = ctx
    for l in range(1, cfg.n_layers):
        for g in range(4):
            w = bf16_bits_to_f64(ss.debug_read_group(l, g))
            codes, s, z = ss.debug_get_substitute(l, g)
            rc, rs, rz = quantize(w, bits=ss.bits)
            assert codes.max() <= (1 << ss.bits) - 1
            assert np.array_equal(codes, rc), (l, g)
            assert np.array_equal(bf16_bits_to_f64(s), rs) and np.array_equal(bf16_bits_to_f64(z), rz), (l, g)


def test_q2_k2_one_hot_exact(ctx):
    cfg, ss = ctx
    for g in range(4):
        N, K = ss.group_shape(g)
        what = dequantize(*quantize(bf16_bits_to_f64(ss.debug_read_group(1, g)), bits=ss.bits))
        for k0 in range(0, K, 32):
            M = min(32, K - k0)
            x = np.zeros((M, K), np.uint16)
            x[np.arange(M), k0 + np.arange(M)] = 0x3F80
            y = ss.debug_matmul(0, 1, g, x).astype(np.float64)
            assert np.array_equal(y, what[:, k0:k0 + M].T), (g, k0)


@pytest.mark.parametrize("M", [1, 6, 13, 32])
def test_q2_k2_random_activations(ctx, M):
    cfg, ss = ctx
    rng = np.random.default_rng(100 + M)
    for g in range(4):
        N, K = ss.group_shape(g)
        what = dequantize(*quantize(bf16_bits_to_f64(ss.debug_read_group(1, g)), bits=ss.bits))
        xb = W.f32_to_bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
        y = ss.debug_matmul(0, 1, g, xb)
        ref = bf16_bits_to_f64(xb) @ what.T
        bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(what).T) + 1e-6
        assert np.all(np.abs(y - ref) <= bound), (g, M, float(np.max(np.abs(y - ref))))


@pytest.mark.parametrize("bits", [2, 3])
def test_q2_draft_logits_match_oracle(cuda_required, bits):
    cfg, D, k = SMALL, 3, 4
    ss = _ctx(cfg, n_resident=0, D=D, k=k, bits=bits)
    ors = Session(cfg, SEED, n_resident=0, bits=bits, mode="bf16", max_nodes=256)
    prompt = mtbench_prompt(SEED, 2, cfg.vocab, 40)
    assert ss.prefill(prompt) == ors.prefill(prompt)
    tr = ss.draft_tree(D, k, 0.2)
    g_draft = ss.debug_forward(0, tr["tokens"], tr["parents"])
    tree = Tree([int(t) for t in tr["tokens"]], [int(p) for p in tr["parents"]],
                [int(d) for d in tr["depths"]], [float(s) for s in tr["scores"]])
    o_draft = ors.forward_tree("draft", tree)
    assert_close_scaled(g_draft[:1 + k * (D - 1)], o_draft[:1 + k * (D - 1)], what=f"{bits}-bit draft logits")
    ss.close()


@pytest.mark.parametrize("cfg,n_res,D,k,bits", [(TINY, 1, 4, 6, 2), (SMALL, 0, 6, 2, 2), (SMALL, 0, 6, 2, 3)],
                         ids=["tiny-2", "small-allsub-2", "small-allsub-3"])
def test_q2_sd_equals_ar(cuda_required, cfg, n_res, D, k, bits):
    ss = _ctx(cfg, n_resident=n_res, D=D, k=k, bits=bits)
    for p in range(2):
        prompt = mtbench_prompt(SEED, p, cfg.vocab, 32 + 17 * p)
        sd, hist = ss.generate(prompt, 32, D, k, 0.2)
        ar, _ = ss.generate(prompt, 32, 0, 1, 0.2)
        assert sd == ar, f"prompt {p}: SubSpec ({bits}-bit draft) output differs from the GPU AR output"
        assert_matches_oracle_ar(cfg, prompt, sd, SEED)
    ss.close()


@pytest.mark.parametrize("bits", [2, 3])
def test_q2_qwen7b_footprint_and_lossless(cuda_required, bits):
    """Qwen2.5-7B shape, 8 GiB, 0 resident: substitutes 2.04 / 2.86 GB (vs 3.67 at 4 bits), the ring
    grows by the difference, sampled GEMV rows match the oracle, and SD == GPU AR bitwise."""
    from paper_2509_18344_b200.binding import SubSpec
    ss = _ctx(QWEN7B, cap=8 * GIB, n_resident=0, D=6, k=6, bits=bits)
    st = ss.stats()
    L, H, F = QWEN7B.n_layers, QWEN7B.hidden, QWEN7B.ffn
    qd = (QWEN7B.n_heads + 2 * QWEN7B.n_kv_heads) * QWEN7B.head_dim
    params = qd * H + H * QWEN7B.n_heads * QWEN7B.head_dim + 2 * F * H + H * F
    per16 = {2: 5, 3: 7}[bits]                                   # B/weight x 16: codes + bf16 s, z per 64
    assert st["substitute_bytes"] == L * params * per16 // 16
    assert st["ring_bytes"] > {2: 4.5e9, 3: 3.9e9}[bits]         # vs ~3.26 GB with 4-bit substitutes
    rng = np.random.default_rng(5)
    for g in (0, 3):
        N, K = ss.group_shape(g)
        rows = np.sort(rng.choice(N, 64, replace=False))
        w = bf16_bits_to_f64(ss.debug_read_group(3, g))
        what = dequantize(*quantize(w[rows], bits=bits))
        xb = W.f32_to_bf16_bits(rng.standard_normal((6, K)).astype(np.float32))
        y = ss.debug_matmul(0, 3, g, xb)[:, rows]
        ref = bf16_bits_to_f64(xb) @ what.T
        bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(what).T) + 1e-6
        assert np.all(np.abs(y - ref) <= bound), g
    prompt = mtbench_prompt(SEED, 0, QWEN7B.vocab, 64)
    sd, _ = ss.generate(prompt, 12, 6, 6, 0.2)
    ar, _ = ss.generate(prompt, 12, 0, 1, 0.2)
    assert sd == ar
    ss.close()


def test_q2_abi_errors(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec, SubSpecError
    ss = SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6)
    with pytest.raises(SubSpecError, match="INVALID"):
        ss.set_substitute_bits(5)                     # 4, 3 or 2 only
    ss.set_substitute_bits(2)
    ss.load_synthetic(SEED, n_resident=1)
    with pytest.raises(SubSpecError, match="STRUCTURE"):
        ss.set_substitute_bits(4)                     # the layout is fixed at placement
    with pytest.raises(SubSpecError, match="INVALID"):
        ss.build_substitutes(4, 64)                   # must match the placed layout
    ss.build_substitutes(2, 64)
    ss.close()
