"""The opt-in draft paths against the default one: the fused MLP kernel (mlp.cu, SS_FUSE_MLP=1)
and the RMSNorm folded into the next qkv GEMV (SS_XNORM=1).

Both compute gate_up -> SiLU*mul -> down (+ residual, + fused RMSNorm) from the same substitutes;
only the fp32 summation order of the down contraction differs (Stream-K segments vs cluster split),
so the draft logits agree to fp32/bf16 rounding (bound: 2e-2 x logit scale, R3 tolerance).
Covers the resident (bf16) and substitute (Q4) weight paths, M = 1 / 6 / 25 (NT = 1 / 1 / 4).
"""
import os
import numpy as np
import pytest

from synth.configs import TINY, SMALL
from synth.prompts import mtbench_prompt

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _logits(cfg, n_res, M, fused, var="SS_FUSE_MLP"):
    from paper_2509_18344_b200.binding import SubSpec
    old = os.environ.get(var)
    os.environ[var] = "1" if fused else "0"
    try:
        ss = SubSpec(cfg, 512 << 20, max_depth=8, max_top_k=6, max_chunk=256)
        ss.load_weights(SEED, n_resident=n_res)
        ss.build_substitutes(4, 64)
    finally:
        if old is None:
            del os.environ[var]
        else:
            os.environ[var] = old
    ss.prefill(mtbench_prompt(SEED, 1, cfg.vocab, 40))
    toks = (np.arange(M, dtype=np.int32) * 37 + 5) % cfg.vocab
    par = np.arange(-1, M - 1, dtype=np.int32)
    out = ss.debug_forward(0, toks, par)
    ss.close()
    return out


@pytest.mark.parametrize("cfg,n_res", [(TINY, 0), (TINY, 1), (SMALL, 0)], ids=["tiny", "tiny-res1", "small"])
@pytest.mark.parametrize("M", [1, 6, 25])
def test_fused_mlp_matches_two_gemvs(cuda_required, cfg, n_res, M):
    a = _logits(cfg, n_res, M, False)
    b = _logits(cfg, n_res, M, True)
    scale = np.abs(a).max()
    assert np.abs(a - b).max() <= 2e-2 * scale


@pytest.mark.parametrize("cfg,n_res", [(TINY, 1), (SMALL, 0)], ids=["tiny-res1", "small"])
@pytest.mark.parametrize("M", [1, 6])
def test_folded_rmsnorm_matches_default(cuda_required, cfg, n_res, M):
    a = _logits(cfg, n_res, M, False, "SS_XNORM")
    b = _logits(cfg, n_res, M, True, "SS_XNORM")
    scale = np.abs(a).max()
    assert np.abs(a - b).max() <= 2e-2 * scale


_CW16_CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from synth import weights as W
from synth.configs import SMALL
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64
from paper_2509_18344_b200.binding import SubSpec
ss = SubSpec(SMALL, 512 << 20, max_depth=4, max_top_k=6)
ss.load_weights(0x5EED, n_resident=1)
ss.build_substitutes(4, 64)
N, K = ss.group_shape(0)
what = dequantize(*quantize(bf16_bits_to_f64(ss.debug_read_group(1, 0))))
exact = True
for k0 in range(0, K, 32):
    x = np.zeros((32, K), np.uint16)
    x[np.arange(32), k0 + np.arange(32)] = 0x3F80
    exact &= bool(np.array_equal(ss.debug_matmul(0, 1, 0, x).astype(np.float64), what[:, k0:k0 + 32].T))
rng = np.random.default_rng(11)
xb = W.f32_to_bf16_bits(rng.standard_normal((6, K)).astype(np.float32))
y = ss.debug_matmul(0, 1, 0, xb)
ref = bf16_bits_to_f64(xb) @ what.T
bound = K * 2.0**-22 * (np.abs(bf16_bits_to_f64(xb)) @ np.abs(what).T) + 1e-6
print(json.dumps({"exact": exact, "within": bool(np.all(np.abs(y - ref) <= bound))}))
"""


def test_qkv_16_consumer_warps_opt_in(cuda_required):
    """SS_GEMV_CW16=1 (opt-in): the one-CTA-per-SM qkv GEMV with 16 consumer warps (two
    per row block, partial sums added at the flush) — one-hot exact, random within the fp32 bound."""
    import json, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CW16_CHILD, root], env=dict(os.environ, SS_GEMV_CW16="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["exact"] and res["within"], res
