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
