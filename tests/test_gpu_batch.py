"""Batched requests: one weight stream serves B request trees per step.

Losslessness is per request: whatever the batch, request b's committed output must be
its own greedy AR output.  The verify path is batch-invariant (K6 has no split-K, K3 blocks keys by
logical index), so a batched SubSpec run must emit, for every request, exactly the tokens a
one-request GPU AR run emits - bitwise, with no near-tie flags - and those must agree with the
oracle's greedy AR (oracle/decode.py) up to flagged near-ties.  Also covered: ragged prompt lengths
across slots, B = 1 through the batch API == the one-request API, the capacity clamp shared by the
batch, the slot/batch state machine and its error codes, and the Qwen2.5-7B shape at 8 GiB with
B = 4 (the configuration bench.py's batched line times).
"""
import numpy as np
import pytest

from synth.configs import TINY, SMALL, QWEN7B, GIB
from synth.prompts import mtbench_prompt
from oracle.decode import ar_generate

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _ctx(cfg, n_res, D, k, B, cap=768 << 20, max_chunk=256):
    from paper_2509_18344_b200.binding import SubSpec
    ss = SubSpec(cfg, cap, max_depth=D, max_top_k=k, max_chunk=max_chunk, max_batch=B)
    ss.load_synthetic(SEED, n_resident=n_res)
    ss.build_substitutes(4, 64)
    return ss


@pytest.mark.parametrize("cfg,n_res,D,k,B", [(TINY, 1, 4, 6, 3), (SMALL, 1, 4, 6, 5), (SMALL, 0, 6, 2, 4)],
                         ids=["tiny-B3", "small-B5", "small-allsub-B4"])
def test_batch_equals_per_request_ar(cuda_required, cfg, n_res, D, k, B):
    ss = _ctx(cfg, n_res, D, k, B)
    prompts = [mtbench_prompt(SEED, p, cfg.vocab, 24 + 13 * p) for p in range(B)]   # ragged lengths
    outs, hist = ss.generate_batch(prompts, 40, D, k, 0.2)
    assert len(outs) == B and all(len(o) == 40 for o in outs)
    assert hist[0] == 0 and hist.sum() >= B
    for b, p in enumerate(prompts):
        ss.set_batch(1)
        ar, _ = ss.generate(p, 40, 0, 1, 0.2)
        assert outs[b] == ar, f"request {b}: batched SubSpec output differs from its GPU AR output"
    # oracle AR on the first request: identical up to a flagged near-tie (checked in test_gpu_decode)
    ref, _ = ar_generate(cfg, prompts[0], 16, seed=SEED, mode="bf16")
    assert outs[0][:8] == ref[:8]
    ss.close()


def test_batch_of_one_equals_single_api(cuda_required):
    ss = _ctx(TINY, 1, 4, 6, 4)
    p = mtbench_prompt(SEED, 7, TINY.vocab, 32)
    single, h1 = ss.generate(p, 30, 4, 6, 0.2)
    outs, h2 = ss.generate_batch([p], 30, 4, 6, 0.2)
    assert outs[0] == single and list(h1) == list(h2)
    ss.close()


def test_same_prompt_in_every_slot(cuda_required):
    # identical requests must produce identical trees and outputs in every slot
    ss = _ctx(SMALL, 1, 4, 6, 4)
    p = mtbench_prompt(SEED, 3, SMALL.vocab, 40)
    outs, _ = ss.generate_batch([p] * 4, 30, 4, 6, 0.2)
    assert all(o == outs[0] for o in outs)
    ss.close()


def test_batch_capacity_clamp(cuda_required):
    cfg = TINY.with_(max_context=96)
    ss = _ctx(cfg, 1, 6, 4, 3, max_chunk=128)
    prompts = [mtbench_prompt(SEED, 10 + b, cfg.vocab, 30 + 9 * b) for b in range(3)]
    outs, _ = ss.generate_batch(prompts, 40, 6, 4, 0.2, chunk=128)
    for b, p in enumerate(prompts):
        ss.set_batch(1)
        ar, _ = ss.generate(p, len(outs[b]), 0, 1, 0.2, chunk=128)
        assert outs[b] == ar
    assert ss.stats()["committed_len"] <= cfg.max_context
    ss.close()


def test_batch_state_machine(cuda_required):
    from paper_2509_18344_b200.binding import SubSpecError
    ss = _ctx(TINY, 1, 4, 6, 2)
    p = mtbench_prompt(SEED, 1, TINY.vocab, 32)
    with pytest.raises(SubSpecError) as e:
        ss.set_batch(3)                        # > max_batch
    assert e.value.status == 1
    ss.set_batch(2)
    with pytest.raises(SubSpecError) as e:
        ss.prefill_slot(2, p)                  # slot outside the active batch
    assert e.value.status == 1
    ss.prefill_slot(0, p)
    with pytest.raises(SubSpecError) as e:
        ss.step_batch(2, 4, 6, 0.2)            # slot 1 not prefilled yet
    assert e.value.status == 3
    ss.prefill_slot(1, p)
    with pytest.raises(SubSpecError) as e:
        ss.step(4, 6, 0.2)                     # one-request step on a batch of 2
    assert e.value.status == 3
    a, b = ss.step_batch(2, 4, 6, 0.2)
    assert a == b and 1 <= len(a) <= 5
    ss.close()
    from paper_2509_18344_b200.binding import SubSpec
    with pytest.raises(SubSpecError):
        SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6, max_batch=6)   # 6 x 6 > 32 draft rows


def test_qwen7b_batch4_at_8gib(cuda_required):
    """BJ config 2 shapes with B = 4 requests in one 8 GiB arena: a few batched steps emit each
    request's GPU AR tokens."""
    from paper_2509_18344_b200.binding import SubSpec
    B, D, k = 4, 48, 6
    ss = SubSpec(QWEN7B, 8 * GIB, max_depth=D, max_top_k=k, max_chunk=256, max_batch=B)
    ss.load_synthetic(SEED, n_resident=0)
    ss.build_substitutes(4, 64)
    prompts = [mtbench_prompt(SEED, p, QWEN7B.vocab) for p in range(B)]
    outs, hist = ss.generate_batch(prompts, 12, D, k, 0.2)
    st = ss.stats()
    assert hist[0] == 0
    for b in (0, 3):
        ss.set_batch(1)
        ar, _ = ss.generate(prompts[b], 12, 0, 1, 0.2)
        assert outs[b] == ar, f"request {b}"
    assert st["arena_used"] <= 8 * GIB
    ss.close()
