"""Streaming pipeline ordering (A4 / K7): events around every streamed layer group of
one step (ss_debug_step_timeline) must show the causal order the event graph enforces — a group's
compute starts only after its copy has landed, its ring region is released after its compute starts,
the verify consumes the groups in layer order, and the copies of later groups overlap the compute of
earlier ones (the async transfer) — on a small model with streamed layers, plain and codec-coded."""
import numpy as np
import pytest

from synth.configs import SMALL
from synth.prompts import mtbench_prompt

pytestmark = pytest.mark.gpu
SEED = 0x5EED


@pytest.mark.parametrize("compress", [1, 0], ids=["codec", "plain"])
def test_step_timeline_causal(cuda_required, compress):
    from paper_2509_18344_b200.binding import SubSpec
    D, k = 4, 6
    ss = SubSpec(SMALL, 512 << 20, max_depth=D, max_top_k=k, compress_stream=compress)
    ss.load_synthetic(SEED, n_resident=1)
    ss.build_substitutes(4, 64)
    ss.prefill(mtbench_prompt(SEED, 3, SMALL.vocab, 48))
    ss.step(D, k, 0.2)
    rows, ph = ss.debug_step_timeline(D, k, 0.2)
    n_off = SMALL.n_layers - 1
    assert 0 < ph[0] < ph[1] <= ph[2]                         # draft end < verify end <= accept end
    cons = rows[(rows[:, 6] > -1e8) & (rows[:, 7] > -1e8)]
    assert len(cons) == 4 * n_off                              # every streamed group, once
    assert np.all(np.diff(cons[:, 0]) == 1)                    # consumed in stream order
    assert [(int(r[1]), int(r[2])) for r in cons] == [(l, g) for l in range(1, SMALL.n_layers) for g in range(4)]
    copied = cons[cons[:, 5] > -1e8]
    eps = 5e-3                                                 # event timestamp resolution (ms)
    assert np.all(copied[:, 5] >= copied[:, 4] - eps)          # copy end >= copy start
    assert np.all(copied[:, 6] >= copied[:, 5] - eps)          # compute waits for its copy
    assert np.all(cons[:, 7] >= cons[:, 6] - eps)              # ring released after compute started
    assert np.all(cons[:, 6] >= ph[0] - eps)                   # verify groups run after the draft
    assert np.all(cons[:, 7] <= ph[1] + eps)
    ss.close()
