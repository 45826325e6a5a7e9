"""GPU: C-ABI error behaviour (include/subspec.h conventions)."""
import numpy as np
import pytest

from synth.configs import TINY
from synth.prompts import mtbench_prompt

pytestmark = pytest.mark.gpu


def test_status_codes(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec, SubSpecError
    ss = SubSpec(TINY, 256 << 20, max_depth=4, max_top_k=6)
    with pytest.raises(SubSpecError) as e:
        ss.prefill([1, 2, 3])                      # before load/build
    assert e.value.status == 3
    with pytest.raises(SubSpecError) as e:
        ss.build_substitutes(4, 64)
    assert e.value.status == 3
    ss.load_synthetic(0x5EED, 1)
    with pytest.raises(SubSpecError) as e:
        ss.build_substitutes(3, 64)                # only 4-bit g64
    assert e.value.status == 1
    ss.build_substitutes(4, 64)
    with pytest.raises(SubSpecError) as e:
        ss.draft_tree(4, 6, 0.2)                   # no session yet
    assert e.value.status == 3
    with pytest.raises(SubSpecError) as e:
        ss.prefill([TINY.vocab + 5])
    assert e.value.status == 1
    with pytest.raises(SubSpecError) as e:
        ss.prefill(list(range(3000)))              # longer than max_context
    assert e.value.status == 2
    ss.prefill(mtbench_prompt(0x5EED, 0, TINY.vocab, 16))
    with pytest.raises(SubSpecError) as e:
        ss.verify_tree(1)                          # verify before draft
    assert e.value.status == 3
    with pytest.raises(SubSpecError) as e:
        ss.draft_tree(5, 6, 0.2)                   # depth > limits.max_depth
    assert e.value.status == 1
    ss.close()


def test_budget(cuda_required):
    from paper_2509_18344_b200.binding import SubSpec, SubSpecError
    with pytest.raises(SubSpecError) as e:
        SubSpec(TINY, 1 << 20, max_depth=4, max_top_k=6)
    assert e.value.status == 4
