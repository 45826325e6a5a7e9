"""One host copy of the offloaded layers shared by several contexts ("host memory is
shared ... one pinned copy, not G copies"): ss_load_weights_shared with a caller-owned mapping.

Two contexts in one process share an anonymous page-aligned mapping (the multi-process case maps a
POSIX shared-memory segment the same way): the first fills it, the second only attaches.  Both must
decode exactly what a context with its own store decodes (same seed, same target)."""
import ctypes
import mmap

import numpy as np
import pytest

from synth.configs import SMALL
from synth.prompts import mtbench_prompt

pytestmark = pytest.mark.gpu
SEED = 0x5EED


def _ctx():
    from paper_2509_18344_b200.binding import SubSpec
    return SubSpec(SMALL, 512 << 20, max_depth=4, max_top_k=4, max_chunk=256)


def test_two_contexts_share_one_host_store(cuda_required):
    prompt = mtbench_prompt(SEED, 3, SMALL.vocab, 40)
    own = _ctx()
    own.load_synthetic(SEED, n_resident=1)
    own.build_substitutes(4, 64)
    ref, _ = own.generate(prompt, 16, 4, 4, 0.2)
    nbytes = own.host_store_bytes(1)
    own.close()
    assert nbytes > 0

    store = mmap.mmap(-1, nbytes)   # page-aligned anonymous mapping, caller-owned
    addr = ctypes.addressof(ctypes.c_char.from_buffer(store))
    a, b = _ctx(), _ctx()
    a.load_synthetic_shared(SEED, 1, addr, nbytes, fill=True)
    b.load_synthetic_shared(SEED, 1, addr, nbytes, fill=False)   # attaches: nothing generated
    for ss in (a, b):
        ss.build_substitutes(4, 64)
        out, _ = ss.generate(prompt, 16, 4, 4, 0.2)
        assert out == ref
    a.close()
    b.close()
    del addr
    store.close()


def test_shared_store_too_small_is_rejected(cuda_required):
    from paper_2509_18344_b200.binding import SubSpecError
    ss = _ctx()
    nbytes = ss.host_store_bytes(1)
    store = mmap.mmap(-1, 1 << 20)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(store))
    with pytest.raises(SubSpecError):
        ss.load_synthetic_shared(SEED, 1, addr, 1 << 20, fill=True)
    assert nbytes > (1 << 20)
    ss.close()
    del addr
    store.close()
