"""SURVEY §8(f) NEXT-1, cooperative weight streaming (include/subspec.h ss_coop_*), on one GPU: torchrun
starts 2 and 3 ranks that share cuda:0 (CUDA IPC between the processes, as between the GPUs of a node).
Each rank copies 1/G of every streamed group from its host store and pushes it into the peers' rings;
the weights are bit-identical, so every rank's output must equal its non-cooperative output bitwise
(and the oracle's greedy AR output, checked for rank 0), while each rank's host-link bytes fall to 1/G
of a full stream and the rest arrives from the peers."""
import json
import os
import socket
import subprocess
import sys

import pytest

from synth.configs import SMALL
from gpu_util import assert_matches_oracle_ar

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 0x5EED


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_coop_streaming_bit_identical(cuda_required, world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "workers", "coop_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
    assert len(line) == 1, r.stdout[-2000:]
    res = json.loads(line[0][len("RESULT "):])
    assert len(res) == world
    for d in res:
        assert d["coop"] == d["ref"], f"rank {d['rank']}: cooperative output differs"
        assert d["alone_after"] == d["ref"], f"rank {d['rank']}: output after coop_finish differs"
        # host bytes ~ 1/G of the full stream (4 KiB-aligned slices), peers pushed the rest (the two
        # windows differ by up to one pass of prefetch: the cooperative stream restarts at enable)
        assert 0.75 * d["ref_stream_bytes"] <= d["stream_bytes"] * world <= 1.25 * d["ref_stream_bytes"]
        assert d["peer_bytes"] > 0
        assert abs(d["stream_bytes"] * (world - 1) - d["peer_bytes"]) <= 0.02 * d["peer_bytes"] + 4096 * 64
    assert_matches_oracle_ar(SMALL, res[0]["prompt"], res[0]["ref"], SEED)
