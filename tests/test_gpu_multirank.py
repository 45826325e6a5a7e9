"""SURVEY §8(e) readiness on one GPU: bench.py launched by torchrun with two ranks that share cuda:0
(SS_BENCH_DEVICE=0, gloo for the host-side collectives).  Exercises the multi-GPU host path end to end
on real contexts: the node-local rank 0 fills ONE POSIX shared-memory store of the offloaded layers,
rank 1 attaches to it after the barrier (both page-lock their mapping), each rank decodes its own
request with no data-path collective, and rank 0 prints one JSON line whose value is the summed
tokens over the max-over-ranks device time."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(extra_env, world=2, extra_args=()):
    env = dict(os.environ, SS_BENCH_DEVICE="0", SS_DIST_BACKEND="gloo", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(world),
           "--config", "small", "--cap-gib", "1", "--n-resident", "1", "--depth", "4", "--topk", "6",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--prompts", "0", *extra_args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]     # rank 0 alone prints
    return json.loads(lines[0])


def test_two_ranks_share_one_host_store(cuda_required):
    d = _run({})
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["scaling"] == "weak"
    assert d["memory"]["shared_host_store"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["gpu_launches"] > 0


def test_two_ranks_per_rank_store_fallback(cuda_required):
    d = _run({"SS_SHARED_HOST": "0"})
    assert d["n_gpus"] == 2 and d["memory"]["shared_host_store"] is False and d["value"] > 0


def test_two_ranks_cooperative_stream(cuda_required):
    """bench.py --coop (NEXT-1): each rank pulls half of every streamed group over the host link."""
    d = _run({}, extra_args=("--coop",))
    assert d["n_gpus"] == 2 and d["value"] > 0
    s = d["streaming"]
    assert s["mode"].startswith("cooperative") and s["peer_bytes_per_step"] > 0
    assert abs(s["peer_bytes_per_step"] - s["bytes_per_step"]) <= 0.02 * s["bytes_per_step"] + 4096 * 64
