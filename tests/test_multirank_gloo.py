"""CPU, world_size 2 (gloo): the multi-GPU host logic of bench.py — requests partitioned over ranks
with no data-path collective, whole-job time = max over ranks, tokens = sum over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from synth.configs import QWEN7B
    ms, tok = bench.aggregate_ranks(dist, 100.0 * (rank + 1), 7 * (rank + 1))
    prompt = bench.request_for_rank(rank, QWEN7B.vocab)
    class FakeCtx:   # records the cooperative-streaming handshake (NEXT-1) without a GPU
        def coop_export(self):
            return bytes([rank]) * 256

        def coop_enable(self, r, handles):
            self.enabled = (r, handles)
    fc = FakeCtx()
    bench.coop_handshake(fc, dist, rank, world)
    q.put((rank, ms, tok, prompt.tolist(), fc.enabled[0], [h[0] for h in fc.enabled[1]]))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_and_aggregate():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == 200.0 and r[2] == 21.0 for r in res)      # max time, summed tokens
    assert res[0][3] != res[1][3]                                # distinct requests per rank
    for r in res:                                                # coop: own rank, every handle in rank order
        assert r[4] == r[0] and r[5] == list(range(world))
