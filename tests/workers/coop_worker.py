"""One rank of the NEXT-1 cooperative-streaming test (launched by torchrun from tests/test_gpu_coop.py;
every rank on cuda:0, gloo for the handle exchange).  Decodes its own request with cooperative
streaming, then the same request again on a fresh non-cooperative context, and prints both."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from synth.configs import SMALL  # noqa: E402
from synth.prompts import mtbench_prompt  # noqa: E402
from paper_2509_18344_b200.binding import SubSpec  # noqa: E402

SEED = 0x5EED
D, K, T, STEPS = 4, 6, 0.2, 6
CAP = int(os.environ.get("COOP_CAP", str(112 << 20)))   # ring ~39 MB ~ 1.2 coded passes: it wraps every pass


def decode(ss, prompt, rank, world, coop):
    first = ss.prefill(prompt)
    if coop:
        h = ss.coop_export()
        hs = [None] * world
        dist.all_gather_object(hs, h)
        ss.coop_enable(rank, hs)
        dist.barrier()
    ss.reset_stats()
    out = [first]
    for _ in range(STEPS):
        out += ss.step(D, K, T)
    st = ss.stats()
    if coop:
        ss.coop_finish()
        dist.barrier()
    return out, st


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    prompt = [int(t) for t in mtbench_prompt(SEED, rank, SMALL.vocab, 40 + 8 * rank)]
    ss = SubSpec(SMALL, CAP, max_depth=D, max_top_k=K)
    ss.load_synthetic(SEED, n_resident=1)
    ss.build_substitutes(4, 64)
    coop, st = decode(ss, prompt, rank, world, True)
    # the same context continues alone after coop_finish: one more request must still be exact
    alone, _ = decode(ss, prompt, rank, world, False)
    ss.close()
    ref_ss = SubSpec(SMALL, CAP, max_depth=D, max_top_k=K)
    ref_ss.load_synthetic(SEED, n_resident=1)
    ref_ss.build_substitutes(4, 64)
    ref, st_ref = decode(ref_ss, prompt, rank, world, False)
    ref_ss.close()
    res = {"rank": rank, "prompt": prompt, "coop": coop, "alone_after": alone, "ref": ref,
           "stream_bytes": st["stream_bytes"], "peer_bytes": st["peer_bytes"], "ref_stream_bytes": st_ref["stream_bytes"],
           "ring_bytes": st["ring_bytes"]}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print("RESULT " + json.dumps(allres), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
