"""Host->device bandwidth with 1, 2 and 4 concurrent copy streams (pinned source), and chunk sizes."""
import torch, time
n = 1 << 30
dev = torch.device("cuda")
src = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
dst = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
def run(k, chunk):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    best = 0
    for rep in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                for off in range(0, n, chunk):
                    dst[i][off:off + chunk].copy_(src[i][off:off + chunk], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        gbs = k * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
        best = max(best, gbs)
    return best
for k in (1, 2, 4):
    for chunk in (n, 64 << 20, 8 << 20):
        print(f"streams {k} chunk {chunk >> 20} MiB: {run(k, chunk):.2f} GB/s", flush=True)
