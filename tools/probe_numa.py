"""Host-link probe: H2D GB/s from 1 GiB slices across a large pinned buffer (NUMA placement of the
pages decides the rate), plus the box's NUMA topology and the GPU's NUMA node."""
import os, subprocess, torch
print(subprocess.run("lscpu | grep -i -E 'numa|socket|model name'; nvidia-smi topo -m; "
                     "cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | "
                     "tr A-Z a-z | sed 's/^0000//;s/^/0000/')/numa_node; cat /proc/meminfo | head -3",
                     shell=True, capture_output=True, text=True).stdout, flush=True)
G = 1 << 30
n = 14 * G
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.view(torch.int64)[:: 512].fill_(1)   # touch pages
d = torch.empty(G, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for off in range(0, 14):
        best = 0
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); d.copy_(h[off * G:(off + 1) * G], non_blocking=True); e1.record(s); e1.synchronize()
            best = max(best, G / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        print(f"slice {off:2d} GiB: {best:.2f} GB/s", flush=True)
    for mb in (32, 128, 272):
        b = mb << 20
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(20):
            d[:b].copy_(h[i * b:(i + 1) * b], non_blocking=True)
        e1.record(s); e1.synchronize()
        print(f"{mb} MiB copies x20: {20 * b / (e0.elapsed_time(e1) * 1e-3) / 1e9:.2f} GB/s", flush=True)
