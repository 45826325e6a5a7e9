"""Host/box probe: cores, RAM, GPU, pinned H2D/D2H bandwidth (cudaMemcpyAsync from pinned memory)."""
import json, os, subprocess, time
import torch

def main():
    out = {"cpu_count": os.cpu_count()}
    try:
        out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        pass
    out["mem_total_gb"] = int(open("/proc/meminfo").readline().split()[1]) / 2**20
    out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max", "--format=csv"], capture_output=True, text=True).stdout
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        ts = []
        with torch.cuda.stream(s):
            for i in range(10):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s); fn(); e1.record(s); e1.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
        best[name + "_gbs"] = n / min(ts) / 1e9
    out.update(best)
    print(json.dumps(out, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/probe_host.json", "w"), indent=1)

if __name__ == "__main__":
    main()
