"""Summaries of the round's ncu evidence -> profiles/ (launch-list shares, K2 full-capture metrics)."""
import collections, csv, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)
out = []

# ---- launch list (gpu__time_duration per launch, cold/serialised: compare shares) ----
rows = list(csv.reader(open(os.path.join(src, f"launches_{tag}.csv"))))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    v = float(r[vi].replace(",", ""))
    us = v / 1e3 if r[ui] in ("ns", "nsecond") else (v if r[ui] in ("us", "usecond") else v * 1e3)
    name = re.sub(r"\(.*", "", r[ki]).replace("void ss::", "").replace("ss::", "")
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
out.append(f"# ncu launch list of bench.py's timed region (SS_PROFILE_TIMED=1, --profile-from-start off; {len(data)} launches captured, tag {tag})\n")
out.append("Per-launch `gpu__time_duration.sum` under ncu (serialised, cold caches): compare SHARES, not absolutes.\n")
out.append("| kernel | launches | total us | avg us | share |\n|---|---:|---:|---:|---:|")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {v[1] / tot:.3f} |")
out.append("")

# ---- full captures of the K2 dequant-GEMV ----
def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(r)))
    return rr[0], rr[1], rr[2]

want = ["Kernel Name", "Grid Size", "Block Size", "launch__cluster_dim_x", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
traffic = {}
for name, rep in (("gate_up (N=37888, K=3584, M=6)", f"k2_gate_up_{tag}.ncu-rep"), ("qkv (N=4608, K=3584, M=6)", f"k2_qkv_{tag}.ncu-rep"),
                  ("down (N=3584, K=18944, M=6)", f"k2_down_{tag}.ncu-rep"),
                  ("2-bit gate_up (N=37888, K=3584, M=6; NEXT-3)", f"k2q2_gate_up_{tag}.ncu-rep"),
                  ("tcgen05 bf16 head (N=152064, K=3584, M=6)", f"head_{tag}.ncu-rep"),
                  ("K3 tree attention in a draft pass (M=6 nodes, 4 kv heads)", f"attn_{tag}.ncu-rep"),
                  ("K6 tcgen05 verify GEMM gate_up (N=37888, K=3584, M=289)", f"k6_gate_up_{tag}.ncu-rep"),
                  ("K6 tcgen05 verify head + argmax (N=152064, K=3584, M=289)", f"k6_head_{tag}.ncu-rep")):
    path = os.path.join(src, rep)
    if not os.path.exists(path):
        continue
    hdr, units, r = raw(path)
    out.append(f"## ncu --set full: {name}\n")
    out.append("| metric | value | unit |\n|---|---|---|")
    for w in want:
        if w in hdr:
            out.append(f"| `{w}` | {r[hdr.index(w)]} | {units[hdr.index(w)]} |")
    stalls = []
    for i, hh in enumerate(hdr):
        if hh.startswith("smsp__pcsamp_warps_issue_stalled_") and not hh.endswith("not_issued"):
            try:
                stalls.append((int(r[i]), hh.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    out.append("\nTop warp-stall samples: " + ", ".join(f"{n} {s}" for s, n in [(s, n) for n, s in stalls[:6]]) + "\n")
    # SASS lines with the most stall samples (source page)
    src_csv = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src_csv)))
    hi = next((i for i, rr in enumerate(srows) if "Address" in rr and "Source" in rr), None)
    if hi is not None:
        sh = srows[hi]
        ia, isr = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)")

        def fnum(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        body = srows[hi + 1:]
        tot_s = sum(fnum(rr[isr]) for rr in body if len(rr) > isr)
        top = sorted((rr for rr in body if len(rr) > isr), key=lambda rr: -fnum(rr[isr]))[:5]
        out.append(f"Top SASS lines by stall samples (of {tot_s:.0f}): " +
                   "; ".join(f"`{rr[ia].strip()[:48]}` {fnum(rr[isr]):.0f}" for rr in top) + "\n")
    rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
    wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic[name] = rd * mult.get(units[hdr.index("dram__bytes_read.sum")], 1) + wr * mult.get(units[hdr.index("dram__bytes_write.sum")], 1)
open(os.path.join(dst, f"ncu_summary_{tag}.md"), "w").write("\n".join(out) + "\n")
if traffic:
    json.dump({"traffic_bytes_per_launch": traffic.get("gate_up (N=37888, K=3584, M=6)"),
               "per_kernel_traffic_bytes": traffic,
               "algorithmic_bytes": {"gate_up": 37888 * 3584 // 2 + 37888 * 3584 // 64 * 4 + 6 * 3584 * 2 + 6 * 37888 * 2,
                                     "qkv": 4608 * 3584 // 2 + 4608 * 3584 // 64 * 4 + 6 * 3584 * 2 + 6 * 4608 * 2,
                                     "down": 3584 * 18944 // 2 + 3584 * 18944 // 64 * 4 + 6 * 18944 * 2 + 6 * 3584 * 2,
                                     "2-bit gate_up": 37888 * 3584 // 4 + 37888 * 3584 // 64 * 4 + 6 * 3584 * 2 + 6 * 37888 * 2,
                                     "head": 152064 * 3584 * 2 + 6 * 3584 * 2},
               "source": f"gpurun_out/{{k2_*,head}}_{tag}.ncu-rep (ncu --set full)"},
              open(os.path.join(dst, "k2_traffic.json"), "w"), indent=1)
print("\n".join(out))
