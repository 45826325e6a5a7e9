"""NEXT-4: Table-2-style ablation ladder and App. F depth point on synthetic weights.

Runs bench.py variants in fresh processes and writes
profiles/ablation_<tag>.json.  Variants: full SubSpec; async transfer off (--no-async, ss_options.async_stream = 0: each
streamed group is copied only after the previous group's compute); sharpening off
(T = 1); a shallower tree (D = 24); and the offloading AR baseline through the same engine
(D = 0, the paper's "None" row) for the speedup; the draft without the shared KV-cache
(--separate-draft-kv, Table 2's row before "+ shared KV"); and the draft temperature
sweep of Table 5 (T = 0.2 .. 1.2).  On random weights tau is not the paper's: the
ladder measures what each switch costs or saves in step time on B200.
"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
steps = ["--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-ar", "--prompts", "0"]
variants = [
    ("full (D=48, k=6, T=0.2, async)", {}, []),
    ("async transfer off", {}, ["--no-async"]),
    ("sharpening off (T=1)", {}, ["--temp", "1.0"]),
    ("shallower tree (D=24)", {}, ["--depth", "24"]),
    ("separate draft KV (no '+ shared KV')", {}, ["--separate-draft-kv"]),
    *[(f"draft temperature T={t}", {}, ["--temp", str(t)]) for t in (0.4, 0.6, 0.8, 1.2)],
    # 16 timed steps: the ring prefetched before the timed region is not hidden under a draft here
    ("offloading AR baseline (D=0)", {}, ["--depth", "0", "--topk", "1", "--steps", "16"]),
]
out = []
for name, env, extra in variants:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *steps, *extra], env=e, capture_output=True,
                       text=True, timeout=1200)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if not line:
        out.append({"variant": name, "error": r.stderr[-500:]})
        print(name, "FAILED", r.stderr[-300:], flush=True)
        continue
    d = json.loads(line[-1])
    rec = {"variant": name, "env": env, "args": extra, "tokens_per_s": d["value"], "ms_per_step": d["ms_per_step"],
           "tau_mean": d.get("tau_mean"), "step_breakdown_ms": d.get("step_breakdown_ms"),
           "stream_duty_cycle": (d.get("streaming") or {}).get("duty_cycle"), "clocks": d.get("clocks")}
    out.append(rec)
    print(json.dumps(rec), flush=True)
base = next((o for o in out if o["variant"].startswith("offloading AR") and "tokens_per_s" in o), None)
if base:
    for o in out:
        if "tokens_per_s" in o:
            o["speedup_vs_offloading_AR"] = o["tokens_per_s"] / base["tokens_per_s"]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"ablation_{tag}.json"), "w"), indent=1)
