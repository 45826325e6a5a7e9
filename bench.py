#!/usr/bin/env python
"""bench.py — SubSpec tree-speculative decode on B200 (BASELINE.json metric: decode tokens/s and mean
acceptance length at the VRAM cap; dequant-GEMM HBM GB/s).

A "step" is one SubSpec decode step = D draft passes + one verification pass + acceptance/commit
(Eq. 2, :86) on one synthetic MT-Bench-shaped request.  Default workload:
BASELINE.json config 2 — Qwen2.5-7B shape, random-init bf16 target, 8 GiB emulated VRAM cap, all 28
decoder layers offloaded with 4-bit/g64 substitutes, D = 48, k = 6, T = 0.2.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config qwen2.5-7b]

Under torchrun each rank runs its own independent request on its own GPU (weak scaling, no
data-path collective; torch.distributed only for the barrier and the max/sum of the timings).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth.configs import PRESETS, GIB  # noqa: E402
from synth.prompts import mtbench_prompt  # noqa: E402

SEED = 0x5EED


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen2.5-7b", choices=sorted(PRESETS))
    ap.add_argument("--cap-gib", type=float, default=8.0)
    ap.add_argument("--n-resident", type=int, default=0, help="0 = paper-faithful; -1 = planner max")
    ap.add_argument("--depth", type=int, default=48)
    ap.add_argument("--topk", type=int, default=6)
    ap.add_argument("--temp", type=float, default=0.2)
    ap.add_argument("--batch", type=int, default=1,
                    help="request slots per GPU sharing one weight stream (SURVEY 8(f) NEXT-2); 1 = the paper's batch 1")
    ap.add_argument("--sub-bits", type=int, default=4, choices=[4, 3, 2],
                    help="substitute code bits (4 = the paper's setting, P:278; 2 = NEXT-3, P:343)")
    ap.add_argument("--quant", default="rtn", choices=["rtn", "hqq"],
                    help="substitute quantizer: min/max RTN or HQQ's half-quadratic zero (NEXT-3, R28)")
    ap.add_argument("--embed-gpu", action="store_true",
                    help="embedding GPU-resident in the arena (PAPER.md:534) instead of mapped host memory (R24)")
    ap.add_argument("--no-async", action="store_true",
                    help="Table-2 ablation: no copy/compute overlap in the verify streaming (PAPER.md:305-308)")
    ap.add_argument("--prompts", type=int, default=4, help="prompt sweep: MT-Bench-shaped prompts (0 = skip)")
    ap.add_argument("--repeats", type=int, default=1, help="prompt sweep: repeats of each prompt")
    ap.add_argument("--no-compress", action="store_true",
                    help="stream plain bf16 layers (ss_options.compress_stream = 0) instead of the lossless codec")
    ap.add_argument("--separate-draft-kv", action="store_true",
                    help="NEXT-4 ablation: the draft keeps its own KV-cache (Table 2 without '+ shared KV')")
    ap.add_argument("--coop", action="store_true",
                    help="NEXT-1 cooperative weight streaming under torchrun: rank r pulls 1/N of every streamed "
                         "group over its host link and pushes it to the peers over NVLink (ss_coop_*)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ar", action="store_true", help="skip the offloading AR baseline line (SURVEY §8(d))")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------------------------
class OracleSample:
    """Bounded sample of the oracle (oracle/, fp32-BLAS mode) on the SAME workload: real SubSpec steps
    (D draft passes of the frontier, sharpened top-k, one verify of all 1 + kD nodes, greedy accept,
    KV commit) on a 1/L slice of the full-size model — ONE of its L decoder layers (full width) and the
    first V/L rows of its head (so the head GEMMs and the top-k over the vocabulary are 1/L of a step's
    too).  Every per-layer and per-vocabulary cost of a step is L x the slice's, so the step time is
    L x the measured sample step; tau is the slice model's own acceptance (measured, not borrowed)."""

    def __init__(self, cfg, depth, topk, temp, bits=4, quant="rtn"):
        from oracle.decode import Session
        self.L = cfg.n_layers
        self.vs = max(128, (cfg.vocab // self.L) // 128 * 128)
        self.cfg1 = cfg.with_(name=cfg.name + "-slice", n_layers=1, vocab=self.vs)
        self.depth, self.topk, self.temp, self.bits = depth, topk, temp, bits
        t0 = time.time()
        self.sess = Session(self.cfg1, SEED, n_resident=0, bits=bits, mode="bf16-fp32", max_nodes=max(1 + topk * depth, 256),
                            quant=quant)
        self.prompt = [int(t) % self.vs for t in mtbench_prompt(SEED, 0, cfg.vocab)]
        self.root = self.sess.prefill(self.prompt)
        self.setup = time.time() - t0

    def step_seconds(self):
        """One real SubSpec step of the slice model -> (seconds for the full-size step, emitted tokens)."""
        if self.sess.kv.P + 1 + self.topk * self.depth >= self.cfg1.max_context:   # start over when full
            self.sess.kv.P = 0
            self.root = self.sess.prefill(self.prompt)
        t0 = time.perf_counter()
        tree, path, emitted = self.sess.step(self.root, self.depth, self.topk, self.temp)
        dt = time.perf_counter() - t0
        self.root = emitted[-1]
        return dt * self.L, len(emitted)

    def describe(self):
        return (f"real SubSpec steps (D={self.depth}, k={self.topk}, T={self.temp}) of a 1/{self.L} slice of the "
                f"{self.cfg1.name[:-6]} model: 1 of {self.L} decoder layers at full width ({self.bits}-bit substitute) "
                f"+ the first {self.vs} head rows, fp32-BLAS NumPy oracle; step time = {self.L} x the slice's step "
                f"time; tau = the slice model's own acceptance (a 1-layer draft agrees with its target more often "
                f"than the {self.L}-layer one: compare steps_per_s)")


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = PRESETS[a.config]
    sample = OracleSample(cfg, a.depth, a.topk, a.temp, bits=a.sub_bits, quant=a.quant)
    times, toks = [], []
    for i in range(a.warmup + a.steps):
        s, n = sample.step_seconds()
        if i >= a.warmup:
            times.append(s)
            toks.append(n)
    step_s = statistics.mean(times)
    tau = float(np.mean(toks))
    value = sum(toks) / sum(times)
    cores = blas_threads()
    line = {"metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded random-init weights, MT-Bench-shaped prompt)",
            "config": workload_config(a, cfg), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": sample.describe()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "tau_mean": tau, "steps_per_s": 1.0 / step_s,
            "oracle_timing": {"setup_s": sample.setup, "sample_seconds_per_step": step_s / sample.L,
                              "scale": sample.L, "wall_seconds_in_run": sum(times) / sample.L}}
    print(json.dumps(line), flush=True)


def ngram_repetition(tokens, n=4):
    """Fraction of the sequence's n-grams that occurred earlier in it (a greedy-loop detector)."""
    seen, rep = set(), 0
    grams = [tuple(tokens[i:i + n]) for i in range(len(tokens) - n + 1)]
    for g in grams:
        rep += g in seen
        seen.add(g)
    return rep / max(1, len(grams))


def workload_config(a, cfg):
    batch = "" if a.batch == 1 else f", {a.batch} requests per GPU sharing one weight stream (NEXT-2)"
    return {"workload": f"{cfg.name} SubSpec step, {a.cap_gib:g} GiB cap, n_resident={a.n_resident}, "
                        f"{a.sub_bits}-bit g64 {a.quant.upper()} substitutes, D={a.depth} k={a.topk} T={a.temp}, MT-Bench-shaped prompt{batch}",
            "model_shape": cfg.name, "vram_cap_gib": a.cap_gib, "n_resident": a.n_resident, "depth": a.depth,
            "top_k": a.topk, "sharpen_t": a.temp, "batch": a.batch, "max_context": cfg.max_context,
            "l2": "inputs larger than L2 (>= 4.76 GB of draft weights per draft pass; 13 GB streamed per verify)",
            "parallelism": (f"requests partitioned, {a.gpus} GPU(s); layer stream shared (NEXT-1: 1/{a.gpus} per host "
                            f"link + NVLink peer copies)" if a.coop and a.gpus > 1 else
                            f"requests partitioned, {a.gpus} GPU(s), no collective")}


def aggregate_ranks(dist, ms, tokens, device="cpu"):
    """Whole-job timing across ranks: max of the per-rank device times, sum of the tokens."""
    if dist is None:
        return ms, tokens
    import torch
    t = torch.tensor([float(ms)], device=device, dtype=torch.float64)
    n = torch.tensor([float(tokens)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n)
    return float(t), float(n)


def request_for_rank(rank, vocab):
    """Requests are partitioned over ranks (BJ config 5): rank r decodes prompt r."""
    return mtbench_prompt(SEED, rank, vocab)


def k2_bytes(N, K, M, bits=4):
    # codes N*K*bits/8 + meta N*K/64*4 + X M*K*2 + Y M*N*2
    return N * K * bits // 8 + N * K // 64 * 4 + M * K * 2 + M * N * 2


def load_weights_for_job(ss, dist, local, n_resident):
    """the node holds ONE copy of the offloaded layers.  Under torchrun the node-local
    rank 0 creates a POSIX shared-memory segment and fills it; the other ranks attach after a
    barrier (each process page-locks its mapping).  Falls back to a per-rank store when /dev/shm is
    too small or SS_SHARED_HOST=0.  Returns the SharedMemory handle (kept alive) or None."""
    if dist is None or n_resident < 0 or os.environ.get("SS_SHARED_HOST", "1") == "0":
        ss.load_synthetic(SEED, n_resident=n_resident)
        return None
    import torch
    from multiprocessing import shared_memory
    nbytes = ss.host_store_bytes(n_resident)
    name = f"ss_store_{os.environ.get('MASTER_PORT', '0')}"
    ok = 1
    shm = None
    if local == 0:
        try:
            st = os.statvfs("/dev/shm")
            if st.f_bavail * st.f_frsize < nbytes + (1 << 30):
                raise OSError("/dev/shm too small")
            shm = shared_memory.SharedMemory(name=name, create=True, size=nbytes)
        except Exception:
            ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=dist_device(local))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag) == 0:
        if shm is not None:
            shm.close()
            shm.unlink()
        ss.load_synthetic(SEED, n_resident=n_resident)
        return None
    import ctypes
    if local == 0:
        addr = ctypes.addressof(ctypes.c_char.from_buffer(shm.buf))
        ss.load_synthetic_shared(SEED, n_resident, addr, nbytes, fill=True)
    dist.barrier()
    if local != 0:
        shm = shared_memory.SharedMemory(name=name)
        try:   # attaching processes must not unlink the segment at exit (the creator does)
            from multiprocessing import resource_tracker
            resource_tracker.unregister(shm._name, "shared_memory")
        except Exception:
            pass
        addr = ctypes.addressof(ctypes.c_char.from_buffer(shm.buf))
        ss.load_synthetic_shared(SEED, n_resident, addr, nbytes, fill=False)
    return shm


def coop_handshake(ss, dist, rank, world):
    """NEXT-1 (include/subspec.h ss_coop_*): every rank exports its 256-byte handle, the handles are
    all-gathered in rank order, every rank enables cooperative streaming with them, then a barrier (no
    rank may stream into a peer's ring before that peer has drained and reset its own)."""
    handles = [None] * world
    dist.all_gather_object(handles, ss.coop_export())
    ss.coop_enable(rank, handles)
    dist.barrier()
    return handles


def dist_device(local):
    return "cpu" if os.environ.get("SS_DIST_BACKEND", "nccl") == "gloo" else f"cuda:{local}"


def run_ours(a):
    import torch
    rank, world, local = dist_env()
    dev = int(os.environ.get("SS_BENCH_DEVICE", local))   # test override: several ranks on one GPU (gloo)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("SS_DIST_BACKEND", "nccl") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2509_18344_b200.binding import SubSpec
    cfg = PRESETS[a.config]
    D, k, T = a.depth, a.topk, a.temp
    t_setup = time.time()
    Bq = a.batch
    ss = SubSpec(cfg, int(a.cap_gib * GIB), device=dev, max_depth=D, max_top_k=max(k, 6), max_chunk=256,
                 max_batch=Bq, embed_on_host=0 if a.embed_gpu else 1, async_stream=0 if a.no_async else 1,
                 separate_draft_kv=1 if a.separate_draft_kv else 0, compress_stream=0 if a.no_compress else 1)
    if a.sub_bits != 4:
        ss.set_substitute_bits(a.sub_bits)
    shm = load_weights_for_job(ss, dist, local, a.n_resident)
    ss.build_substitutes(a.sub_bits, 64, method=a.quant)
    if Bq == 1:
        ss.prefill(request_for_rank(rank, cfg.vocab))
        step = lambda: [ss.step(D, k, T)]                     # noqa: E731
    else:   # rank r decodes requests r*B .. r*B + B - 1, all B in one step
        ss.set_batch(Bq)
        for b in range(Bq):
            ss.prefill_slot(b, request_for_rank(rank * Bq + b, cfg.vocab))
        step = lambda: ss.step_batch(Bq, D, k, T)            # noqa: E731
    coop = bool(a.coop and dist is not None)
    if coop:   # every rank has prefilled (one target pass each); from here on the ranks verify in lockstep
        coop_handshake(ss, dist, rank, world)
    t_setup = time.time() - t_setup
    prompt0 = request_for_rank(rank, cfg.vocab)

    def timed_window(step_fn, n_steps):
        """Device time of n_steps steps (CUDA events on the compute stream, barrier + sync on both sides;
        the region ends when the copy stream has prefetched the ring again: steady state)."""
        cs = ss.compute_stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(cs)
        out = [step_fn() for _ in range(n_steps)]
        ring_full = torch.cuda.Event()
        ring_full.record(ss.copy_stream)
        cs.wait_event(ring_full)
        e1.record(cs)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return e0.elapsed_time(e1), out

    for _ in range(a.warmup):
        step()
    ss.reset_stats()
    clocks = ClockSampler(dev)
    clocks.start()
    prof = os.environ.get("SS_PROFILE_TIMED") == "1"   # ncu --profile-from-start off: the timed steps only
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    ms, outs = timed_window(step, a.steps)
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    ck = clocks.stop()
    st = ss.stats()
    emitted_seq = [t for o in outs for r in o for t in r]
    taus = [len(r) for o in outs for r in o]
    emitted = sum(taus)
    # ---- dominant kernel: K2 dequant-GEMV, live sweep over every layer (weights from HBM) ----
    M = k * Bq   # frontier rows of a draft pass (all requests)
    groups = [ss.group_shape(g) for g in range(4)]
    per_group = {}
    for g, name in enumerate(("qkv", "o", "gate_up", "down")):
        t = ss.debug_time_matmul(-1, g, M, iters=3)
        per_group[name] = {"N": groups[g][0], "K": groups[g][1], "us": t * 1e3,
                           "gbs": k2_bytes(*groups[g], M, a.sub_bits) / (t * 1e-3) / 1e9}
    t_sweep = ss.debug_time_matmul(-1, -2, M, iters=3)       # avg per launch, 4 groups x L layers
    bytes_layer = sum(k2_bytes(N, K, M, a.sub_bits) for N, K in groups)
    k2_gbs = bytes_layer / (4 * t_sweep * 1e-3) / 1e9
    t_head = ss.debug_time_matmul(0, -1, M, iters=5)
    head_gbs = (cfg.vocab * cfg.hidden * 2 + M * cfg.hidden * 2 + M * cfg.vocab * 4) / (t_head * 1e-3) / 1e9
    # K2 inside a real draft pass: per-launch (first CTA entry .. last CTA end) from %globaltimer traces
    k2_in_pass = None
    if Bq == 1 and st["n_offloaded"] == cfg.n_layers:
        tr = ss.debug_trace_pass(M, cap=512)
        gemv = [r for r in tr if r[6] > r[2] > 0]
        if len(gemv) >= 4 * cfg.n_layers:
            dur = [(int(r[6]) - int(r[2])) * 1e-9 for r in gemv[:4 * cfg.n_layers]]
            k2_in_pass = {"gbs": cfg.n_layers * bytes_layer / sum(dur) / 1e9,
                          "us_per_layer": sum(dur) / cfg.n_layers * 1e6,
                          "note": "per K2 launch inside one draft pass: from the release of its dependency on the "
                                  "previous kernel (griddepcontrol.wait returns) to its last CTA's end; the weight "
                                  "prefetch issued before that release is not counted against it"}
    # ---- e2e through the C-ABI with host buffers, replaying the SAME steps: re-prefill the same prompt,
    # the same warm-up, then the same K steps (deterministic: identical tokens); each step copies the root
    # token H2D and reads the emitted tokens D2H; the 13 GB of streamed layer weights per step are
    # host->device copies inside the region too ----
    e2e = None
    if not a.no_e2e and Bq == 1:
        root = ss.prefill(prompt0)
        for _ in range(a.warmup):
            ss.draft_tree(D, k, T, root_token=root, want_tree=False)
            ss.verify_tree(want=False)
            root = ss.accept_and_commit(D + 1)[0][-1]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = ss.stats()
        t0 = time.perf_counter()
        e2e_seq = []
        for _ in range(a.steps):
            ss.draft_tree(D, k, T, root_token=root, want_tree=False)
            ss.verify_tree(want=False)
            toks, _ = ss.accept_and_commit(D + 1)
            root = toks[-1]
            e2e_seq.extend(toks)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st1 = ss.stats()
        wall_max, e2e_tok = aggregate_ranks(dist, wall, len(e2e_seq), dist_device(local))
        streamed = (st1["stream_bytes"] - st0["stream_bytes"]) / a.steps
        e2e = {"value": e2e_tok / wall_max, "unit": "tokens/s", "h2d_bytes_per_step": int(4 + streamed),
               "d2h_bytes_per_step": int(4 * (len(e2e_seq) / a.steps) + 4),
               "h2d_breakdown": {"root_token": 4, "streamed_layer_weights": int(streamed)}, "steps": a.steps,
               "ms_per_step": wall / a.steps * 1e3, "same_steps_as_device_window": e2e_seq == emitted_seq}
    elif not a.no_e2e:
        # batched: re-prefill every slot and replay; ss_step_batch's host outputs are the step's D2H
        for b in range(Bq):
            ss.prefill_slot(b, request_for_rank(rank * Bq + b, cfg.vocab))
        for _ in range(a.warmup):
            step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = ss.stats()
        t0 = time.perf_counter()
        e2e_seq = [t for _ in range(a.steps) for r in step() for t in r]
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st1 = ss.stats()
        wall_max, e2e_tok = aggregate_ranks(dist, wall, len(e2e_seq), dist_device(local))
        streamed = (st1["stream_bytes"] - st0["stream_bytes"]) / a.steps
        e2e = {"value": e2e_tok / wall_max, "unit": "tokens/s", "h2d_bytes_per_step": int(streamed),
               "d2h_bytes_per_step": int(4 * Bq * (D + 2)), "h2d_breakdown": {"streamed_layer_weights": int(streamed)},
               "steps": a.steps, "ms_per_step": wall / a.steps * 1e3,
               "same_steps_as_device_window": e2e_seq == emitted_seq}
    # ---- prompt sweep: P MT-Bench-shaped prompts x R repeats (P:275 uses 20 samples; P:293 reports a std) ----
    sweep = None
    if a.prompts > 0 and Bq == 1:
        runs = []
        for rep in range(a.repeats):
            for p in range(a.prompts):
                pr = mtbench_prompt(SEED, 1000 + world * p + rank, cfg.vocab)
                ss.prefill(pr)
                for _ in range(a.warmup):
                    step()
                pms, pouts = timed_window(step, a.steps)
                ptaus = [len(r) for o in pouts for r in o]
                seq = [t for o in pouts for r in o for t in r]
                runs.append({"prompt": p, "repeat": rep, "len": len(pr), "ms_per_step": pms / a.steps,
                             "tokens_per_s": sum(ptaus) / (pms / 1e3), "steps_per_s": a.steps / (pms / 1e3),
                             "tau": float(np.mean(ptaus)), "full_accept_frac": float(np.mean([t == D + 1 for t in ptaus])),
                             "ngram4_repetition": ngram_repetition(seq)})
        tps = [r["tokens_per_s"] for r in runs]
        sps = [r["steps_per_s"] for r in runs]
        sweep = {"prompts": a.prompts, "repeats": a.repeats, "steps_each": a.steps,
                 "tokens_per_s_mean": statistics.mean(tps), "tokens_per_s_std": statistics.pstdev(tps),
                 "steps_per_s_mean": statistics.mean(sps), "steps_per_s_std": statistics.pstdev(sps),
                 "tau_mean": statistics.mean(r["tau"] for r in runs), "runs": runs}
    # context: one whole draft pass (all layers + head + attention/norm/top-k kernels), bytes of the
    # weights it must read (substitutes of offloaded layers, bf16 of resident ones, the bf16 head)
    draft_pass = None
    n_off = st["n_offloaded"]
    n_res = cfg.n_layers - n_off
    pass_bytes = n_off * sum(k2_bytes(N, K, M, a.sub_bits) for N, K in groups) + \
        n_res * sum(2 * N * K for N, K in groups) + cfg.vocab * cfg.hidden * 2
    k3 = None
    if Bq == 1:
        t_pass = ss.debug_time_pass(M, 5, 0)
        draft_pass = {"us": t_pass * 1e3, "weight_bytes": pass_bytes, "gbs": pass_bytes / (t_pass * 1e-3) / 1e9}
        # K3 tree attention inside the pass: its share by leaving it out (attribution only),
        # and the K/V bytes it must read: each frontier node's P prefix keys + its (<= 2) tree keys, K and
        # V, per kv head and layer (the per-(kv head, node) kernel reads the prefix once per node)
        t_noattn = ss.debug_time_pass(M, 5, 1)
        P = ss.stats()["committed_len"]
        kv_key = 2 * cfg.head_dim * 2 * cfg.n_kv_heads                     # bytes per key per layer
        k3_bytes = cfg.n_layers * M * (P + 2) * kv_key
        us = (t_pass - t_noattn) * 1e3
        k3 = {"us_per_pass": us, "us_per_layer": us / cfg.n_layers, "kv_bytes_per_pass": k3_bytes,
              "gbs": k3_bytes / (us * 1e-6) / 1e9 if us > 0 else None, "prefix_len": P, "bound": "latency",
              "note": "pass time with vs without the attention launches (debug_time_pass skip mask 1)"}
    # host link measured in the same run: pinned H2D 1 GiB on the copy stream, best of 5
    hbuf = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{dev}")
    best = 1e9
    with torch.cuda.stream(ss.copy_stream):
        for _ in range(5):
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0.record(ss.copy_stream)
            dbuf.copy_(hbuf, non_blocking=True)
            x1.record(ss.copy_stream)
            x1.synchronize()
            best = min(best, x0.elapsed_time(x1))
    link_gbs = (1 << 30) / (best * 1e-3) / 1e9
    del hbuf, dbuf
    # ---- offloading AR baseline ("None"): the same engine with D = 0 (one token per
    # target pass, nothing drafted) at the planner's maximum residency under the same cap; speedup =
    # SubSpec tokens/s / AR tokens/s, context for the paper's 9.15x ----
    ar = None
    if not a.no_ar and world == 1 and Bq == 1:
        ar_ss = SubSpec(cfg, int(a.cap_gib * GIB), device=dev, max_depth=D, max_top_k=max(k, 6), max_chunk=256,
                        embed_on_host=0 if a.embed_gpu else 1, compress_stream=0 if a.no_compress else 1)
        if a.sub_bits != 4:
            ar_ss.set_substitute_bits(a.sub_bits)
        ar_ss.load_synthetic(SEED, -1)
        ar_ss.build_substitutes(a.sub_bits, 64, method=a.quant)
        ar_ss.prefill(prompt0)
        for _ in range(a.warmup):
            ar_ss.step(0, 1, T)
        cs2 = ar_ss.compute_stream
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(cs2)
        ar_toks = [t for _ in range(a.steps) for t in ar_ss.step(0, 1, T)]
        rf = torch.cuda.Event()
        rf.record(ar_ss.copy_stream)
        cs2.wait_event(rf)
        f1.record(cs2)
        torch.cuda.synchronize()
        ar_ms = f0.elapsed_time(f1)
        ar_st = ar_ss.stats()
        ar = {"tokens_per_s": len(ar_toks) / (ar_ms / 1e3), "ms_per_token": ar_ms / len(ar_toks),
              "n_resident": ar_st["n_resident"], "tokens": len(ar_toks),
              "note": "D = 0 through the same engine, planner-max residency, same cap and codec (SURVEY §8(d) AR "
                      "baseline, P:536); speedup = value / tokens_per_s (tau of random weights, not trained ones)"}
        ar_ss.close()
    # ---- aggregate over ranks ----
    tmax, tot_tokens = aggregate_ranks(dist, ms, emitted, dist_device(local))
    value = tot_tokens / (tmax / 1e3)
    tau = float(np.mean(taus))
    steps_per_s = a.steps / (ms / 1e3)
    peaks = measured_peaks()
    hbm_peak = (peaks or {}).get("hbm_gbs") or 6650.0
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "k2_traffic.json"))).get("traffic_bytes_per_launch")
    except Exception:
        pass
    stream_gbs = st["stream_bytes"] / (st["stream_busy_ms"] * 1e-3) / 1e9 if st["stream_busy_ms"] else None
    # step roofline: streamed bytes over the host link, plus the draft's HBM time not
    # covered by the ring's prefetch of the next verify's layers
    s_host = st["stream_bytes"] / a.steps
    t_roof = s_host / (link_gbs * 1e9) + max(0.0, D * pass_bytes / (hbm_peak * 1e9) - st["ring_bytes"] / (link_gbs * 1e9))
    line = {
        "metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded random-init bf16 weights of the named shape; MT-Bench-shaped prompts)",
        "config": workload_config(a, cfg),
        "tau_mean": tau, "tau_hist": np.bincount(taus, minlength=D + 2).tolist(), "steps_per_s": steps_per_s,
        "full_accept_frac": float(np.mean([t == D + 1 for t in taus])),
        "ngram4_repetition": ngram_repetition(emitted_seq),
        "tokens_per_s_at_paper_tau_27.08": 27.08 * steps_per_s * Bq,
        "requests_per_gpu": Bq,
        "step_breakdown_ms": {"draft": st["draft_ms"] / a.steps, "verify": st["verify_ms"] / a.steps,
                              "accept": st["accept_ms"] / a.steps},
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / (ms / a.steps),
                          "formula": "streamed bytes / host link + max(0, D x draft-pass bytes / HBM peak - ring / host link)"},
        "roofline": {"kernel": f"K2 dequant-GEMV ({a.sub_bits}-bit g64 substitutes, M={M} tokens), all layers x 4 groups",
                     "bound": "hbm", "achieved": k2_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": k2_gbs / hbm_peak,
                     "traffic": traffic, "traffic_launch": "gate_up (ncu --set full, profiles/k2_traffic.json)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                     "per_group": per_group, "in_pass": k2_in_pass, "head_bf16_gemv_gbs": head_gbs,
                     "draft_pass": draft_pass, "k3_attention": k3},
        "streaming": {"mode": f"cooperative over {world} ranks (NEXT-1)" if coop else "per rank",
                      "peer_bytes_per_step": st["peer_bytes"] / a.steps,
                      "codec": "off (plain bf16)" if a.no_compress else "lossless exponent-coded bf16 (K7 codec)",
                      "bf16_bytes_per_step": st["stream_raw_bytes"] / a.steps,
                      "codec_ratio": (st["stream_bytes"] / st["stream_raw_bytes"]) if st["stream_raw_bytes"] else None,
                      "effective_bf16_gbs": st["stream_raw_bytes"] / (st["stream_busy_ms"] * 1e-3) / 1e9 if st["stream_busy_ms"] else None,
                      "bytes_per_step": s_host, "busy_gbs": stream_gbs,
                      "host_link_gbs_measured": link_gbs, "frac": (stream_gbs / link_gbs) if stream_gbs else None,
                      "duty_cycle": (st["stream_busy_ms"] / ms) if ms else None},
        "memory": {"shared_host_store": shm is not None, "embedding": "GPU (P:534)" if a.embed_gpu else "mapped host (R24)",
                   "arena_used": st["arena_used"], "arena_cap": st["arena_cap"], "ring_bytes": st["ring_bytes"],
                   "substitute_bytes": st["substitute_bytes"], "host_pinned_bytes": st["host_pinned_bytes"],
                   "n_resident": st["n_resident"]},
        "gpu_launches": int(st["gpu_launches"]),
        "clocks": ck, "e2e": e2e, "prompt_sweep": sweep, "setup_s": t_setup,
        "ar_baseline": ar, "speedup_vs_ar": (value / ar["tokens_per_s"]) if ar else None,
    }
    if rank == 0:
        if world == 1 and not a.no_cpu_baseline:
            sample = OracleSample(cfg, D, k, T, bits=a.sub_bits, quant=a.quant)
            ts, ns = [], []
            for _ in range(2):
                s_, n_ = sample.step_seconds()
                ts.append(s_)
                ns.append(n_)
            line["cpu_baseline"] = {"value": sum(ns) / sum(ts), "unit": "tokens/s", "cores": blas_threads(),
                                    "kind": "oracle", "sample": sample.describe() + " (2 steps)",
                                    "seconds_per_step": statistics.mean(ts), "tau": float(np.mean(ns))}
        print(json.dumps(line), flush=True)
    if coop:
        ss.coop_finish()
        dist.barrier()   # no rank's ring is still written by a peer
    ss.close()
    if dist:
        dist.barrier()   # every rank has released the shared store before it is unlinked
    if shm is not None:
        shm.close()
        if local == 0:
            shm.unlink()
    if dist:
        dist.destroy_process_group()


def main():
    a = args_()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
