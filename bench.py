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
TAU_FILE = os.path.join(ROOT, "profiles", "bench_tau.json")


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
    ap.add_argument("--sub-bits", type=int, default=4, choices=[4, 2],
                    help="substitute code bits (4 = the paper's setting, P:278; 2 = NEXT-3, P:343)")
    ap.add_argument("--embed-gpu", action="store_true",
                    help="embedding GPU-resident in the arena (PAPER.md:534) instead of mapped host memory (R24)")
    ap.add_argument("--no-async", action="store_true",
                    help="Table-2 ablation: no copy/compute overlap in the verify streaming (PAPER.md:305-308)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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
    """Bounded sample of the oracle on the SAME shape: one decoder layer (target + 4-bit substitute)
    plus the head, `nodes` draft and `nodes` target node-forwards, extrapolated to one full step of
    (1 + k(D-1)) draft + (1 + kD) target node-forwards through all layers.  The seeded weights are
    generated once (setup); every call of step_seconds() re-times the sample."""

    def __init__(self, cfg, depth, topk, nodes=6, bits=4):
        from oracle.model import TargetWeights, draft_layers
        self.cfg, self.depth, self.topk, self.nodes = cfg, depth, topk, nodes
        self.cfg1 = cfg.with_(n_layers=1)
        t0 = time.time()
        self.tw = TargetWeights(self.cfg1, SEED)
        self.dl = draft_layers(self.tw, 0, bits)
        self.setup = time.time() - t0

    def step_seconds(self):
        from oracle.model import KVCache, forward_nodes
        from oracle.tree import tempered_log_softmax, select_topk
        cfg, cfg1, tw, nodes, topk, depth = self.cfg, self.cfg1, self.tw, self.nodes, self.topk, self.depth
        kv = KVCache(cfg1, nodes + 1)
        toks = list(range(1, nodes + 1))
        slots = list(range(nodes))
        anc = [[s] for s in slots]
        pos = [0] * nodes
        t0 = time.perf_counter()
        forward_nodes(cfg1, self.dl, tw, kv, toks, slots, pos, anc)
        t_draft_node = (time.perf_counter() - t0) / nodes
        t0 = time.perf_counter()
        logits = forward_nodes(cfg1, tw.layers, tw, kv, toks, slots, pos, anc)
        t_target_node = (time.perf_counter() - t0) / nodes
        h = np.ones(cfg.hidden)
        t0 = time.perf_counter()
        for _ in range(nodes):
            tw.head @ h
        t_head = (time.perf_counter() - t0) / nodes
        t0 = time.perf_counter()
        lp = np.stack([tempered_log_softmax(logits[i], 0.2) for i in range(min(topk, nodes))])
        select_topk(list(range(len(lp))), [0.0] * len(lp), lp, topk)
        t_select = time.perf_counter() - t0
        L = cfg.n_layers
        n_draft = 1 + topk * (depth - 1)
        n_verify = 1 + topk * depth
        step = (n_draft * ((t_draft_node - t_head) * L + t_head) + n_verify * ((t_target_node - t_head) * L + t_head)
                + depth * t_select)
        info = {"t_draft_node_1layer_s": t_draft_node, "t_target_node_1layer_s": t_target_node, "t_head_s": t_head,
                "t_select_s": t_select, "setup_s": self.setup, "node_forwards": n_draft + n_verify}
        return step, info


def oracle_step_seconds(cfg, depth, topk, nodes=6, bits=4):
    """One-shot OracleSample (setup + one timed sample) -> (seconds/step, info)."""
    return OracleSample(cfg, depth, topk, nodes, bits).step_seconds()


def load_tau():
    try:
        return json.load(open(TAU_FILE))
    except Exception:
        return None


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = PRESETS[a.config]
    tau_rec = load_tau()
    tau = tau_rec["tau"] if tau_rec and tau_rec.get("config") == a.config else 1.0
    times = []
    info = None
    sample = OracleSample(cfg, a.depth, a.topk, bits=a.sub_bits)   # weights generated once, each step re-timed
    for i in range(a.warmup + a.steps):
        s, info = sample.step_seconds()
        if i >= a.warmup:
            times.append(s)
    step_s = statistics.mean(times)
    value = tau / step_s
    cores = blas_threads()
    sample = (f"1 {cfg.name}-shape decoder layer (bf16 target + {a.sub_bits}-bit substitute, fp64 NumPy oracle) + head, 6 draft "
              f"and 6 target node-forwards per step, extrapolated to a D={a.depth},k={a.topk} step "
              f"({info['node_forwards']} node-forwards x {cfg.n_layers} layers); tau={tau:.3f} "
              f"({'from the deterministic GPU run, ' + TAU_FILE if tau_rec else 'assumed 1'})")
    line = {"metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random-init weights, MT-Bench-shaped prompt)",
            "config": workload_config(a, cfg), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "oracle_timing": info}
    print(json.dumps(line), flush=True)


def workload_config(a, cfg):
    batch = "" if a.batch == 1 else f", {a.batch} requests per GPU sharing one weight stream (NEXT-2)"
    return {"workload": f"{cfg.name} SubSpec step, {a.cap_gib:g} GiB cap, n_resident={a.n_resident}, "
                        f"{a.sub_bits}-bit g64 substitutes, D={a.depth} k={a.topk} T={a.temp}, MT-Bench-shaped prompt{batch}",
            "model_shape": cfg.name, "vram_cap_gib": a.cap_gib, "n_resident": a.n_resident, "depth": a.depth,
            "top_k": a.topk, "sharpen_t": a.temp, "batch": a.batch, "max_context": cfg.max_context,
            "l2": "inputs larger than L2 (>= 4.76 GB of draft weights per draft pass; 13 GB streamed per verify)",
            "parallelism": f"requests partitioned, {a.gpus} GPU(s), no collective"}


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
                 max_batch=Bq, embed_on_host=0 if a.embed_gpu else 1, async_stream=0 if a.no_async else 1)
    if a.sub_bits != 4:
        ss.set_substitute_bits(a.sub_bits)
    shm = load_weights_for_job(ss, dist, local, a.n_resident)
    ss.build_substitutes(a.sub_bits, 64)
    if Bq == 1:
        ss.prefill(request_for_rank(rank, cfg.vocab))
        step = lambda: [ss.step(D, k, T)]                     # noqa: E731
    else:   # rank r decodes requests r*B .. r*B + B - 1, all B in one step
        ss.set_batch(Bq)
        for b in range(Bq):
            ss.prefill_slot(b, request_for_rank(rank * Bq + b, cfg.vocab))
        step = lambda: ss.step_batch(Bq, D, k, T)            # noqa: E731
    t_setup = time.time() - t_setup
    for _ in range(a.warmup):
        step()
    ss.reset_stats()
    cs = ss.compute_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0.record(cs)
    emitted, taus = 0, []
    for _ in range(a.steps):
        for t in step():
            emitted += len(t)
            taus.append(len(t))
    # steady state: the region starts with the streaming ring already prefetched for the next verify
    # (by the warm-up steps), so it also ends only when the ring is prefetched again — the copy
    # stream's outstanding prefetch is inside the timed region
    ring_full = torch.cuda.Event()
    ring_full.record(ss.copy_stream)
    cs.wait_event(ring_full)
    e1.record(cs)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    st = ss.stats()
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
    # ---- e2e through the C-ABI with host buffers: root token H2D, emitted tokens D2H ----
    e2e = None
    if not a.no_e2e and Bq > 1:
        # batched: ss_step_batch's host outputs are the step's D2H; roots stay on the device
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = ss.stats()
        t0 = time.perf_counter()
        e2e_tok = 0
        n_e2e = max(2, a.steps)   # as many steps as the device-timed region (tau varies per step)
        for _ in range(n_e2e):
            e2e_tok += sum(len(t) for t in step())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st1 = ss.stats()
        wall, e2e_tok = aggregate_ranks(dist, wall, e2e_tok, dist_device(local))
        streamed = (st1["stream_bytes"] - st0["stream_bytes"]) / n_e2e
        e2e = {"value": e2e_tok / wall, "unit": "tokens/s", "h2d_bytes_per_step": int(streamed),
               "d2h_bytes_per_step": int(4 * Bq * (D + 2)),
               "h2d_breakdown": {"streamed_layer_weights": int(streamed)}, "steps": n_e2e,
               "ms_per_step": wall / n_e2e * 1e3}
    elif not a.no_e2e:
        root = int(ss.step(D, k, T)[-1])
        # one untimed step through the same calls (the host-root draft path has its own graph instance)
        ss.draft_tree(D, k, T, root_token=root, want_tree=False)
        ss.verify_tree(want=False)
        root = ss.accept_and_commit(D + 1)[0][-1]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = ss.stats()
        t0 = time.perf_counter()
        e2e_tok = 0
        n_e2e = max(2, a.steps)   # as many steps as the device-timed region (tau varies per step)
        for _ in range(n_e2e):
            ss.draft_tree(D, k, T, root_token=root, want_tree=False)
            ss.verify_tree(want=False)
            toks, _ = ss.accept_and_commit(D + 1)
            root = toks[-1]
            e2e_tok += len(toks)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st1 = ss.stats()
        wall, e2e_tok = aggregate_ranks(dist, wall, e2e_tok, dist_device(local))
        streamed = (st1["stream_bytes"] - st0["stream_bytes"]) / n_e2e
        e2e = {"value": e2e_tok / wall, "unit": "tokens/s", "h2d_bytes_per_step": int(4 + streamed),
               "d2h_bytes_per_step": int(4 * (e2e_tok / max(1, n_e2e)) + 4),
               "h2d_breakdown": {"root_token": 4, "streamed_layer_weights": int(streamed)}, "steps": n_e2e,
               "ms_per_step": wall / n_e2e * 1e3}
    # context: one whole draft pass (all layers + head + attention/norm/top-k kernels), bytes of the
    # weights it must read (substitutes of offloaded layers, bf16 of resident ones, the bf16 head)
    draft_pass = None
    if Bq == 1:
        n_off = st["n_offloaded"]
        n_res = cfg.n_layers - n_off
        pass_bytes = n_off * sum(k2_bytes(N, K, M, a.sub_bits) for N, K in groups) + \
            n_res * sum(2 * N * K for N, K in groups) + cfg.vocab * cfg.hidden * 2
        t_pass = ss.debug_time_pass(M, 5, 0)
        draft_pass = {"us": t_pass * 1e3, "weight_bytes": pass_bytes, "gbs": pass_bytes / (t_pass * 1e-3) / 1e9}
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
    line = {
        "metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded random-init bf16 weights of the named shape; MT-Bench-shaped prompts)",
        "config": workload_config(a, cfg),
        "tau_mean": tau, "tau_hist": np.bincount(taus, minlength=D + 2).tolist(), "steps_per_s": steps_per_s,
        "tokens_per_s_at_paper_tau_27.08": 27.08 * steps_per_s * Bq,
        "requests_per_gpu": Bq,
        "step_breakdown_ms": {"draft": st["draft_ms"] / a.steps, "verify": st["verify_ms"] / a.steps,
                              "accept": st["accept_ms"] / a.steps},
        "roofline": {"kernel": f"K2 dequant-GEMV ({a.sub_bits}-bit g64 substitutes, M={M} tokens), all layers x 4 groups",
                     "bound": "hbm", "achieved": k2_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": k2_gbs / hbm_peak,
                     "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                     "per_group": per_group, "head_bf16_gemv_gbs": head_gbs, "draft_pass": draft_pass},
        "streaming": {"bytes_per_step": st["stream_bytes"] / a.steps, "busy_gbs": stream_gbs,
                      "host_link_gbs_measured": link_gbs, "frac": (stream_gbs / link_gbs) if stream_gbs else None,
                      "duty_cycle": (st["stream_busy_ms"] / ms) if ms else None},
        "memory": {"shared_host_store": shm is not None,
                   "arena_used": st["arena_used"], "arena_cap": st["arena_cap"], "ring_bytes": st["ring_bytes"],
                   "substitute_bytes": st["substitute_bytes"], "host_pinned_bytes": st["host_pinned_bytes"],
                   "n_resident": st["n_resident"]},
        "gpu_launches": int(st["gpu_launches"]),
        "clocks": ck, "e2e": e2e, "setup_s": t_setup,
    }
    if rank == 0:
        os.makedirs(os.path.dirname(TAU_FILE), exist_ok=True)
        if world == 1 and Bq == 1:
            try:
                json.dump({"config": a.config, "tau": tau, "steps": a.steps, "note": "deterministic seeded workload"},
                          open(TAU_FILE, "w"))
            except Exception:
                pass
        if world == 1 and not a.no_cpu_baseline:
            s, info = oracle_step_seconds(cfg, D, k, bits=a.sub_bits)
            line["cpu_baseline"] = {
                "value": tau / s, "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
                "sample": (f"1 {cfg.name}-shape decoder layer + head, 6 draft + 6 target node-forwards (fp64 NumPy "
                           f"oracle), extrapolated to one D={D},k={k} step ({info['node_forwards']} node-forwards x "
                           f"{cfg.n_layers} layers) at this run's tau={tau:.3f}"),
                "seconds_per_step": s}
        print(json.dumps(line), flush=True)
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
