"""K6 (target GEMM) timing at Qwen2.5-7B widths on a resident layer: tcgen05 vs the legacy mma.sync
kernel, M = 289 (D = 48, k = 6 tree) and 1025 (D = 64, k = 16), per group and for the head with the
verify's argmax epilogue.  Prints one JSON line per (kernel, M).  Used for profiles/k6_*.json and,
under ncu (-k regex:gemm_tc_kernel), for the tensor-pipe capture."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec

Ms = [int(a) for a in sys.argv[1:]] or [289, 1025]
iters = int(os.environ.get("K6_ITERS", "10"))
cfg = QWEN7B.with_(name="qwen2.5-7b-1l", n_layers=1)
ss = SubSpec(cfg, 4 * GIB, max_depth=64, max_top_k=16)
ss.load_synthetic(0x5EED, n_resident=1)
ss.build_substitutes(4, 64)
names = ["qkv", "o", "gate_up", "down", "head"]
VARIANTS = {0: "tcgen05 whole-chunk stages", 2: "tcgen05 half-chunk stages", 1: "legacy mma.sync"}
for var in [int(v) for v in os.environ.get("K6_VARIANTS", "0,2,1").split(",")]:
    ss.debug_set_knob(2, var)
    for M in Ms:
        out = {"kernel": VARIANTS[var], "M": M}
        tot_f, tot_t = 0.0, 0.0
        for gi, g in enumerate([0, 1, 2, 3, -1]):
            N, K = (cfg.vocab, cfg.hidden) if g == -1 else ss.group_shape(g)
            t = ss.debug_time_matmul(0, g, M, iters=iters, which=1)
            fl = 2.0 * M * N * K
            out[names[gi]] = {"us": round(t * 1e3, 2), "tflops": round(fl / (t * 1e-3) / 1e12, 1)}
            tot_f += fl
            tot_t += t
        out["all_tflops"] = round(tot_f / (tot_t * 1e-3) / 1e12, 1)
        print(json.dumps(out), flush=True)
ss.debug_set_knob(2, 0)
