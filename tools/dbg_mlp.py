"""Fused vs unfused draft MLP: debug_forward logits at tiny/small shapes for chains of M nodes."""
import sys, os, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "child":
    from synth.configs import TINY, SMALL, QWEN7B, GIB
    from synth.prompts import mtbench_prompt
    from paper_2509_18344_b200.binding import SubSpec
    cfg = {"tiny": TINY, "small": SMALL}[sys.argv[2]]
    nres = int(sys.argv[3]); M = int(sys.argv[4])
    ss = SubSpec(cfg, 512 << 20, max_depth=8, max_top_k=6, max_chunk=256)
    ss.load_weights(0x5EED, n_resident=nres)
    ss.build_substitutes(4, 64)
    ss.prefill(mtbench_prompt(0x5EED, 1, cfg.vocab, 40))
    toks = np.arange(1, M + 1, dtype=np.int32)
    par = np.arange(-1, M - 1, dtype=np.int32)
    out = ss.debug_forward(0, toks, par)
    np.save(sys.argv[5], out)
    sys.exit(0)
for cfg in ("tiny",):
    for nres in (0,):
        for M in (1, 6):
            res = []
            for f in ("0", "1"):
                fn = f"/tmp/dbg_mlp_{f}.npy"
                env = dict(os.environ, SS_FUSE_MLP=f)
                r = subprocess.run([sys.executable, __file__, "child", cfg, str(nres), str(M), fn], env=env,
                                   capture_output=True, text=True, timeout=300)
                if r.returncode:
                    print(cfg, nres, M, "fuse", f, "FAILED", r.stderr[-300:]); res = None; break
                res.append(np.load(fn))
            if res:
                d = np.abs(res[0] - res[1]); sc = np.abs(res[0]).max()
                print(cfg, "nres", nres, "M", M, "maxdiff", d.max(), "scale", sc, "rows bad", np.nonzero(d.max(1) > 1e-2 * sc)[0][:10], flush=True)
