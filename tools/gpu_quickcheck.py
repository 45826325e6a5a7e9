"""Quick GPU bring-up check (tiny config): generator, quantizer, K2, forward, generate vs oracle."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import TINY, SMALL
from synth import weights as W
from synth.prompts import mtbench_prompt
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64
from oracle.decode import ar_generate, sd_generate, Session
from paper_2509_18344_b200.binding import SubSpec

SEED = 0x5EED

def step(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[ok] {name} ({time.time()-t:.2f}s) {r if r is not None else ''}", flush=True)
    except Exception as e:
        print(f"[FAIL] {name}: {e}", flush=True)
        traceback.print_exc()

def main(cfgname="tiny"):
    cfg = {"tiny": TINY, "small": SMALL}[cfgname]
    ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, max_chunk=256)
    specs = W.tensor_specs(cfg)
    def gen():
        bad = []
        for tid, name, shape, kind, sigma in specs[:6] + specs[-2:]:
            g = ss.debug_gen_tensor(SEED, tid, shape, kind, sigma)
            ref = W.gen_tensor_bits(SEED, tid, shape, kind, sigma)
            if not np.array_equal(g.reshape(ref.shape), ref): bad.append(name)
        assert not bad, bad
    step("generator parity", gen)
    step("load_weights", lambda: ss.load_synthetic(SEED, n_resident=1))
    model = W.generate_model(cfg, SEED)
    def groups():
        for l in range(cfg.n_layers):
            g0 = ss.debug_read_group(l, 0)
            ref = np.concatenate([model[f"l{l}.wq"], model[f"l{l}.wk"], model[f"l{l}.wv"]])
            assert np.array_equal(g0, ref), f"qkv l{l}"
            g2 = ss.debug_read_group(l, 2)
            F = cfg.ffn
            ref2 = np.zeros_like(g2)
            for b in range(F // 64):
                ref2[128*b:128*b+64] = model[f"l{l}.wg"][64*b:64*b+64]
                ref2[128*b+64:128*b+128] = model[f"l{l}.wu"][64*b:64*b+64]
            assert np.array_equal(g2, ref2), f"gate_up l{l}"
            assert np.array_equal(ss.debug_read_group(l, 1), model[f"l{l}.wo"])
            assert np.array_equal(ss.debug_read_group(l, 3), model[f"l{l}.wd"])
    step("group layouts", groups)
    step("build_substitutes", lambda: ss.build_substitutes(4, 64))
    def subs():
        for g in range(4):
            codes, s, z = ss.debug_get_substitute(1, g)
            wb = ss.debug_read_group(1, g)
            rc, rs, rz = quantize(bf16_bits_to_f64(wb))
            assert np.array_equal(codes, rc), f"codes g{g} mismatches {np.sum(codes != rc)}"
            assert np.array_equal(bf16_bits_to_f64(s), rs), f"s g{g}"
            assert np.array_equal(bf16_bits_to_f64(z), rz), f"z g{g}"
    step("K1 substitutes bit-exact", subs)
    def onehot():
        for g in range(4):
            N, K = ss.group_shape(g)
            wb = ss.debug_read_group(1, g)
            rc, rs, rz = quantize(bf16_bits_to_f64(wb))
            what = dequantize(rc, rs, rz)
            for k0 in range(0, K, 32):
                M = min(32, K - k0)
                x = np.zeros((M, K), np.uint16)
                for m in range(M): x[m, k0 + m] = 0x3F80
                y = ss.debug_matmul(0, 1, g, x)
                assert np.array_equal(y.astype(np.float64), what[:, k0:k0+M].T), f"one-hot g{g} k0 {k0}: {np.abs(y - what[:, k0:k0+M].T).max()}"
    step("K2 one-hot exact dequant", onehot)
    def randx():
        rng = np.random.default_rng(0)
        for g in range(4):
            N, K = ss.group_shape(g)
            wb = ss.debug_read_group(1, g)
            what = dequantize(*quantize(bf16_bits_to_f64(wb)))
            for M in (1, 6, 13, 32):
                xf = rng.standard_normal((M, K)).astype(np.float32)
                xb = W.f32_to_bf16_bits(xf)
                y = ss.debug_matmul(0, 1, g, xb)
                ref = bf16_bits_to_f64(xb) @ what.T
                err = np.abs(y - ref).max() / np.abs(ref).max()
                assert err < 1e-5, (g, M, err)
                # resident (bf16) GEMV and GEMM on layer 0
                y0 = ss.debug_matmul(0, 0, g, xb)
                ref0 = bf16_bits_to_f64(xb) @ bf16_bits_to_f64(ss.debug_read_group(0, g)).T
                assert np.abs(y0 - ref0).max() / np.abs(ref0).max() < 1e-5, ("bf16 gemv", g, M)
            for M in (1, 100, 256):
                xf = rng.standard_normal((M, K)).astype(np.float32)
                xb = W.f32_to_bf16_bits(xf)
                y0 = ss.debug_matmul(1, 0, g, xb)
                ref0 = bf16_bits_to_f64(xb) @ bf16_bits_to_f64(ss.debug_read_group(0, g)).T
                assert np.abs(y0 - ref0).max() / np.abs(ref0).max() < 1e-5, ("gemm", g, M)
    step("K2/K6 random activations", randx)
    prompt = mtbench_prompt(SEED, 0, cfg.vocab, 32)
    def gen_cmp():
        out, hist = ss.generate(prompt, 24, 4, 6, 0.2)
        ref, _ = ar_generate(cfg, prompt, 24, seed=SEED, mode="bf16")
        st = ss.stats()
        # teacher-forced oracle logits along the GPU sequence: gap at each disagreement
        s = Session(cfg, SEED, mode="bf16", max_nodes=256)
        from oracle.tree import Tree
        seq = list(prompt) + list(out)
        toks = [int(t) for t in seq]
        n = len(toks)
        lg = s.forward_tree("target", Tree(toks, [i - 1 for i in range(n)], list(range(n)), [0.0] * n))
        info = []
        for j in range(len(out)):
            row = lg[len(prompt) - 1 + j]
            top = np.argsort(-row)[:2]
            if top[0] != out[j]:
                info.append((j, int(out[j]), int(top[0]), float(row[top[0]] - row[out[j]]), float(row[top[0]] - row[top[1]])))
        return f"\n gpu {out}\n ref {ref}\n disagreements (pos, gpu, oracle, l[oracle]-l[gpu], oracle gap) {info}\n hist {hist.tolist()} stats {st}"
    step("generate vs oracle AR", gen_cmp)
    def gen_ar():
        out, hist = ss.generate(prompt, 24, 0, 1, 0.2)
        return f"AR gpu {out}"
    step("generate D=0", gen_ar)
    ss.close()

if __name__ == "__main__":
    main(*(sys.argv[1:] or ["tiny"]))
