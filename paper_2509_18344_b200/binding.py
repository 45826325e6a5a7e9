"""Thin ctypes binding of libsubspec (include/subspec.h).  Argument marshalling only: every
step of the decode path runs in the library's CUDA kernels.  PyTorch provides the device arena
(the emulated VRAM cap) and the two CUDA streams; nothing else.

There is no CPU fallback: if libsubspec.so is missing or no CUDA device is present, construction
raises.
"""
import ctypes
import os

import numpy as np

from .build import LIB

c_int32, c_int64, c_float, c_double, c_void_p, c_size_t, c_uint64 = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t,
    ctypes.c_uint64)

STATUS = {0: "SS_OK", 1: "SS_ERR_INVALID", 2: "SS_ERR_CAPACITY", 3: "SS_ERR_STRUCTURE", 4: "SS_ERR_BUDGET",
          5: "SS_ERR_CUDA"}


class ModelConfigC(ctypes.Structure):
    _fields_ = [("n_layers", c_int32), ("hidden", c_int32), ("n_heads", c_int32), ("n_kv_heads", c_int32),
                ("head_dim", c_int32), ("ffn", c_int32), ("vocab", c_int32), ("max_context", c_int32),
                ("rope_theta", c_float), ("rms_eps", c_float), ("qkv_bias", c_int32), ("precision", c_int32)]


SS_BF16, SS_FP32 = 0, 1


class OptionsC(ctypes.Structure):
    _fields_ = [("embed_on_host", c_int32), ("async_stream", c_int32), ("cuda_graphs", c_int32),
                ("fuse_norm", c_int32), ("separate_draft_kv", c_int32), ("compress_stream", c_int32)]


class HostLayerC(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("attn_norm", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "mlp_norm", "wg", "wu",
                                        "wd")]


class HostWeightsC(ctypes.Structure):
    _fields_ = [("embed", c_void_p), ("layers", ctypes.POINTER(HostLayerC)), ("final_norm", c_void_p),
                ("head", c_void_p)]


class LimitsC(ctypes.Structure):
    _fields_ = [("max_depth", c_int32), ("max_top_k", c_int32), ("max_chunk", c_int32), ("max_batch", c_int32)]


class QuantSpecC(ctypes.Structure):
    _fields_ = [("bits", c_int32), ("group_size", c_int32), ("method", c_int32), ("hqq_iters", c_int32)]


QUANT_METHODS = {"rtn": 0, "hqq": 1}


class DraftParamsC(ctypes.Structure):
    _fields_ = [("depth", c_int32), ("top_k", c_int32), ("sharpen_t", c_float)]


class StatsC(ctypes.Structure):
    _fields_ = [("steps", c_int64), ("tokens_emitted", c_int64), ("prefill_tokens", c_int64),
                ("gpu_launches", c_int64), ("draft_ms", c_double), ("verify_ms", c_double),
                ("accept_ms", c_double), ("stream_bytes", c_double), ("stream_busy_ms", c_double),
                ("arena_used", c_int64), ("arena_cap", c_int64), ("ring_bytes", c_int64),
                ("host_pinned_bytes", c_int64), ("substitute_bytes", c_int64), ("n_resident", c_int32),
                ("n_offloaded", c_int32), ("committed_len", c_int32), ("last_d_eff", c_int32),
                ("peer_bytes", c_double), ("stream_raw_bytes", c_double)]


P = ctypes.POINTER
_FUNCS = {
    "ss_create": [P(ModelConfigC), P(LimitsC), P(OptionsC), ctypes.c_int, c_void_p, c_size_t, c_void_p, c_void_p,
                  P(c_void_p)],
    "ss_load_weights": [c_void_p, P(HostWeightsC), c_int32],
    "ss_load_weights_synthetic": [c_void_p, c_uint64, c_int32],
    "ss_set_substitute_bits": [c_void_p, c_int32],
    "ss_host_store_bytes": [c_void_p, c_int32, P(c_size_t)],
    "ss_load_weights_synthetic_shared": [c_void_p, c_uint64, c_int32, c_void_p, c_size_t, c_int32],
    "ss_build_substitutes": [c_void_p, P(QuantSpecC)],
    "ss_prefill": [c_void_p, c_void_p, c_int32, c_int32, P(c_int32)],
    "ss_draft_tree": [c_void_p, c_int32, P(DraftParamsC), c_void_p, c_void_p, c_void_p, c_void_p, P(c_int32)],
    "ss_verify_tree": [c_void_p, c_void_p, c_void_p],
    "ss_accept_and_commit": [c_void_p, c_void_p, c_void_p, c_void_p],
    "ss_step": [c_void_p, P(DraftParamsC), c_void_p, P(c_int32)],
    "ss_generate": [c_void_p, c_void_p, c_int32, c_int32, c_int32, P(DraftParamsC), c_void_p, P(c_int32), c_void_p],
    "ss_set_batch": [c_void_p, c_int32],
    "ss_prefill_slot": [c_void_p, c_int32, c_void_p, c_int32, c_int32, P(c_int32)],
    "ss_step_batch": [c_void_p, P(DraftParamsC), c_int32, c_void_p, c_void_p],
    "ss_generate_batch": [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_int32, P(DraftParamsC), c_void_p, c_void_p,
                          c_void_p],
    "ss_get_stats": [c_void_p, P(StatsC)],
    "ss_coop_export": [c_void_p, c_void_p],
    "ss_coop_enable": [c_void_p, c_int32, c_int32, c_void_p],
    "ss_coop_finish": [c_void_p],
    "ss_reset_stats": [c_void_p],
    "ss_debug_gen_tensor": [c_void_p, c_uint64, c_int32, c_int64, c_int64, c_int32, c_double, c_void_p],
    "ss_debug_read_group": [c_void_p, c_int32, c_int32, c_void_p],
    "ss_debug_get_substitute": [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p],
    "ss_debug_matmul": [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_void_p],
    "ss_debug_forward": [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p, c_void_p],
    "ss_debug_set_tree": [c_void_p, c_void_p, c_void_p, c_int32, c_int32],
    "ss_debug_read_kv": [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p],
    "ss_debug_read_draft_kv": [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p],
    "ss_debug_decode_group": [c_void_p, c_int32, c_int32, c_void_p, P(c_int32), P(c_uint64)],
    "ss_debug_time_matmul": [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, P(c_float)],
    "ss_debug_time_pass": [c_void_p, c_int32, c_int32, c_int32, P(c_float)],
    "ss_debug_set_knob": [c_void_p, c_int32, c_int32],
    "ss_debug_trace_pass": [c_void_p, c_int32, c_void_p, c_int32, P(c_int32)],
    "ss_debug_cta_trace": [c_void_p, c_int32, c_int32, c_void_p, c_int32, P(c_int32)],
    "ss_debug_step_timeline": [c_void_p, P(DraftParamsC), c_void_p, c_int32, P(c_int32), c_void_p],
}
EXPORTED = list(_FUNCS) + ["ss_last_error", "ss_destroy", "ss_default_options"]

_lib = None


def load_library(path=None):
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SS_LIBSUBSPEC", LIB)   # SS_LIBSUBSPEC: an experimental build
    if not os.path.exists(path):
        raise RuntimeError(f"libsubspec.so not built ({path}); run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, args in _FUNCS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.ss_last_error.argtypes = [c_void_p]
    lib.ss_last_error.restype = ctypes.c_char_p
    lib.ss_destroy.argtypes = [c_void_p]
    lib.ss_destroy.restype = None
    lib.ss_default_options.argtypes = [P(OptionsC)]
    lib.ss_default_options.restype = None
    _lib = lib
    return lib


class SubSpecError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    return a.ctypes.data_as(c_void_p) if a is not None else None


def model_config_c(cfg, precision=SS_BF16):
    return ModelConfigC(cfg.n_layers, cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn, cfg.vocab,
                        cfg.max_context, cfg.rope_theta, cfg.rms_eps, int(cfg.qkv_bias), int(precision))


class SubSpec:
    """One decode session on one GPU: the C-ABI context plus its torch-owned arena and streams."""

    def __init__(self, cfg, arena_bytes, device=0, max_depth=48, max_top_k=6, max_chunk=256, max_batch=1,
                 precision=SS_BF16, **options):
        """options: ss_options fields (embed_on_host, async_stream, cuda_graphs, fuse_norm, separate_draft_kv,
        compress_stream)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("SubSpec needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.cfg = cfg
        self.device = device
        self.precision = precision
        self.limits = LimitsC(max_depth, max_top_k, max_chunk, max_batch)
        self.options = OptionsC()
        self.lib.ss_default_options(ctypes.byref(self.options))
        for k, v in options.items():
            if k not in dict(OptionsC._fields_):
                raise TypeError(f"unknown ss_options field {k}")
            setattr(self.options, k, int(v))
        self.arena = torch.empty(int(arena_bytes), dtype=torch.uint8, device=f"cuda:{device}")
        self.compute_stream = torch.cuda.Stream(device=device)
        self.copy_stream = torch.cuda.Stream(device=device)
        torch.cuda.synchronize(device)
        ctx = c_void_p()
        st = self.lib.ss_create(ctypes.byref(model_config_c(cfg, precision)), ctypes.byref(self.limits),
                                ctypes.byref(self.options), device,
                                c_void_p(self.arena.data_ptr()), c_size_t(int(arena_bytes)),
                                c_void_p(self.compute_stream.cuda_stream), c_void_p(self.copy_stream.cuda_stream),
                                ctypes.byref(ctx))
        if st:
            raise SubSpecError(st, "ss_create failed")
        self.ctx = ctx

    def _check(self, st):
        if st:
            raise SubSpecError(st, self.lib.ss_last_error(self.ctx).decode())

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.ss_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the method ---------------------------------------------------------------------
    def set_substitute_bits(self, bits):
        """Substitute code width (4, 3 or 2); before load_weights (sizes the substitutes' layout)."""
        self._check(self.lib.ss_set_substitute_bits(self.ctx, bits))

    def load_weights(self, weights, n_resident=0):
        """weights: dict name -> uint16 array of bf16 bits in synth/weights.py's naming ("embed",
        "l{l}.wq", ..., "final_norm", "head"), [out x in] row-major.  Only marshalled: the library
        copies and tiles them on the device."""
        c = self.cfg
        keep = {}

        def ptr(name, shape):
            a = np.ascontiguousarray(weights[name], dtype=np.uint16)
            if a.shape != tuple(shape):
                raise ValueError(f"{name}: shape {a.shape} != {tuple(shape)}")
            keep[name] = a
            return a.ctypes.data_as(c_void_p)

        layers = (HostLayerC * c.n_layers)()
        for l in range(c.n_layers):
            L = layers[l]
            L.attn_norm = ptr(f"l{l}.attn_norm", (c.hidden,))
            L.wq = ptr(f"l{l}.wq", (c.q_dim, c.hidden))
            L.wk = ptr(f"l{l}.wk", (c.kv_dim, c.hidden))
            L.wv = ptr(f"l{l}.wv", (c.kv_dim, c.hidden))
            if c.qkv_bias:
                L.bq = ptr(f"l{l}.bq", (c.q_dim,))
                L.bk = ptr(f"l{l}.bk", (c.kv_dim,))
                L.bv = ptr(f"l{l}.bv", (c.kv_dim,))
            L.wo = ptr(f"l{l}.wo", (c.hidden, c.q_dim))
            L.mlp_norm = ptr(f"l{l}.mlp_norm", (c.hidden,))
            L.wg = ptr(f"l{l}.wg", (c.ffn, c.hidden))
            L.wu = ptr(f"l{l}.wu", (c.ffn, c.hidden))
            L.wd = ptr(f"l{l}.wd", (c.hidden, c.ffn))
        hw = HostWeightsC(ptr("embed", (c.vocab, c.hidden)), layers, ptr("final_norm", (c.hidden,)),
                          ptr("head", (c.vocab, c.hidden)))
        self._check(self.lib.ss_load_weights(self.ctx, ctypes.byref(hw), n_resident))

    def load_synthetic(self, seed, n_resident=0):
        """Weights from the library's device-side synthetic generator."""
        self._check(self.lib.ss_load_weights_synthetic(self.ctx, c_uint64(seed), n_resident))

    def host_store_bytes(self, n_resident=0):
        out = c_size_t()
        self._check(self.lib.ss_host_store_bytes(self.ctx, n_resident, ctypes.byref(out)))
        return out.value

    def load_synthetic_shared(self, seed, n_resident, store_addr, store_bytes, fill):
        """Offloaded layers in a caller-owned host store (address of a page-aligned mapping that
        outlives this context, e.g. multiprocessing.shared_memory); fill=True generates them."""
        self._keep_store = store_addr
        self._check(self.lib.ss_load_weights_synthetic_shared(self.ctx, c_uint64(seed), n_resident,
                                                               c_void_p(store_addr), store_bytes, 1 if fill else 0))

    def build_substitutes(self, bits=4, group=64, method="rtn", hqq_iters=0):
        m = QUANT_METHODS[method] if isinstance(method, str) else int(method)
        self._check(self.lib.ss_build_substitutes(self.ctx, ctypes.byref(QuantSpecC(bits, group, m, hqq_iters))))

    def prefill(self, prompt, chunk=256):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = c_int32()
        self._check(self.lib.ss_prefill(self.ctx, _ptr(p), len(p), chunk, ctypes.byref(out)))
        return out.value

    def draft_tree(self, depth, top_k, sharpen_t, root_token=-1, want_tree=True, n_req=1):
        """n_req > 1 (batched slots): every array is [n_req, n_nodes]."""
        n_max = 1 + top_k * depth
        arrs = [np.zeros(n_req * n_max, np.int32), np.zeros(n_req * n_max, np.int32), np.zeros(n_req * n_max, np.int32),
                np.zeros(n_req * n_max, np.float32)] if want_tree else [None] * 4
        n = c_int32()
        self._check(self.lib.ss_draft_tree(self.ctx, root_token, ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)),
                                           *[_ptr(a) for a in arrs], ctypes.byref(n)))
        if not want_tree:
            return n.value
        nn = n.value
        cut = (lambda a: a[:nn]) if n_req == 1 else (lambda a: a[:n_req * nn].reshape(n_req, nn))
        return {"tokens": cut(arrs[0]), "parents": cut(arrs[1]), "depths": cut(arrs[2]), "scores": cut(arrs[3])}

    def verify_tree(self, n_nodes=None, want=True, n_req=1):
        if not want:
            self._check(self.lib.ss_verify_tree(self.ctx, None, None))
            return None
        am = np.zeros(n_req * n_nodes, np.int32)
        gap = np.zeros(n_req * n_nodes, np.float32)
        self._check(self.lib.ss_verify_tree(self.ctx, _ptr(am), _ptr(gap)))
        if n_req > 1:
            return am.reshape(n_req, n_nodes), gap.reshape(n_req, n_nodes)
        return am, gap

    def accept_and_commit_batch(self, n_req, stride):
        """Batched accept/commit: per-slot emitted tokens and committed tree slots (root first)."""
        toks = np.zeros(n_req * stride, np.int32)
        path = np.zeros(n_req * stride, np.int32)
        n = np.zeros(n_req, np.int32)
        self._check(self.lib.ss_accept_and_commit(self.ctx, _ptr(toks), _ptr(n), _ptr(path)))
        return ([toks[b * stride: b * stride + n[b]].tolist() for b in range(n_req)],
                [path[b * stride: b * stride + n[b]].tolist() for b in range(n_req)])

    def accept_and_commit(self, cap):
        toks = np.zeros(cap, np.int32)
        path = np.zeros(cap, np.int32)
        n = np.zeros(1, np.int32)
        self._check(self.lib.ss_accept_and_commit(self.ctx, _ptr(toks), _ptr(n), _ptr(path)))
        return toks[:n[0]].tolist(), path[:n[0]].tolist()

    def step(self, depth, top_k, sharpen_t):
        toks = np.zeros(depth + 1, np.int32)
        n = c_int32()
        self._check(self.lib.ss_step(self.ctx, ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)), _ptr(toks),
                                     ctypes.byref(n)))
        return toks[:n.value].tolist()

    def generate(self, prompt, max_new, depth, top_k, sharpen_t, chunk=256):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = np.zeros(max_new, np.int32)
        hist = np.zeros(depth + 2, np.int32)
        n = c_int32()
        self._check(self.lib.ss_generate(self.ctx, _ptr(p), len(p), max_new, chunk,
                                         ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)), _ptr(out),
                                         ctypes.byref(n), _ptr(hist)))
        return out[:n.value].tolist(), hist

    # ---- batched requests (NEXT-2) ---------------------------------------------------------
    def set_batch(self, n_req):
        self._check(self.lib.ss_set_batch(self.ctx, n_req))

    def prefill_slot(self, slot, prompt, chunk=256):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = c_int32()
        self._check(self.lib.ss_prefill_slot(self.ctx, slot, _ptr(p), len(p), chunk, ctypes.byref(out)))
        return out.value

    def step_batch(self, n_req, depth, top_k, sharpen_t):
        stride = depth + 1
        toks = np.zeros(n_req * stride, np.int32)
        n = np.zeros(n_req, np.int32)
        self._check(self.lib.ss_step_batch(self.ctx, ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)), stride,
                                           _ptr(toks), _ptr(n)))
        return [toks[b * stride: b * stride + n[b]].tolist() for b in range(n_req)]

    def generate_batch(self, prompts, max_new, depth, top_k, sharpen_t, chunk=256):
        lens = np.array([len(p) for p in prompts], np.int32)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts]), dtype=np.int32)
        B = len(prompts)
        out = np.zeros(B * max_new, np.int32)
        n = np.zeros(B, np.int32)
        hist = np.zeros(depth + 2, np.int32)
        self._check(self.lib.ss_generate_batch(self.ctx, B, _ptr(cat), _ptr(lens), max_new, chunk,
                                               ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)), _ptr(out),
                                               _ptr(n), _ptr(hist)))
        return [out[b * max_new: b * max_new + n[b]].tolist() for b in range(B)], hist

    def stats(self):
        s = StatsC()
        self._check(self.lib.ss_get_stats(self.ctx, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in StatsC._fields_}

    def reset_stats(self):
        self._check(self.lib.ss_reset_stats(self.ctx))

    # ---- NEXT-1: cooperative weight streaming (see ss_coop_export / ss_coop_enable) ---------
    def coop_export(self):
        """This rank's 256-byte handle (bytes) for the other ranks."""
        buf = (ctypes.c_uint8 * 256)()
        self._check(self.lib.ss_coop_export(self.ctx, buf))
        return bytes(buf)

    def coop_enable(self, rank, handles):
        """handles: every rank's coop_export() bytes, in rank order.  The caller barriers afterwards."""
        world = len(handles)
        arr = (ctypes.c_uint8 * (256 * world))()
        for h, b in enumerate(handles):
            if len(b) != 256:
                raise ValueError("coop handle must be 256 bytes")
            ctypes.memmove(ctypes.byref(arr, 256 * h), b, 256)
        self._check(self.lib.ss_coop_enable(self.ctx, rank, world, arr))

    def coop_finish(self):
        """Every rank, at a common point; the caller barriers afterwards."""
        self._check(self.lib.ss_coop_finish(self.ctx))

    # ---- debug / parity -----------------------------------------------------------------
    def debug_gen_tensor(self, seed, tid, shape, kind, sigma):
        rows, cols = (shape[0], shape[1]) if len(shape) == 2 else (1, shape[0])
        out = np.zeros(rows * cols, np.uint16)
        self._check(self.lib.ss_debug_gen_tensor(self.ctx, c_uint64(seed), tid, rows, cols,
                                                 {"mat": 0, "gain": 1, "bias": 2}[kind], sigma, _ptr(out)))
        return out.reshape(shape)

    def group_shape(self, group):
        c = self.cfg
        return [(c.qkv_rows, c.hidden), (c.hidden, c.q_dim), (2 * c.ffn, c.hidden), (c.hidden, c.ffn)][group]

    def debug_read_group(self, layer, group):
        N, K = self.group_shape(group)
        out = np.zeros(N * K, np.uint16)
        self._check(self.lib.ss_debug_read_group(self.ctx, layer, group, _ptr(out)))
        return out.reshape(N, K)

    def debug_get_substitute(self, layer, group):
        N, K = self.group_shape(group)
        codes = np.zeros(N * K, np.uint8)
        s = np.zeros(N * K // 64, np.uint16)
        z = np.zeros(N * K // 64, np.uint16)
        self._check(self.lib.ss_debug_get_substitute(self.ctx, layer, group, _ptr(codes), _ptr(s), _ptr(z)))
        return codes.reshape(N, K), s.reshape(N, K // 64), z.reshape(N, K // 64)

    def debug_matmul(self, which, layer, group, x_bits):
        N, K = self.group_shape(group)
        x = np.ascontiguousarray(x_bits, dtype=np.uint16)
        M = x.shape[0]
        y = np.zeros(M * N, np.float32)
        self._check(self.lib.ss_debug_matmul(self.ctx, which, layer, group, _ptr(x), M, _ptr(y)))
        return y.reshape(M, N)

    def debug_forward(self, which, tokens, parents, hidden=False):
        """tokens/parents [n] (or [B][n] with B active slots) -> logits [n, V] (or [B, n, V]);
        hidden=True also returns the final normed hidden rows [.., n, hidden]."""
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        p = np.ascontiguousarray(parents, dtype=np.int32)
        n = t.shape[-1]
        rows = t.size
        out = np.zeros(rows * self.cfg.vocab, np.float32)
        hid = np.zeros(rows * self.cfg.hidden, np.float32) if hidden else None
        self._check(self.lib.ss_debug_forward(self.ctx, which, _ptr(t), _ptr(p), n, _ptr(out), _ptr(hid)))
        shape = t.shape
        lg = out.reshape(*shape, self.cfg.vocab)
        return (lg, hid.reshape(*shape, self.cfg.hidden)) if hidden else lg

    def debug_set_tree(self, tokens, parents, top_k):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        p = np.ascontiguousarray(parents, dtype=np.int32)
        self._check(self.lib.ss_debug_set_tree(self.ctx, _ptr(t), _ptr(p), len(t), top_k))

    def debug_read_kv(self, layer, pos0, n):
        """Committed K/V rows: bf16 bit patterns (uint16), or float32 values in SS_FP32 mode."""
        c = self.cfg
        k = np.zeros(c.n_kv_heads * n * c.head_dim, np.float32 if self.precision == SS_FP32 else np.uint16)
        v = np.zeros_like(k)
        self._check(self.lib.ss_debug_read_kv(self.ctx, layer, pos0, n, _ptr(k), _ptr(v)))
        return k.reshape(c.n_kv_heads, n, c.head_dim), v.reshape(c.n_kv_heads, n, c.head_dim)

    def debug_decode_group(self, layer, group):
        """(natural [N x K] bf16 bits as the verify's GPU decoder produces them, codec mode, streamed bytes)."""
        N, K = self.group_shape(group)
        out = np.zeros(N * K, np.uint16)
        mode, nb = c_int32(), c_uint64()
        self._check(self.lib.ss_debug_decode_group(self.ctx, layer, group, _ptr(out), ctypes.byref(mode), ctypes.byref(nb)))
        return out.reshape(N, K), mode.value, nb.value

    def debug_read_draft_kv(self, layer, pos0, n):
        """The draft's own committed K/V rows (separate_draft_kv contexts), bf16 bit patterns."""
        c = self.cfg
        k = np.zeros(c.n_kv_heads * n * c.head_dim, np.uint16)
        v = np.zeros_like(k)
        self._check(self.lib.ss_debug_read_draft_kv(self.ctx, layer, pos0, n, _ptr(k), _ptr(v)))
        return k.reshape(c.n_kv_heads, n, c.head_dim), v.reshape(c.n_kv_heads, n, c.head_dim)

    def debug_time_pass(self, M, iters=5, skip=0):
        ms = c_float()
        self._check(self.lib.ss_debug_time_pass(self.ctx, M, iters, skip, ctypes.byref(ms)))
        return ms.value

    def debug_trace_pass(self, M, cap=256):
        out = np.zeros(cap * 16, np.int64)
        n = c_int32()
        self._check(self.lib.ss_debug_trace_pass(self.ctx, M, _ptr(out), cap, ctypes.byref(n)))
        return out[: n.value * 16].reshape(n.value, 16)

    def debug_step_timeline(self, depth, top_k, sharpen_t, cap=1024):
        """One step with events around each streamed group: (rows [n, 8], phases [3]); see subspec.h."""
        out = np.zeros(cap * 8, np.float64)
        ph = np.zeros(3, np.float64)
        n = c_int32()
        self._check(self.lib.ss_debug_step_timeline(self.ctx, ctypes.byref(DraftParamsC(depth, top_k, sharpen_t)),
                                                    _ptr(out), cap, ctypes.byref(n), _ptr(ph)))
        return out[:n.value * 8].reshape(-1, 8), ph

    def debug_cta_trace(self, M, launch, cap=1024):
        out = np.zeros(cap * 5, np.int64)
        n = c_int32()
        self._check(self.lib.ss_debug_cta_trace(self.ctx, M, launch, _ptr(out), cap, ctypes.byref(n)))
        return out[: n.value * 5].reshape(n.value, 5)

    def debug_set_knob(self, knob, value):
        self._check(self.lib.ss_debug_set_knob(self.ctx, knob, value))

    def debug_time_matmul(self, layer, group, M, iters=20, which=0):
        ms = c_float()
        self._check(self.lib.ss_debug_time_matmul(self.ctx, which, layer, group, M, iters, ctypes.byref(ms)))
        return ms.value
