"""Model shape presets (SURVEY.md §8 "Model shapes"; BASELINE.json configs).

Shapes only — the paper names the models but not their
dimensions; the numbers below are the public config.json values [EXT].
"""
from dataclasses import dataclass, asdict, replace


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    max_context: int = 2048          # static KV-cache
    rope_theta: float = 1e6
    rms_eps: float = 1e-6
    qkv_bias: bool = True

    @property
    def q_dim(self):
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self):
        return self.n_kv_heads * self.head_dim

    @property
    def qkv_rows(self):
        return self.q_dim + 2 * self.kv_dim

    def params_per_layer(self):
        return (self.qkv_rows * self.hidden + self.hidden * self.q_dim
                + 2 * self.ffn * self.hidden + self.hidden * self.ffn)

    def to_dict(self):
        return asdict(self)

    def with_(self, **kw):
        return replace(self, **kw)


# BJ config 1 (tiny random-init Llama-style model)
TINY = ModelConfig("tiny", n_layers=2, hidden=256, n_heads=4, n_kv_heads=2, head_dim=64,
                   ffn=768, vocab=1024, rope_theta=1e4, rms_eps=1e-6, qkv_bias=True)
# a mid-size parity config: head_dim 128, GQA 4:1, several 128-row tiles, ragged trees
SMALL = ModelConfig("small", n_layers=3, hidden=1024, n_heads=8, n_kv_heads=2, head_dim=128,
                    ffn=2816, vocab=4096, rope_theta=1e6, rms_eps=1e-6, qkv_bias=True)
QWEN7B = ModelConfig("qwen2.5-7b", n_layers=28, hidden=3584, n_heads=28, n_kv_heads=4, head_dim=128,
                     ffn=18944, vocab=152064, rope_theta=1e6, rms_eps=1e-6, qkv_bias=True)
LLAMA8B = ModelConfig("llama-3.1-8b", n_layers=32, hidden=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                      ffn=14336, vocab=128256, rope_theta=5e5, rms_eps=1e-5, qkv_bias=False)
QWEN32B = ModelConfig("qwen2.5-32b", n_layers=64, hidden=5120, n_heads=40, n_kv_heads=8, head_dim=128,
                      ffn=27648, vocab=152064, rope_theta=1e6, rms_eps=1e-6, qkv_bias=True)

PRESETS = {c.name: c for c in (TINY, SMALL, QWEN7B, LLAMA8B, QWEN32B)}

GIB = 1 << 30
