"""ORACLE — test infrastructure only.

A plain, slow, CPU implementation (NumPy, float64) of what one SubSpec
tree-speculative decode step computes (arXiv 2509.18344; §4, Fig. 3,
Eq. 2).  It shares no code with the CUDA path in
`paper_2509_18344_b200/` and never imports it.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import anything under `oracle/`.  The product path never routes
through here.

Modules
  numerics  bf16 round-to-nearest-even from float64, RMSNorm, RoPE, SiLU
  quant     O.2  RTN min/max group quantizer (4-bit, group 64) and dequantizer
  model     O.3  forward of a set of tree nodes with the ancestor-closure mask
  tree      O.4  tempered log-softmax scoring and global top-k tree growth
  verify    O.5-O.7 target argmax, greedy acceptance walk, KV commit
  decode    O.8-O.10 AR reference, chunked prefill, the SD loop with capacity clamp

Pins (tests/test_oracle_*.py): PAPER/SPEC worked examples (quantizer ramp,
Fig. 4 false-positive path, tempered-softmax examples, accept hand examples),
brute-force enumeration of tree selection and acceptance, chain == sequential
and path-replay bitwise identities, a torch-CPU library cross-check of the
forward (scaled_dot_product_attention / rms_norm / silu), and the greedy
lossless invariant SD == AR.  "parity unpinned": only the magnitude of tau on
random weights (no paper number applies to synthetic weights).
"""
