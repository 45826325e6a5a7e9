"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no quantizer, no forward, no
tree search).  It only fixes:
  * model shape presets (`configs`),
  * the counter-based weight generator (`weights`),
    which the CUDA library re-implements independently (csrc/gen.cu) — the
    two are pinned against each other by bitwise checksums,
  * the MT-Bench-shaped synthetic prompt recipe (`prompts`).
"""
