import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth.configs import SMALL
from oracle.quant import quantize, dequantize
from oracle.numerics import bf16_bits_to_f64
from paper_2509_18344_b200.binding import SubSpec
cfg = SMALL
ss = SubSpec(cfg, 512 << 20, max_depth=4, max_top_k=6, max_chunk=256)
ss.load_weights(0x5EED, n_resident=1); ss.build_substitutes()
g = 3
N, K = ss.group_shape(g)
what = dequantize(*quantize(bf16_bits_to_f64(ss.debug_read_group(1, g))))
for rep in range(3):
    for k0 in range(0, K, 32):
        x = np.zeros((32, K), np.uint16)
        for m in range(32): x[m, k0 + m] = 0x3F80
        y = ss.debug_matmul(0, 1, g, x).astype(np.float64)
        ref = what[:, k0:k0+32].T
        bad = np.argwhere(y != ref)
        if len(bad):
            ms = sorted(set(bad[:, 0].tolist())); ns = sorted(set(bad[:, 1].tolist()))
            print(f"rep {rep} k0 {k0}: {len(bad)} bad; m {ms[:10]} n tiles {sorted(set(n//128 for n in ns))} n {ns[:8]}")
            m0, n0 = bad[0]
            print("   y", y[m0, n0], "ref", ref[m0, n0], "y-ref", y[m0,n0]-ref[m0,n0], "x2?", y[m0,n0]/ref[m0,n0] if ref[m0,n0] else None)
print("done")
