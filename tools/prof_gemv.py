"""Driver for ncu captures of the GEMV kernels at Qwen2.5-7B shapes (8 GiB cap, 0 resident).

Launch order (each debug_time_matmul call: L warm-up launches + L timed, L = 28): K2 gemv_q_kernel
qkv 0..55, gate_up 56..111, down 112..167, o 168..223; then the tcgen05 bf16 head (gemv_kernel) 0..5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import QWEN7B, GIB
from paper_2509_18344_b200.binding import SubSpec
M = int(sys.argv[1]) if len(sys.argv) > 1 else 6
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ss = SubSpec(QWEN7B, 8 * GIB, max_depth=48, max_top_k=6)
ss.load_synthetic(0x5EED, 0)
ss.build_substitutes(bits, 64)
for g in (0, 2, 3, 1):
    t = ss.debug_time_matmul(-1, g, M, iters=1)
    print("group", g, "us", t * 1e3, flush=True)
t = ss.debug_time_matmul(0, -1, M, iters=5)
print("head us", t * 1e3, flush=True)
