"""One small SubSpec run for compute-sanitizer (tiny shape with one offloaded + streamed layer, the
eager and the CUDA-graph draft path, D = 4, k = 6): every kernel of the step launches at least once
(K1 quantizer, K2 cluster split-K + Stream-K GEMVs, tcgen05 head GEMV + EPI_TOPK, K3, K6 tcgen05
verify GEMM, K7 copy ring + zdecode, K8, K9).  tools/sanitize.sh runs it under memcheck, racecheck,
synccheck and initcheck."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import TINY
from synth.prompts import mtbench_prompt
from paper_2509_18344_b200.binding import SubSpec

graphs = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ss = SubSpec(TINY, 256 << 20, device=0, max_depth=4, max_top_k=6, max_chunk=256, cuda_graphs=graphs)
ss.load_synthetic(0x5EED, n_resident=1)
ss.build_substitutes(4, 64)
prompt = mtbench_prompt(0x5EED, 0, TINY.vocab, 40)
out, _ = ss.generate(prompt, 12, depth=4, top_k=6, sharpen_t=0.2)
print("sanitize run ok:", out)
ss.close()
