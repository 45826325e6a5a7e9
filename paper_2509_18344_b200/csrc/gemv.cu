// K2 — fused dequant-GEMV/GEMM for the draft (M = frontier tokens <= 32).
// Y[M x N] = X[M x K] * W_hat^T with W_hat = RNE_bf16(code*s + z)
// ("low-bit GEMM kernels"; 4 bit / group 64).
//
// B200 design:
//  * persistent grid (one CTA per SM); the (row-tile, k-chunk) space of 128x128 tile-chunks is
//    split into equal contiguous ranges per CTA (Stream-K); because the weight layout is
//    tile-chunk contiguous, a CTA streams ONE contiguous byte range;
//  * a producer warp streams tile-chunks with cp.async.bulk (TMA engine) into an S-stage
//    shared-memory ring guarded by mbarriers; the weight part of the first stages is issued
//    BEFORE griddepcontrol.wait, overlapping the previous kernel (PDL);
//  * 8 consumer warps dequantise 4-bit codes in registers (lop3 + sub + fma.bf16x2) straight
//    into mma.m16n8k16 A fragments (weights as the 16-row A operand, tokens as N = 8..32);
//  * row tiles split across CTAs are reduced deterministically by the last-arriving CTA in
//    fixed slot order, which then runs the fused epilogue (bias+RoPE+KV write / residual /
//    SiLU*mul / logits).
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace ss {

constexpr int kGemvConsumerWarps = 8;
constexpr int kGemvThreads = (kGemvConsumerWarps + 1) * 32;

template <bool Q4, int NT>
struct GemvCfg {
  static constexpr int kWBytes = Q4 ? kQ4TileBytes : kBF16TileBytes;
  static constexpr int kXBytes = NT * kXChunkBytesPerNT;
  static constexpr int kStageBytes = kWBytes + kXBytes;
  static constexpr int kRingBudget = 88 * 1024;   // 2 CTAs/SM: this kernel + the next (PDL)
  static constexpr int kStages = (kRingBudget / kStageBytes) < 2 ? 2 : (kRingBudget / kStageBytes > 8 ? 8 : kRingBudget / kStageBytes);
  static constexpr int kTileFloats = kTileRows * NT * 8;
  static constexpr int kSmem = kStages * kStageBytes + kTileFloats * 4 + 2 * kStages * 8 + 64;
};

SS_HD int64_t owner_of(int64_t t, int64_t T, int G) { return ((t + 1) * G - 1) / T; }

static int gemv_grid_for(int N, int K, int grid) {
  const int64_t T = int64_t(N / 128) * (K / 128);
  return int(T < grid ? T : grid);   // every CTA gets >= 1 tile-chunk, so segment counts are exact
}

int gemv_max_segments(int N, int K, int grid) {
  int64_t nC = K / 128, T = int64_t(N / 128) * nC;
  grid = gemv_grid_for(N, K, grid);
  int mx = 1;
  for (int64_t r = 0; r < N / 128; ++r) {
    int s = int(owner_of((r + 1) * nC - 1, T, grid) - owner_of(r * nC, T, grid) + 1);
    if (s > mx) mx = s;
  }
  return mx;
}

SS_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <bool Q4, int NT>
__global__ void __launch_bounds__(kGemvThreads, 2) gemv_kernel(const GemvParams p) {
  using C = GemvCfg<Q4, NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  float* otile = reinterpret_cast<float*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes + C::kTileFloats * 4);
  uint64_t* empty = full + C::kStages;
  int* flag = reinterpret_cast<int*>(empty + C::kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nC = p.K >> 7;
  const int64_t T = int64_t(p.N >> 7) * nC;
  const int G = gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * T / G, hi = int64_t(blockIdx.x + 1) * T / G;
  const int Mpad = NT * 8;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch();   // all CTAs are resident (grid <= #SMs): let the next kernel prefetch now

  if (warp == kGemvConsumerWarps) {
    // ------------------------------ producer -------------------------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int64_t n = hi - lo;
      const int pre = int(n < C::kStages ? n : C::kStages);
      // weights do not depend on the previous kernel: issue before the grid-dependency wait
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], C::kStageBytes);
        bulk_g2s_hint(ring + i * C::kStageBytes, p.W + (lo + i) * C::kWBytes, C::kWBytes, &full[i], pol);
      }
      griddep_wait();
      for (int i = 0; i < pre; ++i) {
        const int c = int((lo + i) % nC);
        bulk_g2s(ring + i * C::kStageBytes + C::kWBytes, p.X + int64_t(c) * NT * 1024, C::kXBytes, &full[i]);
      }
      for (int64_t i = pre; i < n; ++i) {
        const int s = int(i % C::kStages);
        const uint32_t ph = uint32_t((i / C::kStages) - 1) & 1;
        mbar_wait(&empty[s], ph);
        const int c = int((lo + i) % nC);
        mbar_arrive_expect_tx(&full[s], C::kStageBytes);
        bulk_g2s_hint(ring + s * C::kStageBytes, p.W + (lo + i) * C::kWBytes, C::kWBytes, &full[s], pol);
        bulk_g2s(ring + s * C::kStageBytes + C::kWBytes, p.X + int64_t(c) * NT * 1024, C::kXBytes, &full[s]);
      }
    }
    return;
  }

  // ------------------------------ consumers --------------------------------
  griddep_wait();
  const int g = lane >> 2, t4 = lane & 3;
  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  auto flush = [&](int64_t r, int64_t c_first, int64_t c_last) {
    // c_first..c_last: chunks of row tile r handled by this CTA
    const bool complete = (c_first == 0 && c_last == nC - 1);
    float* dst;
    int ld;
    int64_t slot = 0, nseg = 1, first = 0;
    if (complete) {
      dst = otile;
      ld = Mpad;
    } else {
      first = owner_of(r * nC, T, G);
      nseg = owner_of((r + 1) * nC - 1, T, G) - first + 1;
      slot = blockIdx.x - first;
      dst = p.partials + (r * p.max_seg + slot) * int64_t(kTileRows * Mpad);
      ld = Mpad;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n0 = warp * 16 + g, m = j * 8 + 2 * t4;
      dst[n0 * ld + m] = acc[j][0];
      dst[n0 * ld + m + 1] = acc[j][1];
      dst[(n0 + 8) * ld + m] = acc[j][2];
      dst[(n0 + 8) * ld + m + 1] = acc[j][3];
      acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    }
    const int ctid = threadIdx.x, nthr = kGemvConsumerWarps * 32;
    if (!complete) {
      __threadfence();
      named_bar(1, nthr);
      if (ctid == 0) {
        const int old = atomicAdd(&p.counters[r], 1);
        *flag = (old == nseg - 1);
      }
      named_bar(1, nthr);
      if (!*flag) return;
      __threadfence();
      const float* base = p.partials + r * p.max_seg * int64_t(kTileRows * Mpad);
      for (int e = ctid; e < kTileRows * Mpad; e += nthr) {
        float s = 0.f;
        for (int q = 0; q < nseg; ++q) s += __ldcg(base + q * int64_t(kTileRows * Mpad) + e);
        otile[e] = s;
      }
      if (ctid == 0) p.counters[r] = 0;
    }
    named_bar(1, nthr);
    apply_epilogue(p.epi, otile, Mpad, int(r), 0, Mpad, ctid, nthr);
    named_bar(1, nthr);
  };

  int64_t cur_r = lo / nC, c_first = lo % nC;
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t r = i / nC;
    const int c = int(i % nC);
    if (r != cur_r) {
      flush(cur_r, c_first, nC - 1);
      cur_r = r;
      c_first = c;
    }
    const int s = int((i - lo) % C::kStages);
    const uint32_t ph = uint32_t((i - lo) / C::kStages) & 1;
    mbar_wait(&full[s], ph);
    const uint8_t* wst = ring + s * C::kStageBytes;
    const uint8_t* xst = wst + C::kWBytes;
    if constexpr (Q4) {
      const uint4 c0 = *reinterpret_cast<const uint4*>(wst + ((warp * 2 + 0) * 32 + lane) * 16);
      const uint4 c1 = *reinterpret_cast<const uint4*>(wst + ((warp * 2 + 1) * 32 + lane) * 16);
      const uint32_t m0 = *reinterpret_cast<const uint32_t*>(wst + kQ4CodeBytes + ((warp * 2 + (t4 >> 1)) * 16 + g) * 4);
      const uint32_t m1 = *reinterpret_cast<const uint32_t*>(wst + kQ4CodeBytes + ((warp * 2 + (t4 >> 1)) * 16 + g + 8) * 4);
      const uint32_t s0 = (m0 & 0xFFFFu) * 0x10001u, z0 = (m0 >> 16) * 0x10001u;
      const uint32_t s1 = (m1 & 0xFFFFu) * 0x10001u, z1 = (m1 >> 16) * 0x10001u;
      const uint32_t w0[4] = {c0.x, c0.y, c0.z, c0.w};
      const uint32_t w1[4] = {c1.x, c1.y, c1.z, c1.w};
#pragma unroll
      for (int st = 0; st < 8; ++st) {
        const int pp = 2 * (st & 1);
        const uint32_t a0 = dq_pair(w0[st >> 1], pp, s0, z0);
        const uint32_t a1 = dq_pair(w1[st >> 1], pp, s1, z1);
        const uint32_t a2 = dq_pair(w0[st >> 1], pp + 1, s0, z0);
        const uint32_t a3 = dq_pair(w1[st >> 1], pp + 1, s1, z1);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint2 b = *reinterpret_cast<const uint2*>(xst + ((((j * 8 + st) * 4 + t4) * 8 + g) * 8));
          mma_bf16_16816(acc[j], a0, a1, a2, a3, b.x, b.y);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r0 = *reinterpret_cast<const uint4*>(wst + (((warp * 2 + 0) * 4 + q) * 32 + lane) * 16);
        const uint4 r1 = *reinterpret_cast<const uint4*>(wst + (((warp * 2 + 1) * 4 + q) * 32 + lane) * 16);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int st = 2 * q + hh;
          const uint32_t a0 = hh ? r0.z : r0.x, a2 = hh ? r0.w : r0.y;
          const uint32_t a1 = hh ? r1.z : r1.x, a3 = hh ? r1.w : r1.y;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint2 b = *reinterpret_cast<const uint2*>(xst + ((((j * 8 + st) * 4 + t4) * 8 + g) * 8));
            mma_bf16_16816(acc[j], a0, a1, a2, a3, b.x, b.y);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (hi > lo) flush(cur_r, c_first, (hi - 1) % nC);
}

template <bool Q4, int NT>
static void launch_t(const GemvParams& p, int grid, bool pdl, cudaStream_t st) {
  using C = GemvCfg<Q4, NT>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(gemv_kernel<Q4, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, gemv_kernel<Q4, NT>, p);
}

void launch_gemv(bool q4, const GemvParams& p, int grid, bool pdl, cudaStream_t st) {
  grid = gemv_grid_for(p.N, p.K, grid);
  switch (p.NT) {
    case 1: q4 ? launch_t<true, 1>(p, grid, pdl, st) : launch_t<false, 1>(p, grid, pdl, st); break;
    case 2: q4 ? launch_t<true, 2>(p, grid, pdl, st) : launch_t<false, 2>(p, grid, pdl, st); break;
    case 4: q4 ? launch_t<true, 4>(p, grid, pdl, st) : launch_t<false, 4>(p, grid, pdl, st); break;
    default: break;
  }
}

}  // namespace ss
