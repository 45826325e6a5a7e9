// K6 — dense bf16 GEMM for verification / prefill (M = 1 + kD tree nodes, or a prefill chunk).
// Y[M x N] = X[M x K] * W^T over staged (streamed) or resident bf16 weights,
// fused epilogues incl. the K8 per-tile argmax for the head (logits never written to HBM).
//
// gemm_tc_kernel (default): 5th-generation tensor cores.  A CTA owns 128 weight rows x 128 tokens;
// its accumulator is a 128-lane x 128-column fp32 region of TMEM.  Warp 0 is the producer: each
// stage is one 128-k chunk (32 KB of weights + 32 KB of activations, both already in the canonical
// core-matrix layout, two cp.async.bulk copies); warp 1's
// elected lane issues eight tcgen05.mma (M = 128, N = 128, K = 16, A and B from shared memory) per
// stage and commits them to the stage's "empty" mbarrier.  Narrow matrices split K over a cluster of
// S CTAs (S from (N, K) and the SM count only); the ranks push their partial columns into the owners'
// shared memory (distributed shared memory) and each owner sums them in rank order, then runs the
// fused epilogue for its 128 / S tokens.
// Batch invariance: every launch uses the same MMA shape (N = 128) and the same K split for a given
// matrix, so each output element's reduction order does not depend on M: a node's logits in a
// 289-node verify equal an AR step's bitwise.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "gemv_core.cuh"

namespace ss {

constexpr int kGemmConsumerWarps = 8;
constexpr int kGemmThreads = (kGemmConsumerWarps + 1) * 32;
constexpr int kGemmTokNT = 16;                                // 128 tokens per CTA
constexpr int kGemmXBytes = kGemmTokNT * kXChunkBytesPerNT;   // 32 KB
constexpr int kGemmStageBytes = kBF16TileBytes + kGemmXBytes; // 64 KB
constexpr int kGemmStages = 3;
constexpr int kGemmSmem = kGemmStages * kGemmStageBytes + 2 * kGemmStages * 8 + 64;

// legacy mma.sync kernel (ss_debug_set_knob 2 = 1): 128 x 128 tiles, ldmatrix operands
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_kernel(const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGemmStages * kGemmStageBytes);
  uint64_t* empty = full + kGemmStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = p.tile0 + int(blockIdx.x), tt = blockIdx.y;   // r: the matrix's row tile (epilogue)
  const int nC = p.K >> 7;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemmConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* wbase = p.W + int64_t(r - p.tile0) * nC * kBF16TileBytes;
  if (warp == kGemmConsumerWarps) {
    if (lane == 0) {
      const int pre = nC < kGemmStages ? nC : kGemmStages;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], kGemmStageBytes);
        bulk_g2s(ring + i * kGemmStageBytes, wbase + int64_t(i) * kBF16TileBytes, kBF16TileBytes, &full[i]);
      }
      griddep_wait();
      for (int i = 0; i < pre; ++i)
        bulk_g2s(ring + i * kGemmStageBytes + kBF16TileBytes,
                 p.X + (int64_t(i) * p.NT + tt * kGemmTokNT) * 1024, kGemmXBytes, &full[i]);
      for (int i = pre; i < nC; ++i) {
        const int s = i % kGemmStages;
        mbar_wait(&empty[s], uint32_t(i / kGemmStages - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kGemmStageBytes);
        bulk_g2s(ring + s * kGemmStageBytes, wbase + int64_t(i) * kBF16TileBytes, kBF16TileBytes, &full[s]);
        bulk_g2s(ring + s * kGemmStageBytes + kBF16TileBytes, p.X + (int64_t(i) * p.NT + tt * kGemmTokNT) * 1024,
                 kGemmXBytes, &full[s]);
      }
    }
  } else {
    griddep_wait();
    const int g = lane >> 2, t4 = lane & 3;
    float acc[kGemmTokNT][4];
#pragma unroll
    for (int j = 0; j < kGemmTokNT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int i = 0; i < nC; ++i) {
      const int s = i % kGemmStages;
      mbar_wait(&full[s], uint32_t(i / kGemmStages) & 1);
      const uint32_t wst = smem_u32(ring + s * kGemmStageBytes);
      const uint32_t xst = wst + kBF16TileBytes;
      // lane L addresses row L % 8 of core matrix L / 8 (ldmatrix.x4)
      const int lq = lane >> 3, lr = lane & 7;
#pragma unroll
      for (int s2 = 0; s2 < 8; s2 += 2) {   // two k-steps of 16 per iteration
        uint32_t a[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)        // A: rows 16 warp .. +15 (row groups 2w, 2w+1), k-step s2 + h
          ldsm_x4(a[h][0], a[h][1], a[h][2], a[h][3], wst + core_off(2 * warp + (lq & 1), 2 * (s2 + h) + (lq >> 1), lr, 0));
#pragma unroll
        for (int j = 0; j < kGemmTokNT; ++j) {
          uint32_t b0, b1, b2, b3;           // B: token group j, k-steps s2 (b0, b1) and s2 + 1 (b2, b3)
          ldsm_x4(b0, b1, b2, b3, xst + core_off(j, 2 * s2 + lq, lr, 0));
          mma_bf16_16816(acc[j], a[0][0], a[0][1], a[0][2], a[0][3], b0, b1);
          mma_bf16_16816(acc[j], a[1][0], a[1][1], a[1][2], a[1][3], b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // all stages consumed and no copies outstanding: reuse the ring as the output tile
    asm volatile("bar.sync 1, %0;" ::"r"(kGemmConsumerWarps * 32) : "memory");
    float* tile = reinterpret_cast<float*>(ring);
    constexpr int ld = kGemmTokNT * 8 + 1;   // +1: conflict-free column scans in the argmax epilogue
#pragma unroll
    for (int j = 0; j < kGemmTokNT; ++j) {
      const int n0 = warp * 16 + g, m = j * 8 + 2 * t4;
      tile[n0 * ld + m] = acc[j][0];
      tile[n0 * ld + m + 1] = acc[j][1];
      tile[(n0 + 8) * ld + m] = acc[j][2];
      tile[(n0 + 8) * ld + m + 1] = acc[j][3];
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kGemmConsumerWarps * 32) : "memory");
    griddep_launch();
    apply_epilogue(p.epi, tile, ld, r, tt * 128, 128, threadIdx.x, kGemmConsumerWarps * 32);
  }
}


// ------------------------------- tcgen05 GEMM ---------------------------------------------------
// kFull = true (default): a stage is a whole 128-k chunk (32 KB of weights + 32 KB of activations, two
// contiguous bulk copies), 3 stages, one CTA per SM.  kFull = false (A/B variant 2): a stage is one
// 64-k half-chunk (16 KB + 16 KB as 32 one-KB bulk copies: the halves are not contiguous in the
// core-matrix layouts), 3 stages, two CTAs per SM — measured 1.8x slower at M = 289 (the 1 KB copies
// starve the tensor core).  Each splits K in the same units for every M (batch invariance, above).
constexpr int kTcThreads = 128;
constexpr int kTcStages = 3;
template <bool kFull>
struct TcCfg {
  static constexpr int kOpBytes = kFull ? 32768 : 16384;          // one operand of one stage
  static constexpr int kStageBytes = 2 * kOpBytes;
  static constexpr int kRingBytes = kTcStages * kStageBytes + 4096;   // + room for the S = 2 owner tile
  static constexpr int kSmem = kRingBytes + 128;
  static constexpr int kKSteps = kFull ? 8 : 4;                   // K = 16 MMAs per stage
  static constexpr uint32_t kSBO = kFull ? 2048 : 1024;           // row-group stride in the stage
  static constexpr int kUnitK = kFull ? 128 : 64;                 // K per stage
};
constexpr uint32_t kTcIdesc = umma_idesc_bf16(128);

template <bool kFull>
__global__ void __launch_bounds__(kTcThreads, kFull ? 1 : 2) gemm_tc_kernel(const GemmParams p) {
  using C = TcCfg<kFull>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRingBytes);
  uint64_t* empty = full + kTcStages;
  uint64_t* done = empty + kTcStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t S = cluster_nrank(), q = cluster_rank();
  const int tt = blockIdx.y, r = p.tile0 + int(blockIdx.z);   // r: the matrix's row tile (epilogue)
  const int nC = p.K >> 7, nU = p.K / C::kUnitK;
  const int h0 = int(int64_t(q) * nU / S), h1 = int(int64_t(q + 1) * nU / S), nh = h1 - h0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint8_t* wtile = p.W + int64_t(r - p.tile0) * nC * kBF16TileBytes;
  const uint8_t* xbase = reinterpret_cast<const uint8_t*>(p.X);
  // kFull: unit h = chunk h; weights 32 KB at chunk h of the row tile, activations 32 KB at
  // (h * NT + tt * 16) * 2 KB.  Half-chunks: row group g's 8 cores of half h % 2 are 1 KB at
  // g * 2048 + half * 1024 of chunk h / 2; token group tg's at ((c * NT + tg) * 16 + half * 8) * 128 B;
  // both land as core (g, kg') at (g * 8 + kg') * 128.
  auto w_src = [&](int h, int g) { return wtile + int64_t(h >> 1) * kBF16TileBytes + g * 2048 + (h & 1) * 1024; };
  auto x_src = [&](int h, int g) { return xbase + ((int64_t(h >> 1) * p.NT + tt * 16 + g) * 16 + (h & 1) * 8) * 128; };
  auto issue_w = [&](int st, int h) {
    if constexpr (kFull) {
      if (lane == 0) bulk_g2s(ring + st * C::kStageBytes, wtile + int64_t(h) * kBF16TileBytes, C::kOpBytes, &full[st]);
    } else {
      if (lane < 16) bulk_g2s(ring + st * C::kStageBytes + lane * 1024, w_src(h, lane), 1024, &full[st]);
    }
  };
  auto issue_x = [&](int st, int h) {
    if constexpr (kFull) {
      if (lane == 0)
        bulk_g2s(ring + st * C::kStageBytes + C::kOpBytes, xbase + (int64_t(h) * p.NT + tt * 16) * 2048, C::kOpBytes, &full[st]);
    } else {
      if (lane < 16) bulk_g2s(ring + st * C::kStageBytes + C::kOpBytes + lane * 1024, x_src(h, lane), 1024, &full[st]);
    }
  };
  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    const int pre = nh < kTcStages ? nh : kTcStages;
    for (int i = 0; i < pre; ++i) {   // weights of the first stages: independent of the previous kernel
      if (lane == 0) mbar_arrive_expect_tx(&full[i], C::kStageBytes);
      __syncwarp();
      issue_w(i, h0 + i);
    }
    griddep_wait();
    for (int i = 0; i < pre; ++i) issue_x(i, h0 + i);
    for (int i = pre; i < nh; ++i) {
      const int s = i % kTcStages;
      mbar_wait(&empty[s], uint32_t(i / kTcStages - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], C::kStageBytes);
      __syncwarp();
      if constexpr (kFull) {
        issue_w(s, h0 + i);
        issue_x(s, h0 + i);
      } else {
        uint8_t* dst = ring + s * C::kStageBytes + lane * 1024;
        if (lane < 16)
          bulk_g2s(dst, w_src(h0 + i, lane), 1024, &full[s]);
        else
          bulk_g2s(dst, x_src(h0 + i, lane - 16), 1024, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (elected lane) ------------------------------
    const uint32_t ring0 = smem_u32(ring);
    for (int i = 0; i < nh; ++i) {
      const int s = i % kTcStages;
      mbar_wait(&full[s], uint32_t(i / kTcStages) & 1);
      tc_fence_after();
      const uint64_t wd = umma_desc(ring0 + s * C::kStageBytes, 128, C::kSBO);
      const uint64_t xd = umma_desc(ring0 + s * C::kStageBytes + C::kOpBytes, 128, C::kSBO);
#pragma unroll
      for (int kk = 0; kk < C::kKSteps; ++kk)   // K = 16 per MMA: two cores = 256 B = 16 descriptor units
        umma_ss_w(tbase, wd + uint64_t(kk * 16), xd + uint64_t(kk * 16), kTcIdesc, (i > 0 || kk > 0) ? 1u : 0u);
      umma_commit_w(&empty[s]);
    }
    umma_commit_w(done);
  }
  // ------------------------------ epilogue (all four warps) ------------------------------
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  griddep_launch();
  const int n = 32 * warp + lane;                       // weight row of this thread (TMEM lane)
  const uint32_t tl = tbase + (uint32_t(32 * warp) << 16);
  float* tile = reinterpret_cast<float*>(ring);
  if (S == 1) {
    constexpr int ld = 129;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tl + c0, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[n * ld + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 128);
    apply_epilogue(p.epi, tile, ld, r, tt * 128, 128, threadIdx.x, kTcThreads);
    return;
  }
  // split-K over the cluster: owner o of token columns [o T, o T + T), T = 128 / S; rank q pushes its
  // partial columns into staging[q][mm][n] of the owner (after every rank's ring is drained)
  const int T = 128 / int(S);
  cluster_sync_all();
#pragma unroll 1
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tl + c0, v);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = c0 + j, o = m / T, mm = m - o * T;
      uint32_t a = smem_u32(tile + (int(q) * T + mm) * 128 + n), ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(uint32_t(o)));
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "r"(v[j]) : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();   // every push landed
  if (warp == 1) tmem_dealloc(tbase, 128);
  const int ld = T + 1;
  float* otile = tile + int(S) * T * 128;   // [128][T + 1] after the S x T x 128 staging
  for (int it = threadIdx.x; it < 128 * T; it += kTcThreads) {
    const int nn = it % 128, mm = it / 128;
    float acc = tile[mm * 128 + nn];
    for (int qq = 1; qq < int(S); ++qq) acc += tile[(qq * T + mm) * 128 + nn];
    otile[nn * ld + mm] = acc;
  }
  __syncthreads();
  apply_epilogue(p.epi, otile, ld, r, tt * 128 + int(q) * T, T, threadIdx.x, kTcThreads);
}

// K split of a matrix: the smallest S in {1, 2, 4, 8} with (N / 128) * S >= the SM count, keeping
// >= 4 chunks (512 k) per rank.  Depends on (N, K, device) only — never on M.
int gemm_tc_split(int N, int K, int sms) {
  int S = 1;
  while (S < 8 && (N / 128) * S < sms && (K / 128) / (2 * S) >= 4) S *= 2;
  return S;
}

void launch_gemm(const GemmParams& p, bool pdl, cudaStream_t st, int variant) {
  static unsigned long long init_mask = 0;   // function attributes are per device
  static int sms_of[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(init_mask >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
    cudaFuncSetAttribute(gemm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<false>::kSmem);
    cudaFuncSetAttribute(gemm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<true>::kSmem);
    cudaDeviceGetAttribute(&sms_of[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    init_mask |= 1ull << (dev & 63);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.stream = st;
  if (variant == 1) {
    cfg.gridDim = dim3(p.N / 128, (p.NT * 8) / 128);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kGemmSmem;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, gemm_kernel, p);
    return;
  }
  const int S = gemm_tc_split(p.split_n > 0 ? p.split_n : p.N, p.K, sms_of[dev & 63]);   // the whole matrix's plan
  cfg.gridDim = dim3(S, (p.NT * 8) / 128, p.N / 128);
  cfg.blockDim = dim3(kTcThreads);
  const bool fullc = variant != 2;   // whole-chunk stages unless the half-chunk A/B variant
  cfg.dynamicSmemBytes = fullc ? TcCfg<true>::kSmem : TcCfg<false>::kSmem;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = S;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (fullc)
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<true>, p);
  else
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<false>, p);
}

}  // namespace ss
