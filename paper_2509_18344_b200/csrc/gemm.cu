// K6 — dense bf16 GEMM for verification / prefill (M = 1 + kD tree nodes, or a prefill chunk).
// Y[M x N] = X[M x K] * W^T over staged (streamed) or resident bf16 weights,
// fused epilogues incl. the K8 per-tile argmax for the head (logits never written to HBM).
// Each output element reduces over K in a fixed order independent of M (no split-K), so the
// target path is batch-invariant: a node's logits are bitwise those of an AR step.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace ss {

constexpr int kGemmConsumerWarps = 8;
constexpr int kGemmThreads = (kGemmConsumerWarps + 1) * 32;
constexpr int kGemmTokNT = 16;                                // 128 tokens per CTA
constexpr int kGemmXBytes = kGemmTokNT * kXChunkBytesPerNT;   // 32 KB
constexpr int kGemmStageBytes = kBF16TileBytes + kGemmXBytes; // 64 KB
constexpr int kGemmStages = 3;
constexpr int kGemmSmem = kGemmStages * kGemmStageBytes + 2 * kGemmStages * 8 + 64;

__global__ void __launch_bounds__(kGemmThreads, 1) gemm_kernel(const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGemmStages * kGemmStageBytes);
  uint64_t* empty = full + kGemmStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x, tt = blockIdx.y;
  const int nC = p.K >> 7;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemmConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* wbase = p.W + int64_t(r) * nC * kBF16TileBytes;
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

void launch_gemm(const GemmParams& p, bool pdl, cudaStream_t st) {
  static unsigned long long init_mask = 0;   // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(init_mask >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
    init_mask |= 1ull << (dev & 63);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.N / 128, (p.NT * 8) / 128);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = kGemmSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, gemm_kernel, p);
}

}  // namespace ss
