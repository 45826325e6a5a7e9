// K2 — the draft's 4-/2-bit substitute dequant-GEMV (M = frontier tokens <= 32) on the legacy tensor
// path (mma.sync).  SURVEY §8(a) A2c/g/h/i: Y[M x N] = X[M x K] * W_hat^T with W_hat = code*s + z per
// 64-group ("highly optimized low-bit GEMM kernels"; 4 bit / group 64, PAPER.md:278;
// reading R3 in DESIGN.md: the affine dequantisation is applied exactly, in fp32).
//
// B200 design:
//  * weights are tile-chunk contiguous (128 rows x 128 k, 9 KB for Q4): a CTA streams its work
//    with cp.async.bulk (TMA engine) into an S-stage shared-memory ring guarded by mbarriers; the
//    weight part of the first stages is issued BEFORE griddepcontrol.wait (PDL), overlapping the
//    previous kernel's tail;
//  * 8 consumer warps turn 4-bit codes into exact bf16 (128 + code) with ONE lop3 per pair and feed
//    them straight into mma.m16n8k16 as the 16-row A operand (tokens are N); the codes are stored in
//    A-fragment order (common.cuh), the activations' B fragments come from the core-matrix layout with
//    ldmatrix; every k-step stays inside one 64-group, the producers of X publish its 64-group sums,
//    and y += s*sum((128+c)x) + (z - 128 s)*sum(x) applies the group scale/zero in fp32;
//  * narrow matrices (qkv, o, down) use cluster split-K: the S CTAs of a cluster split a row tile's K
//    and reduce their partial tiles through distributed shared memory, in rank order, then run the
//    fused epilogue (bias+RoPE+KV write / residual + RMSNorm / SiLU*mul); tall ones use Stream-K.
// Why not tcgen05 here: a tcgen05 version (A dequantised into TMEM by converter warps, one thread
// issuing the MMAs into per-group TMEM accumulators, accumulator warps applying the affine) was built
// and measured: at M = 6 its per-chunk hand-offs (converter -> MMA issuer ->
// accumulator, each an mbarrier wake-up, plus ~13 instructions per tcgen05.mma issued from a
// sub-partition shared with busy warps) cap it at ~2.7 TB/s, below this register-resident design.
// The bf16 GEMV (head, resident layers: no dequantisation, no per-group affine) is on tcgen05 (gemv.cu).
#include "common.cuh"
#include "epilogue.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

namespace ss {

// Consumer warps per CTA.  16 (default): one CTA per SM, two warp groups, each warp two chunks of a
// four-chunk stage, a 220 KB ring (4 stages); measured per draft pass at Qwen2.5-7B, M = 6: 1976 us vs
// 2073 us for 8 warps at two CTAs per SM (88 KB rings), 2032 us for 24 warps (72 registers),
// 1999 us for 16 warps with 2-3 stages (tools/k2_variants.sh)
#ifndef SS_K2_CW
#define SS_K2_CW 16
#endif
#ifndef SS_K2_WCH
#define SS_K2_WCH 2           // tile-chunks per consumer warp per stage
#endif
#ifndef SS_K2_RING1_KB
#define SS_K2_RING1_KB 220    // shared-memory budget of the one-CTA-per-SM variants
#endif
constexpr int kGemvQConsumerWarps = SS_K2_CW;
constexpr int kGemvQThreads = (kGemvQConsumerWarps + 1) * 32;
constexpr int kGemvQGroups = kGemvQConsumerWarps / 8;   // warp groups: group q takes stage chunks q*WCH..
constexpr int kGemvQCtasPerSm = kGemvQGroups == 1 ? 2 : 1;

// NT: token groups of the activation layout; QB: code bits (4, 3 or 2); NTC: token groups the MMAs read
template <int NT, int QB, int NTC>
struct GemvQCfg {
  static constexpr int kCPS = kGemvQGroups * SS_K2_WCH;           // tile-chunks per pipeline stage
  static constexpr int kWBytes = QB == 2 ? kQ2TileBytes : (QB == 3 ? kQ3TileBytes : kQ4TileBytes);
  static constexpr int kCodeBytes = QB == 2 ? kQ2CodeBytes : (QB == 3 ? kQ3CodeBytes : kQ4CodeBytes);
  static constexpr int kXBytes = NT * kXChunkBytesPerNT;
  static constexpr int kSBytes = 2 * NT * 8 * 4;                  // group sums of x: [2 groups][Mpad] fp32
  static constexpr int kStageBytes = kCPS * (kWBytes + kXBytes + kSBytes);
  static constexpr int kMaxStages = 16;
  static constexpr int kTileFloats = kTileRows * NT * 8;
  static constexpr int kXPreTokens = 8;
  static constexpr int kXPreFloats = kXPreTokens * kTileRows;
  static constexpr int kStagingFloats = (NT * 8 + kGemvMaxCluster - 1) * kTileRows;
  static constexpr int kGPartFloats = kGemvQGroups > 1 ? kGemvQGroups * kTileFloats : 0;   // per-group partial tiles
  static constexpr int smem_for(int S) {
    return S * kStageBytes + kTileFloats * 4 + kStagingFloats * 4 + 2 * kMaxStages * 8 + 64 + 512 + kXPreFloats * 4 +
           kGPartFloats * 4;
  }
};

// One pipeline stage (nch tile-chunks of codes + the matching activation chunks + group sums)
// accumulated into this warp's 16 rows x 8 NTC tokens.
template <int NT, int NTC, int QB, int NCH>
SS_DEV void consume_n(const uint8_t* stage, int ci0, float (&acc)[NTC][4], int warp, int lane) {
  using C = GemvQCfg<NT, QB, NTC>;
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t kMagic = 0x43004300u;   // bf16x2 (128, 128)
  const int lq = lane >> 3, lr = lane & 7;   // ldmatrix: lane supplies row lr of core matrix lq
#pragma unroll
  for (int cc = 0; cc < NCH; ++cc) {
    const int ci = ci0 + cc;
    const uint8_t* wst = stage + ci * C::kWBytes;
    const uint32_t xst = smem_u32(stage + C::kCPS * C::kWBytes + ci * C::kXBytes);
    const float* xsum = reinterpret_cast<const float*>(stage + C::kCPS * (C::kWBytes + C::kXBytes) + ci * C::kSBytes);
#pragma unroll
    for (int G = 0; G < 2; ++G) {
      uint4 cw;
      uint32_t hw = 0u;          // Q3: the lane's high-bit word
      if constexpr (QB == 2 || QB == 3) {   // [row g word][row g+8 word]
        const uint2 c2 = *reinterpret_cast<const uint2*>(wst + ((warp * 2 + G) * 32 + lane) * 8);
        cw = make_uint4(c2.x, 0u, c2.y, 0u);
        if constexpr (QB == 3) hw = *reinterpret_cast<const uint32_t*>(wst + kQ2CodeBytes + ((warp * 2 + G) * 32 + lane) * 4);
      } else {                   // [row g: word0, word1][row g+8: word0, word1]
        cw = *reinterpret_cast<const uint4*>(wst + ((warp * 2 + G) * 32 + lane) * 16);
      }
      const uint32_t m0 = *reinterpret_cast<const uint32_t*>(wst + C::kCodeBytes + G * 512 + (warp * 16 + g) * 4);
      const uint32_t m1 = *reinterpret_cast<const uint32_t*>(wst + C::kCodeBytes + G * 512 + (warp * 16 + g + 8) * 4);
      // B fragments of the group's 4 k-steps, per computed token group: 2 ldmatrix.x4 (steps 0-1, 2-3)
      uint32_t b[NTC][8];
#pragma unroll
      for (int j = 0; j < NTC; ++j) {
        ldsm_x4(b[j][0], b[j][1], b[j][2], b[j][3], xst + core_off(j, 8 * G + lq, lr, 0));
        ldsm_x4(b[j][4], b[j][5], b[j][6], b[j][7], xst + core_off(j, 8 * G + 4 + lq, lr, 0));
      }
      // one accumulator chain per token tile (16 consumer warps per SM hide the MMA latency; two
      // chains per group measured slower)
      float cg[NTC][4];
#pragma unroll
      for (int j = 0; j < NTC; ++j) cg[j][0] = cg[j][1] = cg[j][2] = cg[j][3] = 0.f;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        uint32_t a0, a1, a2, a3;
        if constexpr (QB == 2 || QB == 3) {   // pairs 2 k4 (a0/a1) and 2 k4 + 1 (a2/a3) at bit 2p
          a0 = lop3_and_or2(cw.x >> (4 * k4), kMagic);
          a1 = lop3_and_or2(cw.z >> (4 * k4), kMagic);
          a2 = lop3_and_or2(cw.x >> (4 * k4 + 2), kMagic);
          a3 = lop3_and_or2(cw.z >> (4 * k4 + 2), kMagic);
          if constexpr (QB == 3) {   // high bits of pair p of row g + 8h: (hw >> (8h + p - 2)) & 0x00040004
            auto hb = [&](int sh) { return sh >= 0 ? hw >> sh : hw << (-sh); };
            a0 = lop3_and_or_hi(hb(2 * k4 - 2), a0);
            a1 = lop3_and_or_hi(hb(8 + 2 * k4 - 2), a1);
            a2 = lop3_and_or_hi(hb(2 * k4 - 1), a2);
            a3 = lop3_and_or_hi(hb(8 + 2 * k4 - 1), a3);
          }
        } else {
          const uint32_t wg = (k4 < 2) ? cw.x : cw.y, wg8 = (k4 < 2) ? cw.z : cw.w;
          const int pp = 2 * (k4 & 1);
          a0 = lop3_and_or(wg >> (4 * pp), kMagic);
          a1 = lop3_and_or(wg8 >> (4 * pp), kMagic);
          a2 = lop3_and_or(wg >> (4 * pp + 4), kMagic);
          a3 = lop3_and_or(wg8 >> (4 * pp + 4), kMagic);
        }
#pragma unroll
        for (int j = 0; j < NTC; ++j) mma_bf16_16816(cg[j], a0, a1, a2, a3, b[j][2 * k4], b[j][2 * k4 + 1]);
      }
      // y += s * sum((128 + c) x) + (z - 128 s) * sum(x)      (exact affine dequant, fp32)
      const float s0 = __uint_as_float(m0 << 16), z0 = __uint_as_float(m0 & 0xFFFF0000u);
      const float s1 = __uint_as_float(m1 << 16), z1 = __uint_as_float(m1 & 0xFFFF0000u);
      const float zz0 = fmaf(-128.0f, s0, z0), zz1 = fmaf(-128.0f, s1, z1);   // exact
#pragma unroll
      for (int j = 0; j < NTC; ++j) {
        const float2 xs = *reinterpret_cast<const float2*>(xsum + G * NT * 8 + j * 8 + 2 * t4);
        acc[j][0] = fmaf(s0, cg[j][0], fmaf(zz0, xs.x, acc[j][0]));
        acc[j][1] = fmaf(s0, cg[j][1], fmaf(zz0, xs.y, acc[j][1]));
        acc[j][2] = fmaf(s1, cg[j][2], fmaf(zz1, xs.x, acc[j][2]));
        acc[j][3] = fmaf(s1, cg[j][3], fmaf(zz1, xs.y, acc[j][3]));
      }
    }
  }
}

// warp w consumes chunks [q*WCH, q*WCH + WCH) of a stage (q = w / 8, its warp group) for row block
// w % 8; two chunks are one straight-line body (the scheduler interleaves both chunks' loads and MMA
// chains: -0.4% per draft pass vs a loop with an early exit); a short last stage takes fewer
template <int NT, int NTC, int QB>
SS_DEV void consume_q(const uint8_t* stage, int nch, float (&acc)[NTC][4], int warp, int lane) {
  const int c0 = (warp >> 3) * SS_K2_WCH, rb = warp & 7;
  const int n = nch - c0 < SS_K2_WCH ? nch - c0 : SS_K2_WCH;
  if constexpr (SS_K2_WCH == 2) {
    if (n == 2) consume_n<NT, NTC, QB, 2>(stage, c0, acc, rb, lane);
    else if (n == 1) consume_n<NT, NTC, QB, 1>(stage, c0, acc, rb, lane);
  } else {
    if (n >= 1) consume_n<NT, NTC, QB, 1>(stage, c0, acc, rb, lane);
  }
}

static int gemv_grid_for(int N, int K, int grid) {
  const int64_t T = int64_t(N / 128) * (K / 128);
  return int(T < grid ? T : grid);   // every Stream-K CTA gets >= 1 tile-chunk
}
static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
// split factor of the cluster mode: ~per_sm CTAs per SM (hint, default 2), <= 8 (portable), <= chunks
static int gemv_q_split(int N, int K, int sms, int hint) {
  const int tiles = N / 128, nC = K / 128;
  const int per_sm = hint > 0 ? hint : kGemvQCtasPerSm;
  int S = (per_sm * sms) / tiles;
  if (S < 1) S = 1;
  if (S > 8) S = 8;
  if (S > nC) S = nC;
  return S;
}

// accumulators -> [128 x Mpad] fp32 tile (row-major in n), then clear
// (token_major: [Mpad][128], the cluster reduction's layout).  With several warp groups each group
// writes its own partial tile to gpart and the copies are summed into dst in group order
// (deterministic); the caller's next named barrier orders dst for the other threads.
template <int NT, int NTC>
SS_DEV void stash_q(float (&acc)[NTC][4], float* dst, int warp, int lane, bool token_major, float* gpart, int tid,
                    int nthr) {
  const int g = lane >> 2, t4 = lane & 3, Mpad = NT * 8, rb = warp & 7;
  float* out = kGemvQGroups > 1 ? gpart + (warp >> 3) * (kTileRows * Mpad) : dst;
#pragma unroll
  for (int j = 0; j < NTC; ++j) {
    const int n0 = rb * 16 + g, m = j * 8 + 2 * t4;
    if (token_major) {
      out[m * kTileRows + n0] = acc[j][0];
      out[(m + 1) * kTileRows + n0] = acc[j][1];
      out[m * kTileRows + n0 + 8] = acc[j][2];
      out[(m + 1) * kTileRows + n0 + 8] = acc[j][3];
    } else {
      *reinterpret_cast<float2*>(out + n0 * Mpad + m) = make_float2(acc[j][0], acc[j][1]);
      *reinterpret_cast<float2*>(out + (n0 + 8) * Mpad + m) = make_float2(acc[j][2], acc[j][3]);
    }
    acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  }
  if constexpr (kGemvQGroups > 1) {
    named_bar(1, nthr);
    constexpr int kTF = kTileRows * NT * 8;
    for (int e = tid; e < kTF; e += nthr) {
      float v = gpart[e];
#pragma unroll
      for (int q = 1; q < kGemvQGroups; ++q) v += gpart[q * kTF + e];
      dst[e] = v;
    }
  }
}


template <int NT, int NTC, bool kCluster, int QB>
__global__ void __launch_bounds__(kGemvQThreads, kGemvQCtasPerSm) gemv_q_kernel(const GemvParams p) {
  constexpr int CW = kGemvQConsumerWarps;
  using C = GemvQCfg<NT, QB, NTC>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int kStages = p.stages;
  uint8_t* ring = smem;
  float* otile = reinterpret_cast<float*>(smem + kStages * C::kStageBytes);
  float* staging = otile + C::kTileFloats;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes + (C::kTileFloats + C::kStagingFloats) * 4);
  uint64_t* empty = full + C::kMaxStages;
  int* flag = reinterpret_cast<int*>(empty + C::kMaxStages);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(flag) + 64);   // [128]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(flag) + 4;      // x prefetch barrier (in the flag block)
  float* xpre = scratch + 128;                                  // [kXPreFloats] residual rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SS_TRACE_MIN(0);
  unsigned long long* ct = p.cta_trace ? p.cta_trace + 5 * blockIdx.x : nullptr;
  if (ct && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    ct[0] = sm;
    ct[1] = gtime();
  }
  const int nC = p.K >> 7;
  const int64_t T = int64_t(p.N >> 7) * nC;
  const int Mpad = NT * 8;
  uint32_t crank = 0, csize = 1;
  if constexpr (kCluster) {
    crank = cluster_rank();
    csize = cluster_nrank();
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    mbar_init(xbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch();   // grid <= one CTA per SM: let the next kernel prefetch now

  if (warp == CW) {
    // ------------------------------ producer -------------------------------
    Work w = make_work<kCluster>(p.N, p.K, crank, csize);
    const int64_t n_stage = w.stages(nC, C::kCPS);
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int pre = int(n_stage < kStages ? n_stage : kStages);
      Work wx = w;   // replayed below for the activation copies of the prefetched stages
      const uint32_t per_chunk = uint32_t(C::kWBytes + C::kXBytes + C::kSBytes);
      auto issue_w = [&](int st, const Work& ww, int n) {
        mbar_arrive_expect_tx(&full[st], uint32_t(n) * per_chunk);
        bulk_g2s_hint(ring + st * C::kStageBytes, p.W + (int64_t(ww.r) * nC + ww.c) * C::kWBytes,
                      uint32_t(n) * C::kWBytes, &full[st], pol);
      };
      auto issue_x = [&](int st, const Work& ww, int n) {
        uint8_t* base = ring + st * C::kStageBytes + C::kCPS * C::kWBytes;
        bulk_g2s(base, p.X + int64_t(ww.c) * NT * 1024, uint32_t(n) * C::kXBytes, &full[st]);
        bulk_g2s(base + C::kCPS * C::kXBytes, p.XS + int64_t(ww.c) * 2 * NT * 8, uint32_t(n) * C::kSBytes, &full[st]);
      };
      // weights do not depend on the previous kernel: issue before the grid-dependency wait
      for (int i = 0; i < pre; ++i) {
        const int n = w.take(C::kCPS);
        issue_w(i, w, n);
        w.next(nC, n);
      }
      // L2 prefetch of the next matrix (independent of every activation): this CTA's slice, in
      // 64 KB TMA prefetches, so HBM keeps streaming through the dependent steps that follow
      auto prefetch_next = [&]() {
        const int64_t per = ((p.pf_bytes / gridDim.x) + 15) & ~int64_t(15);
        const int64_t b0 = per * blockIdx.x;
        const int64_t b1 = b0 + per < p.pf_bytes ? b0 + per : p.pf_bytes;
        for (int64_t o = b0; o < b1; o += 65536) {
          const int64_t n = b1 - o < 65536 ? b1 - o : 65536;
          prefetch_l2(p.pf + o, uint32_t(n));
        }
      };
      if (p.pf && p.pf_bytes > 0) prefetch_next();
      griddep_wait();
      SS_TRACE_CTA0(1);
      for (int i = 0; i < pre; ++i) {
        const int n = wx.take(C::kCPS);
        issue_x(i, wx, n);
        wx.next(nC, n);
      }
      int st = pre % kStages;
      uint32_t ph = pre / kStages;   // 0 or 1 (pre <= kStages)
      for (int64_t i = pre; i < n_stage; ++i) {
        mbar_wait(&empty[st], (ph - 1) & 1);
        const int n = w.take(C::kCPS);
        issue_w(st, w, n);
        issue_x(st, w, n);
        w.next(nC, n);
        if (++st == kStages) {
          st = 0;
          ++ph;
        }
      }
    }
    if constexpr (kCluster) {
      if (csize > 1) {   // take part in the cluster barriers of every tile's reduction
        const int64_t per = int64_t(w.c_end - w.c_begin);
        const int64_t tiles = per ? w.left / per : 0;
        for (int64_t t = 0; t < tiles; ++t) {
          cluster_sync_all();
          if (t + 1 < tiles) cluster_sync_all();
        }
      }
    }
    return;
  }

  // ------------------------------ consumers --------------------------------
  griddep_wait();
  if (threadIdx.x == 0) SS_TRACE_CTA0(2);
  const int nthr = CW * 32;
  float acc[NTC][4];
#pragma unroll
  for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  float* gpart = xpre + C::kXPreFloats;   // per-warp-group partial tiles (several warp groups only)
  auto stash = [&](float* dst) { stash_q<NT, NTC>(acc, dst, warp, lane, false, gpart, threadIdx.x, nthr); };   // [128][Mpad]

  uint32_t xph = 0;   // phase of xbar
  auto flush = [&](int r, int c_first, int c_last, bool last) {
    if constexpr (kCluster) {
      if (csize == 1) {
        stash(otile);
        named_bar(1, nthr);
        if (threadIdx.x == 0) SS_TRACE_MAX(8);
        apply_epilogue(p.epi, otile, Mpad, r, 0, Mpad, threadIdx.x, nthr, scratch, p.trace, 1, true, Mpad);
        named_bar(1, nthr);
        return;
      }
      // Split-K reduction spread over the cluster: rank q owns token columns [mlo, mhi) of the tile.
      // Every rank stashes its partial tile token-major, pushes each owner's columns into the owner's
      // staging buffer with 16-byte distributed-shared-memory stores, and after ONE cluster barrier
      // each owner sums its staging in rank order (deterministic) and runs the epilogue for its
      // tokens (one arrival per rank at EPI_RESID_NORM's barrier; only rank 0 waits there and
      // normalises, so ranks 1..S-1 exit and the barrier never needs whole clusters co-resident).
      const int S = int(csize);
      const int mlo = int(crank) * Mpad / S, mhi = int(crank + 1) * Mpad / S;
      const int nc = mhi - mlo, ncmax = (Mpad + S - 1) / S;
      // residual epilogues: TMA-load the owned tokens' residual rows of this tile now, so the
      // epilogue's read-modify-write does not pay an L2 round trip after the reduction
      const int nvalid = nc < p.epi.M - mlo ? nc : (p.epi.M - mlo > 0 ? p.epi.M - mlo : 0);
      const bool xp = nvalid > 0 && nc <= C::kXPreTokens &&
                      (p.epi.kind == EPI_RESID || p.epi.kind == EPI_RESID_NORM);
      if (xp && threadIdx.x == 0) {
        mbar_arrive_expect_tx(xbar, uint32_t(nvalid) * kTileRows * 4);
        for (int m = 0; m < nvalid; ++m)
          bulk_g2s(xpre + m * kTileRows, p.epi.x + int64_t(mlo + m) * p.epi.ldx + int64_t(r) * kTileRows, kTileRows * 4, xbar);
      }
      stash_q<NT, NTC>(acc, otile, warp, lane, true, gpart, threadIdx.x, nthr);   // token-major [Mpad][128]
      named_bar(1, nthr);
      for (int i = threadIdx.x; i < Mpad * (kTileRows / 4); i += nthr) {
        const int m = i / (kTileRows / 4), n4 = (i % (kTileRows / 4)) * 4;
        const int q = int(owner_of(m, Mpad, S));          // owner rank of token m
        const int mm = m - q * Mpad / S;
        st_dsmem_f32x4(staging + (crank * ncmax + mm) * kTileRows + n4, uint32_t(q),
                       *reinterpret_cast<const float4*>(otile + m * kTileRows + n4));
      }
      cluster_sync_all();                         // every push landed (release / acquire)
      for (int it = threadIdx.x; it < kTileRows * nc; it += nthr) {
        const int n = it % kTileRows, mm = it / kTileRows;
        float v = staging[mm * kTileRows + n];
        for (int q = 1; q < S; ++q) v += staging[(q * ncmax + mm) * kTileRows + n];
        otile[n * nc + mm] = v;                   // [128][nc] for the epilogue
      }
      if (!last) cluster_sync_all();              // staging is reused by the next tile's pushes
      named_bar(1, nthr);
      if (threadIdx.x == 0) SS_TRACE_MAX(8);
      if (xp) {
        mbar_wait(xbar, xph);
        xph ^= 1;
      }
      apply_epilogue(p.epi, otile, nc, r, mlo, nc, threadIdx.x, nthr, scratch, p.trace, S, crank == 0, Mpad, nullptr,
                     xp ? xpre : nullptr);
      named_bar(1, nthr);
      return;
    } else {
      const bool complete = (c_first == 0 && c_last == nC - 1);
      if (complete) {
        stash(otile);
      } else {
        const int G = gridDim.x;
        const int64_t first = owner_of(int64_t(r) * nC, T, G);
        const int64_t nseg = owner_of(int64_t(r + 1) * nC - 1, T, G) - first + 1;
        const int64_t slot = blockIdx.x - first;
        stash(p.partials + (int64_t(r) * p.max_seg + slot) * int64_t(kTileRows * Mpad));
        __threadfence();
        named_bar(1, nthr);
        if (threadIdx.x == 0) {
          const int old = atomicAdd(&p.counters[r], 1);
          *flag = (old == nseg - 1);
        }
        named_bar(1, nthr);
        if (!*flag) return;
        __threadfence();
        const float* base = p.partials + int64_t(r) * p.max_seg * int64_t(kTileRows * Mpad);
        for (int e = threadIdx.x; e < kTileRows * Mpad; e += nthr) {
          float s = 0.f;
          for (int q = 0; q < nseg; ++q) s += __ldcg(base + q * int64_t(kTileRows * Mpad) + e);
          otile[e] = s;
        }
        if (threadIdx.x == 0) p.counters[r] = 0;
      }
      named_bar(1, nthr);
      apply_epilogue(p.epi, otile, Mpad, r, 0, Mpad, threadIdx.x, nthr);
      named_bar(1, nthr);
    }
  };

  Work w = make_work<kCluster>(p.N, p.K, crank, csize);
  const int64_t n_items = w.left;
  int s = 0;
  uint32_t ph = 0;
  // Outer loop over this CTA's row tiles, inner loop over the tile's stages: the inner loop is a
  // compact basic-block chain and the (large) reduction/epilogue code sits after it, so the hot
  // path never jumps across the flush code (ncu: the single-loop form lost ~20% of the consumer's
  // issue slots to instruction-fetch stalls on two far branches per stage).
  while (w.left > 0) {
    const int cur_r = w.r, c_first = w.c;
    int c_last = w.c;
    do {
      const int nch = w.take(C::kCPS);
      c_last = w.c + nch - 1;
      mbar_wait(&full[s], ph);
      if (threadIdx.x == 0 && w.left == n_items) {
        SS_TRACE_CTA0(3);
        if (ct) ct[2] = gtime();
      }
      consume_q<NT, NTC, QB>(ring + s * C::kStageBytes, nch, acc, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
      w.next(nC, nch);
    } while (w.left > 0 && w.r == cur_r);
    const bool last = w.left == 0;
    if (last && threadIdx.x == 0) {
      SS_TRACE_CTA0(4);
      SS_TRACE_MAX(7);
      if (ct) ct[3] = gtime();
    }
    flush(cur_r, c_first, c_last, last);
  }
  if (threadIdx.x == 0) {
    SS_TRACE_MAX(6);
    if (ct) ct[4] = gtime();
  }
}


// ring stages of an instantiation; sets its smem/cluster attributes once per device (function
// attributes are per device)
template <int NT, int NTC, bool kCluster, int QB>
static int ensure_attrs_q() {
  using C = GemvQCfg<NT, QB, NTC>;
  static std::mutex mu;
  static std::map<int, int> stages_of;
  std::lock_guard<std::mutex> lk(mu);
  const int dev = current_device();
  auto it = stages_of.find(dev);
  if (it != stages_of.end()) return it->second;
  // (two-CTA-per-SM builds, SS_K2_CW = 8) Q2 stages are smaller: a 72 KB budget keeps two CTAs per SM (the Q4/bf16 rings round 88 KB
  // down to ~68 KB of whole stages)
  const int budget = kGemvQCtasPerSm == 2 ? (QB == 2 ? 72 : (QB == 3 ? 80 : 88)) * 1024
                                           : SS_K2_RING1_KB * 1024 - C::smem_for(0);
  int st = budget / C::kStageBytes;
  if (st < 2) st = 2;
  if (st > C::kMaxStages) st = C::kMaxStages;
  cudaFuncSetAttribute(gemv_q_kernel<NT, NTC, kCluster, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(st));
  stages_of[dev] = st;
  return st;
}

// Cluster plan {S, clusters}: the GPC structure caps how many clusters of S CTAs are resident at
// once (e.g. 33 clusters of 8 at 2 CTAs/SM, below qkv's 36 row tiles), and a tile whose cluster is
// not resident waits for a second wave.  Take the largest S <= gemv_cluster_split whose resident
// cluster count covers every row tile (queried with cudaOccupancyMaxActiveClusters).  Cached per
// (device, shape, hint).
struct ClusterPlanQ {
  int S, ncl;
  bool all_resident;
};
template <int NT, int NTC, int QB>
static ClusterPlanQ cluster_plan_q(int N, int K, int sms, int hint = 0) {
  const int stages = ensure_attrs_q<NT, NTC, true, QB>();
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, ClusterPlanQ> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(current_device(), N, K, hint);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  using C = GemvQCfg<NT, QB, NTC>;
  const int tiles = N / 128;
  const int per_sm = hint > 0 ? hint : kGemvQCtasPerSm;
  const int S0 = gemv_q_split(N, K, sms, hint);
  ClusterPlanQ plan{S0, 0, false};
  for (int S = S0; S >= 1; --S) {
    int ncl = sms * per_sm / S;
    if (ncl > tiles) ncl = tiles;
    if (ncl < 1) ncl = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl * S);
    cfg.blockDim = dim3(kGemvQThreads);
    cfg.dynamicSmemBytes = C::smem_for(stages);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = S;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, gemv_q_kernel<NT, NTC, true, QB>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      active = ncl;   // cannot query: keep the arithmetic plan
    }
    if (S == S0) plan = ClusterPlanQ{S0, active < ncl ? active : ncl, active >= tiles};
    if (active >= tiles) {
      plan = ClusterPlanQ{S, tiles, true};
      break;
    }
  }
  if (plan.ncl < 1) plan.ncl = 1;
  cache[key] = plan;
  return plan;
}

// every row tile has its own resident cluster (required by EPI_RESID_NORM's in-kernel barrier)
bool gemv_q_tiles_all_resident(int NT, int N, int K, int sms, int bits) {
  if (N / 128 > 2 * sms) return false;
  if (bits == 2) return NT <= 2 ? cluster_plan_q<2, 1, 2>(N, K, sms).all_resident : cluster_plan_q<4, 4, 2>(N, K, sms).all_resident;
  if (bits == 3) return NT <= 2 ? cluster_plan_q<2, 1, 3>(N, K, sms).all_resident : cluster_plan_q<4, 4, 3>(N, K, sms).all_resident;
  return NT <= 2 ? cluster_plan_q<2, 1, 4>(N, K, sms).all_resident : cluster_plan_q<4, 4, 4>(N, K, sms).all_resident;
}

template <int NT, int NTC, bool kCluster, int QB>
static void launch_tq(const GemvParams& p0, int grid, int S, bool pdl, cudaStream_t st) {
  using C = GemvQCfg<NT, QB, NTC>;
  const int stages = ensure_attrs_q<NT, NTC, kCluster, QB>();
  GemvParams p = p0;
  p.stages = stages;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvQThreads);
  cfg.dynamicSmemBytes = C::smem_for(stages);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (kCluster) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = S;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, gemv_q_kernel<NT, NTC, kCluster, QB>, p);
}

template <int NT, int NTC, int QB>
static void launch_mode_q(const GemvParams& p, int sms, bool pdl, cudaStream_t st) {
  if (p.N / 128 <= 2 * sms) {
    const ClusterPlanQ pl = cluster_plan_q<NT, NTC, QB>(p.N, p.K, sms, p.ctas_per_sm);
    launch_tq<NT, NTC, true, QB>(p, pl.ncl * pl.S, pl.S, pdl, st);
  } else {
    launch_tq<NT, NTC, false, QB>(p, gemv_grid_for(p.N, p.K, sms), 1, pdl, st);
  }
}

// 4-/2-bit substitute GEMV: activation layout NT = 2 (M <= 16) or 4 (M <= 32); the MMAs cover only the
// token groups that hold tokens (NTC = ceil(M / 8): 1, 2 or 4)
void launch_gemv_q(const GemvParams& p, int sms, bool pdl, cudaStream_t st) {
  const int ntc = p.epi.M <= 8 ? 1 : (p.epi.M <= 16 ? 2 : 4);
  if (p.qbits == 2) {
    if (p.NT <= 2) ntc == 1 ? launch_mode_q<2, 1, 2>(p, sms, pdl, st) : launch_mode_q<2, 2, 2>(p, sms, pdl, st);
    else launch_mode_q<4, 4, 2>(p, sms, pdl, st);
  } else if (p.qbits == 3) {
    if (p.NT <= 2) ntc == 1 ? launch_mode_q<2, 1, 3>(p, sms, pdl, st) : launch_mode_q<2, 2, 3>(p, sms, pdl, st);
    else launch_mode_q<4, 4, 3>(p, sms, pdl, st);
  } else {
    if (p.NT <= 2) ntc == 1 ? launch_mode_q<2, 1, 4>(p, sms, pdl, st) : launch_mode_q<2, 2, 4>(p, sms, pdl, st);
    else launch_mode_q<4, 4, 4>(p, sms, pdl, st);
  }
}

}  // namespace ss
