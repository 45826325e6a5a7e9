// K2 — fused dequant-GEMV/GEMM for the draft (M = frontier tokens <= 32).
// Y[M x N] = X[M x K] * W_hat^T with W_hat = code*s + z per 64-group
// ("highly optimized low-bit GEMM kernels"; 4 bit / group 64, PAPER.md:278;
// reading R3 in DESIGN.md: the affine dequantisation is applied exactly, in fp32).
//
// B200 design:
//  * weights are tile-chunk contiguous (128 rows x 128 k, 9 KB for Q4): a CTA streams its work
//    with cp.async.bulk (TMA engine) into an S-stage shared-memory ring guarded by mbarriers; the
//    weight part of the first stages is issued BEFORE griddepcontrol.wait (PDL), overlapping the
//    previous kernel's tail;
//  * 8 consumer warps turn 4-bit codes into exact bf16 (128 + code) with ONE lop3 per pair and
//    feed them straight into mma.m16n8k16 as the 16-row A operand (tokens are N = 8..32); every
//    k-step stays inside one 64-group, the producers of X publish its 64-group sums, and
//    y += s*sum((128+c)x) + (z - 128 s)*sum(x) applies the group scale/zero in fp32;
//  * narrow matrices (qkv, o, down) use cluster split-K: the S CTAs of a cluster split a row
//    tile's K and rank 0 reduces their partial tiles through distributed shared memory, in rank
//    order, then runs the fused epilogue (bias+RoPE+KV write / residual / SiLU*mul / logits);
//    persistent clusters loop over row tiles so that at most one CTA per SM is used and the next
//    kernel can co-reside and prefetch;
//  * the tall bf16 head uses Stream-K (equal contiguous ranges of the tile-chunk space per
//    persistent CTA) with a fixed-order fixup by the last-arriving CTA.
#include "common.cuh"
#include "epilogue.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

namespace ss {

static int gemv_grid_for(int N, int K, int grid) {
  const int64_t T = int64_t(N / 128) * (K / 128);
  return int(T < grid ? T : grid);   // every Stream-K CTA gets >= 1 tile-chunk
}

int gemv_max_segments(int N, int K, int grid) {
  const int64_t nC = K / 128, T = int64_t(N / 128) * nC;
  grid = gemv_grid_for(N, K, grid);
  int mx = 1;
  for (int64_t r = 0; r < N / 128; ++r) {
    const int s = int(owner_of((r + 1) * nC - 1, T, grid) - owner_of(r * nC, T, grid) + 1);
    if (s > mx) mx = s;
  }
  return mx;
}

template <int WF, int NT, bool kCluster>
__global__ void __launch_bounds__(kGemvThreads, WF == 16 ? 1 : 2) gemv_kernel(const GemvParams p) {
  using C = GemvCfg<WF, NT>;
  constexpr int kN = C::kN;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int kStages = p.stages;
  uint8_t* ring = smem;
  float* otile = reinterpret_cast<float*>(smem + kStages * C::kStageBytes);
  float* staging = otile + C::kTileFloats;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::kStagingFloats);
  uint64_t* empty = full + C::kMaxStages;
  uint64_t* a_full = empty + C::kMaxStages;
  uint64_t* a_empty = a_full + C::kASlots;
  uint64_t* d_full = a_empty + C::kASlots;
  uint64_t* d_empty = d_full + C::kDSlots;
  uint64_t* xbar = d_empty + C::kDSlots;                         // residual-row prefetch
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 1);
  int* flag = reinterpret_cast<int*>(xbar + 2);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(flag) + 64);   // [128]
  float* xpre = scratch + 128;                                    // [kXPreFloats] residual rows

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
  uint32_t crank = 0, csize = 1;
  if constexpr (kCluster) {
    crank = cluster_rank();
    csize = cluster_nrank();
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kQ ? 9 : 1);   // Q: MMA commit + 4 convert + 4 accumulate warps
    }
    for (int j = 0; j < C::kASlots; ++j) {
      mbar_init(&a_full[j], 4);
      mbar_init(&a_empty[j], 1);
    }
    for (int j = 0; j < C::kDSlots; ++j) {
      mbar_init(&d_full[j], 1);
      mbar_init(&d_empty[j], 4);
    }
    mbar_init(xbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  griddep_launch();   // grid <= the resident CTAs: let the next kernel prefetch now
  // a CTA with two or more tiles in a cluster of > 1 would need one cluster barrier per tile from
  // every warp; the launcher only plans clusters of one tile each (csize > 1) or csize == 1
  const bool cl_sync = kCluster && csize > 1;

  if (warp == 0) {
    // ------------------------------ producer (TMA) -------------------------------
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
        if constexpr (C::kQ)
          bulk_g2s(base + C::kCPS * C::kXBytes, p.XS + int64_t(ww.c) * 2 * kN, uint32_t(n) * C::kSBytes, &full[st]);
      };
      // weights do not depend on the previous kernel: issue before the grid-dependency wait
      for (int i = 0; i < pre; ++i) {
        const int n = w.take(C::kCPS);
        issue_w(i, w, n);
        w.next(nC, n);
      }
      // L2 prefetch of the next matrix (independent of every activation): this CTA's slice
      if (p.pf && p.pf_bytes > 0) {
        const int64_t per = ((p.pf_bytes / gridDim.x) + 15) & ~int64_t(15);
        const int64_t b0 = per * blockIdx.x;
        const int64_t b1 = b0 + per < p.pf_bytes ? b0 + per : p.pf_bytes;
        for (int64_t o = b0; o < b1; o += 65536) prefetch_l2(p.pf + o, uint32_t(b1 - o < 65536 ? b1 - o : 65536));
      }
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
    __syncwarp();
    if (cl_sync) cluster_sync_all();
    return;
  }

  if (warp == 1) {
    // ------------------------------ MMA issuer -------------------------------
    Work w = make_work<kCluster>(p.N, p.K, crank, csize);
    if (lane == 0) {
      griddep_wait();   // acquire side of the activations' dependency for the async proxy reads
      constexpr uint32_t idesc = umma_idesc_bf16(kN);
      int s = 0;
      uint32_t ph = 0;
      int ja = 0, jd = 0;
      uint32_t ua[C::kASlots] = {}, ud[C::kDSlots] = {};
      while (w.left > 0) {
        const int cur_r = w.r;
        bool first = true;
        do {
          const int nch = w.take(C::kCPS);
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sb = smem_u32(ring + s * C::kStageBytes);
          const uint32_t xb = sb + C::kCPS * C::kWBytes;
          w.next(nC, nch);
          const bool last = w.left == 0 || w.r != cur_r;
          if constexpr (C::kQ) {
            for (int ci = 0; ci < nch; ++ci)
#pragma unroll
              for (int G = 0; G < 2; ++G) {
                mbar_wait(&a_full[ja], ua[ja] & 1);
                mbar_wait(&d_empty[jd], (ud[jd] & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_ts(tbase + jd * kN, tbase + C::kACol0 + ja * 32 + kk * 8,
                          umma_desc(xb + ci * C::kXBytes + G * 1024 + kk * 256, 128, 2048), idesc, kk > 0);
                umma_commit(&a_empty[ja]);
                umma_commit(&d_full[jd]);
                ++ua[ja];
                ++ud[jd];
                ja = (ja + 1) % C::kASlots;
                jd = (jd + 1) % C::kDSlots;
              }
          } else {
            if (first) {
              mbar_wait(&d_empty[jd], (ud[jd] & 1) ^ 1);
              tc_fence_after();
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_ss(tbase + jd * kN, umma_desc(sb + kk * 256, 128, 2048), umma_desc(xb + kk * 256, 128, 2048), idesc,
                      (first && kk == 0) ? 0u : 1u);
            if (last) {
              umma_commit(&d_full[jd]);
              ++ud[jd];
              jd = (jd + 1) % C::kDSlots;
            }
          }
          umma_commit(&empty[s]);
          first = false;
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        } while (w.left > 0 && w.r == cur_r);
      }
    }
    __syncwarp();
    named_bar(3, 160);   // the accumulate warps have read the last accumulator
    tc_fence_after();
    tmem_dealloc(tbase, C::kTmemCols);
    if (cl_sync) cluster_sync_all();
    return;
  }

  // ---------------------------- worker warps 2..9 ----------------------------
  griddep_wait();
  const int tid = threadIdx.x - 64;             // 0..255 over the worker warps
  const int q = warp & 3;                       // TMEM lane quadrant of this warp
  const int row = 32 * q + lane;                // weight row of the tile owned in TMEM
  const uint32_t tl = tbase + (uint32_t(32 * q) << 16);
  const bool is_convert = warp < 6;
  const int Mv = p.epi.M < kN ? p.epi.M : kN;   // valid tokens

  uint32_t xph = 0;   // phase of xbar
  // --- split-K reduction + epilogue of tile r from otile (worker threads only) ---
  auto flush = [&](int r, int c_first, int c_last, bool last) {
    const int nthr = kGemvWorkers;
    if constexpr (kCluster) {
      if (csize == 1) {
        named_bar(1, nthr);
        if (tid == 0) SS_TRACE_MAX(8);
        apply_epilogue(p.epi, otile, kN, r, 0, kN, tid, nthr, scratch, p.trace, 1, true, kN);
        named_bar(1, nthr);
        return;
      }
      // Split-K reduction spread over the cluster: rank q owns token columns [mlo, mhi) of the tile.
      // Every rank has its partial tile token-major in otile, pushes each owner's columns into the
      // owner's staging buffer with 16-byte distributed-shared-memory stores, and after ONE cluster
      // barrier each owner sums its staging in rank order (deterministic) and runs the epilogue for
      // its tokens (one arrival per rank at EPI_RESID_NORM's barrier; only rank 0 waits there).
      const int S = int(csize);
      const int mlo = int(crank) * kN / S, mhi = int(crank + 1) * kN / S;
      const int nc = mhi - mlo, ncmax = (kN + S - 1) / S;
      const int nvalid = nc < p.epi.M - mlo ? nc : (p.epi.M - mlo > 0 ? p.epi.M - mlo : 0);
      const bool xp = nvalid > 0 && nc <= C::kXPreTokens && (p.epi.kind == EPI_RESID || p.epi.kind == EPI_RESID_NORM);
      if (xp && tid == 0) {
        mbar_arrive_expect_tx(xbar, uint32_t(nvalid) * kTileRows * 4);
        for (int m = 0; m < nvalid; ++m)
          bulk_g2s(xpre + m * kTileRows, p.epi.x + int64_t(mlo + m) * p.epi.ldx + int64_t(r) * kTileRows, kTileRows * 4, xbar);
      }
      named_bar(1, nthr);
      for (int i = tid; i < kN * (kTileRows / 4); i += nthr) {
        const int m = i / (kTileRows / 4), n4 = (i % (kTileRows / 4)) * 4;
        const int qo = int(owner_of(m, kN, S));          // owner rank of token m
        const int mm = m - qo * kN / S;
        st_dsmem_f32x4(staging + (crank * ncmax + mm) * kTileRows + n4, uint32_t(qo),
                       *reinterpret_cast<const float4*>(otile + m * kTileRows + n4));
      }
      cluster_sync_all();                         // every push landed (release / acquire)
      for (int it = tid; it < kTileRows * nc; it += nthr) {
        const int n = it % kTileRows, mm = it / kTileRows;
        float v = staging[mm * kTileRows + n];
        for (int qq = 1; qq < S; ++qq) v += staging[(qq * ncmax + mm) * kTileRows + n];
        otile[n * nc + mm] = v;                   // [128][nc] for the epilogue
      }
      named_bar(1, nthr);
      if (tid == 0) SS_TRACE_MAX(8);
      if (xp) {
        mbar_wait(xbar, xph);
        xph ^= 1;
      }
      apply_epilogue(p.epi, otile, nc, r, mlo, nc, tid, nthr, scratch, p.trace, S, crank == 0, kN, nullptr,
                     xp ? xpre : nullptr);
      named_bar(1, nthr);
      return;
    } else {
      const bool complete = (c_first == 0 && c_last == nC - 1);
      named_bar(1, nthr);
      if (!complete) {
        const int G = gridDim.x;
        const int64_t first = owner_of(int64_t(r) * nC, T, G);
        const int64_t nseg = owner_of(int64_t(r + 1) * nC - 1, T, G) - first + 1;
        const int64_t slot = blockIdx.x - first;
        float* dst = p.partials + (int64_t(r) * p.max_seg + slot) * int64_t(kTileRows * kN);
        for (int e = tid; e < kTileRows * kN; e += nthr) dst[e] = otile[e];
        __threadfence();
        named_bar(1, nthr);
        if (tid == 0) {
          const int old = atomicAdd(&p.counters[r], 1);
          *flag = (old == nseg - 1);
        }
        named_bar(1, nthr);
        if (!*flag) return;
        __threadfence();
        const float* base = p.partials + int64_t(r) * p.max_seg * int64_t(kTileRows * kN);
        for (int e = tid; e < kTileRows * kN; e += nthr) {
          float sum = 0.f;
          for (int qq = 0; qq < nseg; ++qq) sum += __ldcg(base + qq * int64_t(kTileRows * kN) + e);
          otile[e] = sum;
        }
        if (tid == 0) p.counters[r] = 0;
        named_bar(1, nthr);
      }
      apply_epilogue(p.epi, otile, kN, r, 0, kN, tid, nthr);
      named_bar(1, nthr);
    }
  };
  // the accumulated rows of the tile -> otile: token-major [N][128] in cluster mode (the push layout),
  // row-major [128][N] otherwise (the epilogue / Stream-K partial layout)
  auto to_otile = [&](const float (&y)[kN]) {
#pragma unroll
    for (int t = 0; t < kN; ++t) {
      if constexpr (kCluster) {
        if (csize > 1) otile[t * kTileRows + row] = y[t];
        else otile[row * kN + t] = y[t];
      } else {
        otile[row * kN + t] = y[t];
      }
    }
  };

  Work w = make_work<kCluster>(p.N, p.K, crank, csize);
  const int64_t n_items = w.left;
  int s = 0;
  uint32_t ph = 0;
  int ja = 0, jd = 0;
  uint32_t ua[C::kASlots] = {}, ud[C::kDSlots] = {};
  const uint32_t kMagic = 0x43004300u;   // bf16x2 (128, 128): 128 + code is exact in bf16
  while (w.left > 0) {
    const int cur_r = w.r, c_first = w.c;
    int c_last = w.c;
    float y[kN];
#pragma unroll
    for (int t = 0; t < kN; ++t) y[t] = 0.f;
    do {
      const int nch = w.take(C::kCPS);
      c_last = w.c + nch - 1;
      const uint8_t* stage = ring + s * C::kStageBytes;
      if (C::kQ) mbar_wait(&full[s], ph);   // bf16: the MMAs read the stage, the workers only the accumulator
      if (threadIdx.x == 64 && w.left == n_items) {
        SS_TRACE_CTA0(3);
        if (ct) ct[2] = gtime();
      }
      w.next(nC, nch);
      const bool last_of_tile = w.left == 0 || w.r != cur_r;
      if constexpr (C::kQ) {
        if (is_convert) {
          // ---- codes of row `row` -> exact bf16 (128 + code) pairs -> TMEM A slot (32 columns) ----
          for (int ci = 0; ci < nch; ++ci)
#pragma unroll
            for (int G = 0; G < 2; ++G) {
              const uint8_t* wst = stage + ci * C::kWBytes;
              uint32_t v[32];
              if constexpr (WF == 4) {
                const uint4 c0 = *reinterpret_cast<const uint4*>(wst + G * 4096 + row * 16);
                const uint4 c1 = *reinterpret_cast<const uint4*>(wst + G * 4096 + 2048 + row * 16);
                const uint32_t wd[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                  for (int pp = 0; pp < 4; ++pp) v[4 * j + pp] = lop3_and_or(wd[j] >> (4 * pp), kMagic);
              } else {
                const uint4 c0 = *reinterpret_cast<const uint4*>(wst + G * 2048 + row * 16);
                const uint32_t wd[4] = {c0.x, c0.y, c0.z, c0.w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                  for (int pp = 0; pp < 8; ++pp) v[8 * j + pp] = lop3_and_or2(wd[j] >> (2 * pp), kMagic);
              }
              mbar_wait(&a_empty[ja], (ua[ja] & 1) ^ 1);
              tc_fence_after();
              tmem_st32(tl + C::kACol0 + ja * 32, v);
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&a_full[ja]);
              ++ua[ja];
              ja = (ja + 1) % C::kASlots;
            }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        } else {
          // ---- per-group accumulators -> y += s * acc + (z - 128 s) * sum(x)  (exact affine, fp32) ----
          for (int ci = 0; ci < nch; ++ci)
#pragma unroll
            for (int G = 0; G < 2; ++G) {
              const uint32_t meta = *reinterpret_cast<const uint32_t*>(stage + ci * C::kWBytes + C::kCodeBytes + G * 512 + row * 4);
              const float* xs = reinterpret_cast<const float*>(stage + C::kCPS * (C::kWBytes + C::kXBytes) + ci * C::kSBytes) + G * kN;
              const float sc = __uint_as_float(meta << 16), z = __uint_as_float(meta & 0xFFFF0000u);
              const float zz = fmaf(-128.0f, sc, z);   // exact
              mbar_wait(&d_full[jd], ud[jd] & 1);
              tc_fence_after();
              uint32_t d[kN];
              if constexpr (kN == 16) {
                tmem_ld16(tl + jd * kN, d);
              } else {
                uint32_t d0[16], d1[16];
                tmem_ld16(tl + jd * kN, d0);
                tmem_ld16(tl + jd * kN + 16, d1);
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  d[t] = d0[t];
                  d[16 + t] = d1[t];
                }
              }
              tmem_wait_ld();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&d_empty[jd]);
              ++ud[jd];
              jd = (jd + 1) % C::kDSlots;
#pragma unroll
              for (int t = 0; t < kN; ++t)
                if (t < Mv) y[t] = fmaf(sc, __uint_as_float(d[t]), fmaf(zz, xs[t], y[t]));
            }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      } else {
        if (!is_convert && last_of_tile) {   // bf16: the tile's accumulator, K reduced by the MMAs
          mbar_wait(&d_full[jd], ud[jd] & 1);
          tc_fence_after();
          uint32_t d[kN];
          if constexpr (kN == 16) {
            tmem_ld16(tl + jd * kN, d);
          } else {
            uint32_t d0[16], d1[16];
            tmem_ld16(tl + jd * kN, d0);
            tmem_ld16(tl + jd * kN + 16, d1);
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              d[t] = d0[t];
              d[16 + t] = d1[t];
            }
          }
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[jd]);
          ++ud[jd];
          jd = (jd + 1) % C::kDSlots;
#pragma unroll
          for (int t = 0; t < kN; ++t) y[t] = __uint_as_float(d[t]);
        }
      }
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    } while (w.left > 0 && w.r == cur_r);
    const bool last = w.left == 0;
    if (!is_convert) {
      to_otile(y);
      if (last) named_bar(3, 160);   // let warp 1 free TMEM: every accumulator has been read
    }
    if (last && tid == 0) {
      SS_TRACE_CTA0(4);
      SS_TRACE_MAX(7);
      if (ct) ct[3] = gtime();
    }
    flush(cur_r, c_first, c_last, last);
  }
  if (w.left == 0 && n_items == 0 && !is_convert) named_bar(3, 160);   // no work: still release warp 1
  if (tid == 0) {
    SS_TRACE_MAX(6);
    if (ct) ct[4] = gtime();
  }
}


// split factor of the cluster mode: ~per_sm CTAs per SM (hint, default 2), <= 8 (portable), <= chunks
int gemv_cluster_split(int N, int K, int sms, int hint) {
  const int tiles = N / 128, nC = K / 128;
  const int per_sm = hint > 0 ? hint : 2;
  int S = (per_sm * sms) / tiles;
  if (S < 1) S = 1;
  if (S > 8) S = 8;
  if (S > nC) S = nC;
  return S;
}
bool gemv_use_cluster(int N, int K, int sms) { return N / 128 <= 2 * sms; }
// Stream-K grid of a tall matrix: one CTA per SM for bf16, two for substitutes
int gemv_streamk_grid(bool q4, int N, int K, int sms) { return gemv_grid_for(N, K, sms * (q4 ? 2 : 1)); }

static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// ring stages of an instantiation; sets its smem attribute once per device (function attributes are
// per device).  Substitutes: ~88 KB of ring keeps two CTAs per SM; bf16 (head / resident layers):
// one CTA per SM with a ~190 KB ring.
template <int WF, int NT, bool kCluster>
static int ensure_attrs() {
  using C = GemvCfg<WF, NT>;
  static std::mutex mu;
  static std::map<int, int> stages_of;
  std::lock_guard<std::mutex> lk(mu);
  const int dev = current_device();
  auto it = stages_of.find(dev);
  if (it != stages_of.end()) return it->second;
  const int budget = (WF == 16 ? 190 : 88) * 1024;
  int st = budget / C::kStageBytes;
  if (st < 2) st = 2;
  if (st > C::kMaxStages) st = C::kMaxStages;
  cudaFuncSetAttribute(gemv_kernel<WF, NT, kCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(st));
  stages_of[dev] = st;
  return st;
}

// Cluster plan {S, clusters}: the GPC structure caps how many clusters of S CTAs are resident at
// once (e.g. 33 clusters of 8 at 2 CTAs/SM, below qkv's 36 row tiles).  Take the largest
// S <= gemv_cluster_split whose resident cluster count covers every row tile (one tile per cluster,
// queried with cudaOccupancyMaxActiveClusters); if none does, S = 1 (each CTA loops over row tiles
// with no cluster barrier).  Cached per (device, shape, hint).
struct ClusterPlan {
  int S, ncl;
  bool all_resident;
};
template <int WF, int NT>
static ClusterPlan cluster_plan(int N, int K, int sms, int hint = 0) {
  const int stages = ensure_attrs<WF, NT, true>();
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, ClusterPlan> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(current_device(), N, K, hint);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  using C = GemvCfg<WF, NT>;
  const int tiles = N / 128;
  const int per_sm = WF == 16 ? 1 : (hint > 0 ? hint : 2);
  const int S0 = gemv_cluster_split(N, K, sms, per_sm);
  auto active_of = [&](int S, int ncl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl * S);
    cfg.blockDim = dim3(kGemvThreads);
    cfg.dynamicSmemBytes = C::smem_for(stages);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = S;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, gemv_kernel<WF, NT, true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      active = ncl;   // cannot query: keep the arithmetic plan
    }
    return active;
  };
  ClusterPlan plan{1, std::max(1, std::min(tiles, sms * per_sm)), false};
  for (int S = S0; S >= 2; --S) {
    if (active_of(S, tiles) >= tiles) {
      plan = ClusterPlan{S, tiles, true};
      break;
    }
  }
  if (plan.S == 1) {
    const int act = active_of(1, plan.ncl);
    plan.ncl = std::max(1, std::min(plan.ncl, act));
    plan.all_resident = plan.ncl >= tiles;
  }
  cache[key] = plan;
  return plan;
}

// every row tile has its own resident CTA or cluster (required by EPI_RESID_NORM's in-kernel barrier)
bool gemv_tiles_all_resident(bool q4, int NT, int N, int K, int sms, int bits) {
  if (!gemv_use_cluster(N, K, sms)) return false;
  const int nt = NT <= 2 ? 2 : 4;
  if (!q4) return nt == 2 ? cluster_plan<16, 2>(N, K, sms).all_resident : cluster_plan<16, 4>(N, K, sms).all_resident;
  if (bits == 2) return nt == 2 ? cluster_plan<2, 2>(N, K, sms).all_resident : cluster_plan<2, 4>(N, K, sms).all_resident;
  return nt == 2 ? cluster_plan<4, 2>(N, K, sms).all_resident : cluster_plan<4, 4>(N, K, sms).all_resident;
}

template <int WF, int NT, bool kCluster>
static void launch_t(const GemvParams& p0, int grid, int S, bool pdl, cudaStream_t st) {
  using C = GemvCfg<WF, NT>;
  const int stages = ensure_attrs<WF, NT, kCluster>();
  GemvParams p = p0;
  p.stages = stages;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
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
  cudaLaunchKernelEx(&cfg, gemv_kernel<WF, NT, kCluster>, p);
}

template <int WF, int NT>
static void launch_mode(const GemvParams& p, int sms, bool pdl, cudaStream_t st) {
  if (gemv_use_cluster(p.N, p.K, sms)) {
    const ClusterPlan pl = cluster_plan<WF, NT>(p.N, p.K, sms, p.ctas_per_sm);
    launch_t<WF, NT, true>(p, pl.ncl * pl.S, pl.S, pdl, st);
  } else {
    const int per_sm = WF == 16 ? 1 : 2;
    launch_t<WF, NT, false>(p, gemv_grid_for(p.N, p.K, sms * per_sm), 1, pdl, st);
  }
}

// the K2 dequant-GEMV / bf16 GEMV: NT = 2 (M <= 16) or 4 (M <= 32)
void launch_gemv(bool q4, const GemvParams& p, int grid, bool pdl, cudaStream_t st) {
  const bool nt2 = p.NT <= 2;
  if (!q4) {
    nt2 ? launch_mode<16, 2>(p, grid, pdl, st) : launch_mode<16, 4>(p, grid, pdl, st);
  } else if (p.qbits == 2) {
    nt2 ? launch_mode<2, 2>(p, grid, pdl, st) : launch_mode<2, 4>(p, grid, pdl, st);
  } else {
    nt2 ? launch_mode<4, 2>(p, grid, pdl, st) : launch_mode<4, 4>(p, grid, pdl, st);
  }
}

}  // namespace ss
