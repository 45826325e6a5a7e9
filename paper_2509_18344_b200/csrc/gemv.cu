// The draft's bf16 GEMV on the 5th-generation tensor cores (tcgen05): the head (N = vocab, with the
// EPI_TOPK epilogue of K5: per vocab tile max, sum exp((l - max)/T) and top-k, so draft logits never
// reach HBM) and the GPU-resident layers of a planner placement.
// Y[M x N] = X[M x K] * W^T for M = frontier tokens <= 32.
//
// B200 design:
//  * weights are 128-row x 128-k tile-chunks in the core-matrix layout (common.cuh) -- directly the A
//    operand of tcgen05.mma (SWIZZLE_NONE descriptors, LBO 128 B, SBO 2048 B); the activations, in the
//    same layout, are the B operand (N = 8..32 tokens).  Warp 0 streams stages with cp.async.bulk
//    (TMA) into an mbarrier ring, issuing the weight part of the first stages before
//    griddepcontrol.wait (PDL); warp 1's elected lane issues the MMAs into TMEM accumulators (two
//    slots, so a tile's MMAs overlap the previous tile's read-out); worker warps read TMEM with
//    tcgen05.ld and run the fused epilogues;
//  * narrow matrices use cluster split-K with a push-based DSMEM reduction in rank order; the tall
//    head uses Stream-K with a fixed-order fixup by the last-arriving CTA.
// The WF = 4 / 2 template branches are the tcgen05 dequant-GEMV measured against the mma.sync K2 in
// DESIGN.md §7 (converter warps dequantise codes into TMEM, per-64-group TMEM accumulators); no
// launcher instantiates them -- the product K2 is gemv_q.cu.
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

// MV: token columns that carry tokens (8 when M <= 8, else N): the accumulator registers per row.
// One CTA per SM (the whole TMEM); 14 warps spread 4,4,3,3 over the sub-partitions: <= 128 registers.
template <int WF, int NT, bool kCluster, int MV>
__global__ void __maxnreg__((GemvShape<WF, MV>::kMaxReg)) gemv_kernel(const GemvParams p) {
  using C = GemvCfg<WF, NT>;
  using Sh = GemvShape<WF, MV>;
  constexpr int kN = C::kN;
  static_assert(MV == 8 || MV == kN, "MV");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int kStages = p.stages;
  uint8_t* ring = smem;
  float* otile = reinterpret_cast<float*>(smem + kStages * C::kStageBytes);
  float* staging = otile + C::kTileFloats;
  uint8_t* metabuf = reinterpret_cast<uint8_t*>(staging + C::kStagingFloats);
  uint64_t* full = reinterpret_cast<uint64_t*>(metabuf + C::kMetaBytes);
  uint64_t* empty = full + C::kMaxStages;
  uint64_t* d_full = empty + C::kMaxStages;    // tile accumulator ready (two TMEM slots)
  uint64_t* d_empty = d_full + 2;              // tile accumulator consumed
  uint64_t* xbar = d_empty + 2;                // residual-row prefetch
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
      mbar_init(&empty[s], 1);   // the MMA warp's commit
    }
    for (int j = 0; j < 2; ++j) mbar_init(&d_full[j], 1);
    for (int j = 0; j < 2; ++j) mbar_init(&d_empty[j], 4);
    mbar_init(xbar, 1);
    fence_barrier_init();
  }
  // producer: the weight part of the first stages does not depend on the previous kernel or on TMEM;
  // issue it before the TMEM allocation
  Work wp = make_work<kCluster>(p.N, p.K, crank, csize);
  const int64_t n_stage_p = wp.stages(nC, C::kCPS);
  const int pre = int(n_stage_p < kStages ? n_stage_p : kStages);
  const uint64_t pol = policy_evict_first();
  const uint32_t per_chunk = uint32_t(C::kWBytes + C::kXBytes + C::kSBytes);
  auto issue_w = [&](int st, const Work& ww, int n) {
    mbar_arrive_expect_tx(&full[st], uint32_t(n) * per_chunk);
    bulk_g2s_hint(ring + st * C::kStageBytes, p.W + (int64_t(ww.r) * nC + ww.c) * C::kWBytes, uint32_t(n) * C::kWBytes,
                  &full[st], pol);
  };
  const Work wx0 = wp;   // replayed for the activation copies of the prefetched stages
  if (threadIdx.x == 0)
    for (int i = 0; i < pre; ++i) {
      const int n = wp.take(C::kCPS);
      issue_w(i, wp, n);
      wp.next(nC, n);
    }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // a CTA alone on its SM that allocates all 512 columns always receives column 0, lane 0: the MMA
  // warp uses the constant address (immediates instead of per-MMA register-to-uniform moves)
  const uint32_t tbase = 0;
  if (threadIdx.x == 32 && *tmem_slot != 0) __trap();
  griddep_launch();
  // a CTA with two or more tiles in a cluster of > 1 would need one cluster barrier per tile from
  // every warp; the launcher only plans clusters of one tile each (csize > 1) or csize == 1
  const bool cl_sync = kCluster && csize > 1;
  // debug (built with -DSS_GTRACE): per-chunk clock64 events of CTA 0 (gtrace[c * 8 + e], first 64)
  auto gtr = [&](int g, int e) {
#ifdef SS_GTRACE
    if (p.gtrace && blockIdx.x == 0 && g < 64) p.gtrace[g * 16 + e] = clock64();
#endif
  };

  if (warp == 0) {
    // ------------------------------ producer (TMA) -------------------------------
    Work w = wp;   // continues after the prefetched stages
    if (lane == 0) {
      Work wx = wx0;
      auto issue_x = [&](int st, const Work& ww, int n) {
        uint8_t* base = ring + st * C::kStageBytes + C::kCPS * C::kWBytes;
        bulk_g2s(base, p.X + int64_t(ww.c) * NT * 1024, uint32_t(n) * C::kXBytes, &full[st]);
      };
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
      for (int64_t i = pre; i < n_stage_p; ++i) {
        gtr(int(2 * i), 8);
        mbar_wait(&empty[st], (ph - 1) & 1);
        gtr(int(2 * i), 9);
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
    // ------------------------------ MMA issuer (one elected lane issues) --------------------------
    // per stage: 8 MMAs (M = 128 rows, N = tokens, K = 16) into the tile's TMEM slot tc % 2; the
    // stage is released by a commit to its "empty" barrier, the tile's accumulator by one to d_full
    Work w = make_work<kCluster>(p.N, p.K, crank, csize);
    constexpr uint32_t idesc = umma_idesc_bf16(kN);
    int s = 0;
    uint32_t ph = 0;
    uint32_t tc = 0;   // tile counter
    const uint32_t ring0 = smem_u32(ring);
    while (w.left > 0) {
      const int cur_r = w.r;
      bool first = true;
      do {
        const int nch = w.take(C::kCPS);
        mbar_wait(&full[s], ph);
        gtr(int(tc), 11);
        tc_fence_after();
        const uint32_t sb = ring0 + s * C::kStageBytes;
        const uint64_t xdesc = umma_desc(sb + C::kCPS * C::kWBytes, 128, 2048);   // B: token groups at 2048 B
        w.next(nC, nch);
        const bool last = w.left == 0 || w.r != cur_r;
        const uint32_t j = tc & 1;
        if (first) {
          mbar_wait(&d_empty[j], ((tc >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const uint64_t wdesc = umma_desc(sb, 128, 2048);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss_w(tbase + j * C::kDCols, wdesc + uint64_t(kk * 16), xdesc + uint64_t(kk * 16), idesc,
                    (first && kk == 0) ? 0u : 1u);
        if (last) {
          umma_commit_w(&d_full[j]);
          ++tc;
        }
        umma_commit_w(&empty[s]);
        first = false;
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      } while (w.left > 0 && w.r == cur_r);
    }
    named_bar(3, 128 + 32 * Sh::kMmaWarps);   // every MMA issued and the accumulate warps have read the last one
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc(tbase, C::kTmemCols);
    }
    if (cl_sync) cluster_sync_all();
    return;
  }

  // ---------------------------- worker warps 2..13 ----------------------------
  griddep_wait();
  if (warp >= 2 + kGemvWorkers / 32) return;    // (no further roles)
  const int tid = threadIdx.x - 64;             // 0..383 over the worker warps
  const int q = warp & 3;                       // TMEM lane quadrant of this warp
  const int row = 32 * q + lane;                // weight row of the tile owned in TMEM
  const uint32_t tl = tbase + (uint32_t(32 * q) << 16);
  const bool is_acc = warp >= 10;               // TMEM readers 10..13 (one lane quadrant each); 2..9 epilogue only

  uint32_t xph = 0;   // phase of xbar
  // --- split-K reduction + epilogue of tile r from otile (worker threads only) ---
  auto flush = [&](int r, int c_first, int c_last, bool last) {
    const int nthr = kGemvWorkers;
    named_bar(1, nthr);   // otile written by the accumulate warps
    if constexpr (kCluster) {
      if (csize == 1) {
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
  // the tile's rows -> otile: token-major [N][128] in cluster mode with csize > 1 (the push layout),
  // row-major [128][N] otherwise (the epilogue / Stream-K partial layout); columns >= MV carry no token
  auto to_otile = [&](const float (&y)[MV]) {
    const bool tok_major = kCluster && csize > 1;
#pragma unroll
    for (int t = 0; t < MV; ++t) otile[tok_major ? t * kTileRows + row : row * kN + t] = y[t];
  };

  Work w = make_work<kCluster>(p.N, p.K, crank, csize);
  const int64_t n_items = w.left;
  int s = 0;
  uint32_t ph = 0;
  uint32_t tc = 0;
  while (w.left > 0) {
    const int cur_r = w.r, c_first = w.c;
    int c_last = w.c;
    float y[MV];
#pragma unroll
    for (int t = 0; t < MV; ++t) y[t] = 0.f;
    do {
      const int nch = w.take(C::kCPS);
      c_last = w.c + nch - 1;
      const uint8_t* stage = ring + s * C::kStageBytes;
      if (tid == 0 && w.left == n_items) {
        SS_TRACE_CTA0(3);
        if (ct) ct[2] = gtime();
      }
      w.next(nC, nch);
      const bool last_of_tile = w.left == 0 || w.r != cur_r;
      if (is_acc && last_of_tile) {   // the tile's accumulator, K reduced by the MMAs
        const uint32_t j = tc & 1;
        mbar_wait(&d_full[j], (tc >> 1) & 1);
        tc_fence_after();
        uint32_t d[MV];
        if constexpr (MV == 8) {
          uint32_t d8[8];
          tmem_ld8(tl + j * C::kDCols, d8);
#pragma unroll
          for (int t = 0; t < 8; ++t) d[t] = d8[t];
        } else {
#pragma unroll
          for (int h = 0; h < MV / 16; ++h) {
            uint32_t d16[16];
            tmem_ld16(tl + j * C::kDCols + h * 16, d16);
#pragma unroll
            for (int t = 0; t < 16; ++t) d[16 * h + t] = d16[t];
          }
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[j]);
#pragma unroll
        for (int t = 0; t < MV; ++t) y[t] = __uint_as_float(d[t]);
      }
      if (last_of_tile) ++tc;
    
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    } while (w.left > 0 && w.r == cur_r);
    const bool last = w.left == 0;
    if (is_acc) {
      to_otile(y);
      if (last) named_bar(3, 128 + 32 * Sh::kMmaWarps);   // let warp 1 free TMEM: every accumulator read
    }
    if (last && tid == 0) {
      SS_TRACE_CTA0(4);
      SS_TRACE_MAX(7);
      if (ct) ct[3] = gtime();
    }
    flush(cur_r, c_first, c_last, last);
  }
  if (n_items == 0 && is_acc) named_bar(3, 128 + 32 * Sh::kMmaWarps);   // no work: still release warp 1
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
// Stream-K grid of a tall matrix
int gemv_streamk_grid(bool q4, int N, int K, int sms) {
  (void)q4;
  return gemv_grid_for(N, K, sms);   // one CTA per SM
}

static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// ring stages of an instantiation (one CTA per SM: the ring takes what the 227 KB leave); sets its
// smem attribute once per device (function attributes are per device).
template <int WF, int NT, bool kCluster, int MV>
static int ensure_attrs() {
  using C = GemvCfg<WF, NT>;
  static std::mutex mu;
  static std::map<int, int> stages_of;
  std::lock_guard<std::mutex> lk(mu);
  const int dev = current_device();
  auto it = stages_of.find(dev);
  if (it != stages_of.end()) return it->second;
  const int st = C::stages();
  cudaFuncSetAttribute(gemv_kernel<WF, NT, kCluster, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(st));
  // the whole unified L1/shared array as shared memory
  cudaFuncSetAttribute(gemv_kernel<WF, NT, kCluster, MV>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  stages_of[dev] = st;
  return st;
}

// The occupancy calculator reports 1 resident CTA per SM for any kernel that allocates TMEM (measured,
// tools/probes/occ_probe.cu, although the hardware co-schedules two: tools/probes/coresid_probe.cu).
// Cluster residency is queried on a proxy kernel with the same block size and dynamic shared memory.
__global__ void __launch_bounds__(kGemvMaxThreads) gemv_occ_proxy(int) {}

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
  const int stages = ensure_attrs<WF, NT, true, GemvCfg<WF, NT>::kN>();
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, ClusterPlan> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(current_device(), N, K, hint);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  using C = GemvCfg<WF, NT>;
  const int tiles = N / 128;
  const int per_sm = 1;   // one CTA per SM (the whole TMEM)
  (void)hint;
  const int S0 = gemv_cluster_split(N, K, sms, per_sm);
  auto active_of = [&](int S, int ncl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl * S);
    cfg.blockDim = dim3(kGemvMaxThreads);
    cfg.dynamicSmemBytes = C::smem_for(stages);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = S;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int active = 0;
    cudaFuncSetAttribute(gemv_occ_proxy, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(stages));
    cudaFuncSetAttribute(gemv_occ_proxy, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaOccupancyMaxActiveClusters(&active, gemv_occ_proxy, &cfg) != cudaSuccess) {
      cudaGetLastError();
      active = ncl;   // cannot query: keep the arithmetic plan
    }
    return active;
  };
  ClusterPlan plan{1, std::max(1, std::min(tiles, sms * per_sm)), false};
  for (int S = S0; S >= 2; --S) {
    if (std::min(active_of(S, tiles), sms * per_sm / S) >= tiles) {
      plan = ClusterPlan{S, tiles, true};
      break;
    }
  }
  if (plan.S == 1) {
    const int act = std::min(active_of(1, plan.ncl), sms * per_sm);
    plan.ncl = std::max(1, std::min(plan.ncl, act));
    plan.all_resident = plan.ncl >= tiles;
  }
  cache[key] = plan;
  return plan;
}

// every row tile has its own resident cluster (required by EPI_RESID_NORM's in-kernel barrier)
bool gemv_tiles_all_resident(bool q4, int NT, int N, int K, int sms, int bits) {
  if (q4) return gemv_q_tiles_all_resident(NT, N, K, sms, bits);
  if (!gemv_use_cluster(N, K, sms)) return false;
  return NT <= 2 ? cluster_plan<16, 2>(N, K, sms).all_resident : cluster_plan<16, 4>(N, K, sms).all_resident;
}

template <int WF, int NT, bool kCluster, int MV>
static void launch_t(const GemvParams& p0, int grid, int S, bool pdl, cudaStream_t st) {
  using C = GemvCfg<WF, NT>;
  const int stages = ensure_attrs<WF, NT, kCluster, MV>();
  GemvParams p = p0;
  p.stages = stages;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GemvShape<WF, MV>::kThreads);
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
  cudaLaunchKernelEx(&cfg, gemv_kernel<WF, NT, kCluster, MV>, p);
}

template <int WF, int NT, int MV>
static void launch_mode(const GemvParams& p, int sms, bool pdl, cudaStream_t st) {
  if (gemv_use_cluster(p.N, p.K, sms)) {
    const ClusterPlan pl = cluster_plan<WF, NT>(p.N, p.K, sms, p.ctas_per_sm);
    launch_t<WF, NT, true, MV>(p, pl.ncl * pl.S, pl.S, pdl, st);
  } else {
    launch_t<WF, NT, false, MV>(p, gemv_grid_for(p.N, p.K, sms), 1, pdl, st);
  }
}

// the draft GEMVs: substitutes on the mma.sync kernel (gemv_q.cu), bf16 on tcgen05 (this file);
// NT = 2 (M <= 16) or 4 (M <= 32)
void launch_gemv(bool q4, const GemvParams& p, int grid, bool pdl, cudaStream_t st) {
  if (q4) {
    launch_gemv_q(p, grid, pdl, st);
    return;
  }
  const int mode = p.NT > 2 ? 2 : (p.epi.M <= 8 ? 0 : 1);   // M <= 8: 8 accumulator columns per row
  if (mode == 0) launch_mode<16, 2, 8>(p, grid, pdl, st);
  else if (mode == 1) launch_mode<16, 2, 16>(p, grid, pdl, st);
  else launch_mode<16, 4, 32>(p, grid, pdl, st);
}

}  // namespace ss
