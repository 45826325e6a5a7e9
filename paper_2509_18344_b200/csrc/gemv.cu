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

template <bool Q4, int NT, bool kCluster, int QB = 4>
__global__ void __launch_bounds__(kGemvThreads, SS_GEMV_MIN_BLOCKS) gemv_kernel(const GemvParams p) {
  constexpr int CW = kGemvConsumerWarps;
  using C = GemvCfg<Q4, NT, QB>;
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
        if constexpr (Q4)
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
  const int g = lane >> 2, t4 = lane & 3;
  const int nthr = CW * 32;
  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  auto stash = [&](float* dst) { stash_acc<NT>(acc, dst, warp, lane); };   // [128][Mpad] partial tile

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
#pragma unroll
      for (int j = 0; j < NT; ++j) {   // token-major [Mpad][128] partial tile
        const int n0 = warp * 16 + g, m = j * 8 + 2 * t4;
        otile[m * kTileRows + n0] = acc[j][0];
        otile[(m + 1) * kTileRows + n0] = acc[j][1];
        otile[m * kTileRows + n0 + 8] = acc[j][2];
        otile[(m + 1) * kTileRows + n0 + 8] = acc[j][3];
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
      }
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
      consume_stage<Q4, NT, QB>(ring + s * C::kStageBytes, nch, acc, warp, lane);
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

static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// ring stages of an instantiation; sets its smem/cluster attributes once per device (function
// attributes are per device)
template <bool Q4, int NT, bool kCluster, int QB = 4>
static int ensure_attrs() {
  using C = GemvCfg<Q4, NT, QB>;
  static std::mutex mu;
  static std::map<int, int> stages_of;
  std::lock_guard<std::mutex> lk(mu);
  const int dev = current_device();
  auto it = stages_of.find(dev);
  if (it != stages_of.end()) return it->second;
  // Q2 stages are smaller: a 72 KB budget keeps two CTAs per SM (the Q4/bf16 rings round 88 KB
  // down to ~68 KB of whole stages)
  const int budget = (QB == 2 ? 72 : 88) * 1024;
  int st = budget / C::kStageBytes;
  if (st < 2) st = 2;
  if (st > C::kMaxStages) st = C::kMaxStages;
  cudaFuncSetAttribute(gemv_kernel<Q4, NT, kCluster, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(st));
  stages_of[dev] = st;
  return st;
}

// Cluster plan {S, clusters}: the GPC structure caps how many clusters of S CTAs are resident at
// once (e.g. 33 clusters of 8 at 2 CTAs/SM, below qkv's 36 row tiles), and a tile whose cluster is
// not resident waits for a second wave.  Take the largest S <= gemv_cluster_split whose resident
// cluster count covers every row tile (queried with cudaOccupancyMaxActiveClusters).  Cached per
// (device, shape, hint).
struct ClusterPlan {
  int S, ncl;
  bool all_resident;
};
template <bool Q4, int NT, int QB = 4>
static ClusterPlan cluster_plan(int N, int K, int sms, int hint = 0) {
  const int stages = ensure_attrs<Q4, NT, true, QB>();
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, ClusterPlan> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(current_device(), N, K, hint);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  using C = GemvCfg<Q4, NT, QB>;
  const int tiles = N / 128;
  const int per_sm = hint > 0 ? hint : 2;
  const int S0 = gemv_cluster_split(N, K, sms, hint);
  ClusterPlan plan{S0, 0, false};
  for (int S = S0; S >= 1; --S) {
    int ncl = sms * per_sm / S;
    if (ncl > tiles) ncl = tiles;
    if (ncl < 1) ncl = 1;
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
    if (cudaOccupancyMaxActiveClusters(&active, gemv_kernel<Q4, NT, true, QB>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      active = ncl;   // cannot query: keep the arithmetic plan
    }
    if (S == S0) plan = ClusterPlan{S0, active < ncl ? active : ncl, active >= tiles};
    if (active >= tiles) {
      plan = ClusterPlan{S, tiles, true};
      break;
    }
  }
  if (plan.ncl < 1) plan.ncl = 1;
  cache[key] = plan;
  return plan;
}

// every row tile has its own resident cluster (required by EPI_RESID_NORM's in-kernel barrier)
bool gemv_tiles_all_resident(bool q4, int NT, int N, int K, int sms, int bits) {
  if (!gemv_use_cluster(N, K, sms)) return false;
  if (q4 && bits == 2) {
    switch (NT) {
      case 1: return cluster_plan<true, 1, 2>(N, K, sms).all_resident;
      case 2: return cluster_plan<true, 2, 2>(N, K, sms).all_resident;
      case 3: return cluster_plan<true, 3, 2>(N, K, sms).all_resident;
      case 4: return cluster_plan<true, 4, 2>(N, K, sms).all_resident;
      default: return false;
    }
  }
  switch (NT) {
    case 1: return q4 ? cluster_plan<true, 1>(N, K, sms).all_resident : cluster_plan<false, 1>(N, K, sms).all_resident;
    case 2: return q4 ? cluster_plan<true, 2>(N, K, sms).all_resident : cluster_plan<false, 2>(N, K, sms).all_resident;
    case 3: return q4 ? cluster_plan<true, 3>(N, K, sms).all_resident : cluster_plan<false, 3>(N, K, sms).all_resident;
    case 4: return q4 ? cluster_plan<true, 4>(N, K, sms).all_resident : cluster_plan<false, 4>(N, K, sms).all_resident;
    default: return false;
  }
}

template <bool Q4, int NT, bool kCluster, int QB = 4>
static void launch_t(const GemvParams& p0, int grid, int S, bool pdl, cudaStream_t st) {
  using C = GemvCfg<Q4, NT, QB>;
  const int stages = ensure_attrs<Q4, NT, kCluster, QB>();
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
  cudaLaunchKernelEx(&cfg, gemv_kernel<Q4, NT, kCluster, QB>, p);
}

template <bool Q4, int NT, int QB = 4>
static void launch_mode(const GemvParams& p, int sms, bool pdl, cudaStream_t st) {
  if (gemv_use_cluster(p.N, p.K, sms)) {
    const ClusterPlan pl = cluster_plan<Q4, NT, QB>(p.N, p.K, sms, p.ctas_per_sm);
    launch_t<Q4, NT, true, QB>(p, pl.ncl * pl.S, pl.S, pdl, st);
  } else {
    launch_t<Q4, NT, false, QB>(p, gemv_grid_for(p.N, p.K, sms), 1, pdl, st);
  }
}

void launch_gemv(bool q4, const GemvParams& p, int grid, bool pdl, cudaStream_t st) {
  if (q4 && p.qbits == 2) {   // 2-bit substitutes (NEXT-3)
    switch (p.NT) {
      case 1: launch_mode<true, 1, 2>(p, grid, pdl, st); break;
      case 2: launch_mode<true, 2, 2>(p, grid, pdl, st); break;
      case 3: launch_mode<true, 3, 2>(p, grid, pdl, st); break;
      case 4: launch_mode<true, 4, 2>(p, grid, pdl, st); break;
      default: break;
    }
    return;
  }
  switch (p.NT) {
    case 1: q4 ? launch_mode<true, 1>(p, grid, pdl, st) : launch_mode<false, 1>(p, grid, pdl, st); break;
    case 2: q4 ? launch_mode<true, 2>(p, grid, pdl, st) : launch_mode<false, 2>(p, grid, pdl, st); break;
    case 3: q4 ? launch_mode<true, 3>(p, grid, pdl, st) : launch_mode<false, 3>(p, grid, pdl, st); break;
    case 4: q4 ? launch_mode<true, 4>(p, grid, pdl, st) : launch_mode<false, 4>(p, grid, pdl, st); break;
    default: break;
  }
}

}  // namespace ss
