// K2-MLP — the draft MLP of one layer (gate/up with SiLU*mul, then down with
// the residual add and the next RMSNorm) as ONE persistent launch of resident CTAs.
//
// Phase A: CTA b computes gate_up row tiles b, b + G, ... over the full K (no split, no reduction),
//          applies the SiLU*mul epilogue (activations + their group sums, R3 rounding
//          points) and publishes a per-tile flag (release).
// Phase B: Stream-K over down's tile-chunks (CTA b takes the contiguous range [bT/G, (b+1)T/G), so
//          every CTA streams the same number of bytes); the producer issues a stage's weights at
//          once but its activation chunk c only after gate_up tiles 2c and 2c+1 have published
//          (acquire), so down starts while the slowest gate_up tiles are still running and the
//          kernel boundary (launch + dependency latency, ~5 us) disappears.  Partial tiles are
//          reduced in segment order by the last-arriving CTA, which runs the epilogue (residual, and
//          with EPI_RESID_NORM the fused RMSNorm barrier among the tile finishers).
// All CTAs are co-resident (grid = occupancy x SMs), so the flag and norm waits cannot deadlock.
#include "common.cuh"
#include "epilogue.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

#include <cstdio>
#include <cstdlib>

namespace ss {

constexpr int kFlagStride = 32;   // one flag per 128-byte line: pollers do not share L2 lines

SS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SS_DEV int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SS_DEV void wait_flag(const int* f) {
  if (ld_acquire_s32(f)) return;
  const unsigned long long t0 = gtime();
  while (!ld_acquire_s32(f)) {
    __nanosleep(256);
    if (gtime() - t0 > 4000000000ull) __trap();   // watchdog: never hang the GPU
  }
}

template <bool Q4, int NT>
__global__ void __launch_bounds__(kGemvThreads, SS_GEMV_MIN_BLOCKS) mlp_kernel(const MlpParams p) {
  using C = GemvCfg<Q4, NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int kStages = p.stages;
  uint8_t* ring = smem;
  float* otile = reinterpret_cast<float*>(smem + kStages * C::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes + (C::kTileFloats + C::kStagingFloats) * 4);
  uint64_t* empty = full + C::kMaxStages;
  int* flag = reinterpret_cast<int*>(empty + C::kMaxStages);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(flag) + 64);   // [128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;
  const int Ngu = 2 * p.F, nCa = p.H >> 7, nCd = p.F >> 7;
  const int Mpad = NT * 8;
  if (threadIdx.x == 0) SS_TRACE_MIN(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch();

  if (warp == kGemvConsumerWarps) {
    // ------------------------------ producer -------------------------------
    {
      Work wa = (p.dbg & 4) ? Work{0, 0, 0, 0, 1, 0} : make_work_tiles(Ngu, p.H, b, G, 0, 1);
      const int64_t Td = int64_t(p.H >> 7) * nCd;
      const int Gd = int(Td < G ? Td : G);
      Work wb = b < Gd ? make_work_streamk(p.H, p.F, b, Gd) : Work{0, 0, 0, 0, 1, 0};
      const int64_t nA = wa.stages(nCa, C::kCPS), nB = wb.stages(nCd, C::kCPS);
      const uint64_t pol = policy_evict_first();
      constexpr uint32_t kFull = C::kWBytes + C::kXBytes + C::kSBytes;
      auto slot_wait = [&](int64_t i) {   // stage i reuses slot i % S after round i / S - 1 was consumed
        if (i >= kStages) mbar_wait(&empty[i % kStages], uint32_t((i / kStages) - 1) & 1);
      };
      auto issue_w = [&](int64_t i, const uint8_t* W, int nC, const Work& ww, int n) {
        const int st = int(i % kStages);
        mbar_arrive_expect_tx(&full[st], uint32_t(n) * kFull);
        bulk_g2s_hint(ring + st * C::kStageBytes, W + (int64_t(ww.r) * nC + ww.c) * C::kWBytes, uint32_t(n) * C::kWBytes,
                      &full[st], pol);
      };
      auto issue_x = [&](int64_t i, const uint16_t* X, const float* XS, const Work& ww, int n) {
        const int st = int(i % kStages);
        uint8_t* base = ring + st * C::kStageBytes + C::kCPS * C::kWBytes;
        bulk_g2s(base, X + int64_t(ww.c) * NT * 1024, uint32_t(n) * C::kXBytes, &full[st]);
        if constexpr (Q4) bulk_g2s(base + C::kCPS * C::kXBytes, XS + int64_t(ww.c) * 2 * NT * 8, uint32_t(n) * C::kSBytes, &full[st]);
      };
      // phase A (lane 0): the weights of the first stages go out before the grid-dependency wait
      if (lane == 0) {
        const int64_t pre = nA < kStages ? nA : kStages;
        Work wx = wa;
        for (int64_t i = 0; i < pre; ++i) {
          const int n = wa.take(C::kCPS);
          issue_w(i, p.Wgu, nCa, wa, n);
          wa.next(nCa, n);
        }
        griddep_wait();
        for (int64_t i = 0; i < pre; ++i) {
          const int n = wx.take(C::kCPS);
          issue_x(i, p.Xh, p.XSh, wx, n);
          wx.next(nCa, n);
        }
        for (int64_t i = pre; i < nA; ++i) {
          slot_wait(i);
          const int n = wa.take(C::kCPS);
          issue_w(i, p.Wgu, nCa, wa, n);
          issue_x(i, p.Xh, p.XSh, wa, n);
          wa.next(nCa, n);
        }
      }
      // this CTA's down weights do not depend on phase A: pull them toward L2 now (one contiguous
      // range per covered tile), so phase B's copies hit L2 once the flags are up
      if (lane == 0 && nB > 0 && !(p.dbg & 2) && (p.dbg & 8)) {
        const int64_t lo = int64_t(b) * Td / Gd, hi = int64_t(b + 1) * Td / Gd;
        for (int64_t u = lo; u < hi;) {
          const int64_t r = u / nCd, ue = (r + 1) * nCd < hi ? (r + 1) * nCd : hi;
          const uint8_t* src = p.Wd + (r * nCd + (u - r * nCd)) * C::kWBytes;
          for (int64_t off = 0; off < (ue - u) * C::kWBytes; off += 65536) {
            const int64_t nb = (ue - u) * C::kWBytes - off;
            prefetch_l2(src + off, uint32_t(nb < 65536 ? nb : 65536));
          }
          u = ue;
        }
      }
      __syncwarp();
      // phase B: the whole warp waits (acquire, 32 flags per poll) for every gate_up tile this CTA's
      // down chunks read, then lane 0 streams.  The acquires precede every phase-B copy.
      if (nB > 0 && !(p.dbg & 6)) {
        const int64_t lo = b < Gd ? int64_t(b) * Td / Gd : 0, hi = b < Gd ? int64_t(b + 1) * Td / Gd : 0;
        for (int64_t r = lo / nCd; r * nCd < hi; ++r) {
          const int c0 = int(lo > r * nCd ? lo - r * nCd : 0);
          const int c1 = int(hi < (r + 1) * nCd ? hi - r * nCd : nCd);
          const int t0 = (p.dbg & 1) ? 0 : 2 * c0, t1 = (p.dbg & 1) ? (Ngu >> 7) : 2 * c1;
          for (int base = t0; base < t1; base += 32) {
            const int t = base + lane;
            bool ok = t >= t1;
            const unsigned long long ts = gtime();
            for (;;) {
              if (!ok) ok = ld_acquire_s32(p.flags + kFlagStride * t) != 0;
              if (__all_sync(0xffffffffu, ok)) break;
              __nanosleep(256);
              if (gtime() - ts > 4000000000ull) __trap();   // watchdog: never hang the GPU
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        for (int64_t j = 0; j < ((p.dbg & 2) ? 0 : nB); ++j) {
          const int64_t i = nA + j;
          slot_wait(i);
          const int n = wb.take(C::kCPS);
          issue_w(i, p.Wd, nCd, wb, n);
          issue_x(i, p.Xa, p.XSa, wb, n);
          wb.next(nCd, n);
        }
      }
    }
    return;
  }

  // ------------------------------ consumers --------------------------------
  griddep_wait();
  const int nthr = kGemvConsumerWarps * 32;
  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  auto consume = [&](int nch) {
    mbar_wait(&full[s], ph);
    consume_stage<Q4, NT>(ring + s * C::kStageBytes, nch, acc, warp, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kStages) {
      s = 0;
      ph ^= 1;
    }
  };

  // ---- phase A: gate_up tiles, SiLU*mul epilogue, publish ----
  auto flush_a = [&](int r) {
    stash_acc<NT>(acc, otile, warp, lane);
    named_bar(1, nthr);
    apply_epilogue(p.epi_gu, otile, Mpad, r, 0, Mpad, threadIdx.x, nthr, scratch);
    fence_proxy_async();   // the activations are read by TMA (async proxy) in other CTAs
    named_bar(1, nthr);
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p.flags + kFlagStride * r), "r"(1) : "memory");
    }
  };
  {
    Work wa = (p.dbg & 4) ? Work{0, 0, 0, 0, 1, 0} : make_work_tiles(Ngu, p.H, b, G, 0, 1);
    const bool any = wa.left > 0;
    int cur_r = wa.r;
    while (wa.left > 0) {
      if (wa.r != cur_r) {
        flush_a(cur_r);
        cur_r = wa.r;
      }
      const int nch = wa.take(C::kCPS);
      consume(nch);
      wa.next(nCa, nch);
    }
    if (any) flush_a(cur_r);
  }
  if (threadIdx.x == 0) {
    SS_TRACE_CTA0(4);
    SS_TRACE_MAX(7);
  }

  // ---- phase B: down, Stream-K, fixed-order fixup, residual (+ RMSNorm) epilogue ----
  const int64_t Td = int64_t(p.H >> 7) * nCd;
  const int Gd = int(Td < G ? Td : G);   // Stream-K grid: every participating CTA owns >= 1 chunk
  constexpr int kMaxFin = 8;
  __shared__ int fin[kMaxFin];
  __shared__ unsigned long long norm_target;
  int n_fin = 0;
  auto flush_b = [&](int r, int c_first, int c_last) {
    const bool complete = (c_first == 0 && c_last == nCd - 1);
    if (complete) {
      stash_acc<NT>(acc, otile, warp, lane);
    } else {
      const int64_t first = owner_of(int64_t(r) * nCd, Td, Gd);
      const int64_t nseg = owner_of(int64_t(r + 1) * nCd - 1, Td, Gd) - first + 1;
      const int64_t slot = b - first;
      stash_acc<NT>(acc, p.partials + (int64_t(r) * p.max_seg + slot) * int64_t(kTileRows * Mpad), warp, lane);
      __threadfence();
      named_bar(1, nthr);
      if (threadIdx.x == 0) {
        const int old = atomicAdd(&p.counters[r], 1);
        *flag = (old == nseg - 1);
      }
      named_bar(1, nthr);
      if (!*flag) return;
      __threadfence();
      // segment-order sum; each thread's float4 of every segment is loaded before any add
      const float4* base = reinterpret_cast<const float4*>(p.partials + int64_t(r) * p.max_seg * int64_t(kTileRows * Mpad));
      for (int e = threadIdx.x; e < kTileRows * Mpad / 4; e += nthr) {
        constexpr int kB = 16;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q0 = 0; q0 < nseg; q0 += kB) {
          float4 part[kB];
#pragma unroll
          for (int q = 0; q < kB; ++q)
            if (q0 + q < nseg) part[q] = __ldcg(base + (q0 + q) * int64_t(kTileRows * Mpad / 4) + e);
#pragma unroll
          for (int q = 0; q < kB; ++q)
            if (q0 + q < nseg) {
              v.x += part[q].x;
              v.y += part[q].y;
              v.z += part[q].z;
              v.w += part[q].w;
            }
        }
        reinterpret_cast<float4*>(otile)[e] = v;
      }
      if (threadIdx.x == 0) p.counters[r] = 0;
    }
    named_bar(1, nthr);
    if (threadIdx.x == 0) SS_TRACE_MAX(8);
    // a CTA may finish a tile and still own chunks of the next one: it only arrives at the norm
    // barrier here and normalises its finished tiles after all of its work (norm_finish below)
    apply_epilogue(p.epi_d, otile, Mpad, r, 0, Mpad, threadIdx.x, nthr, scratch, p.trace, 1, false, Mpad, &norm_target);
    if (threadIdx.x == 0 && n_fin < kMaxFin) fin[n_fin] = r;
    ++n_fin;
    named_bar(1, nthr);
  };
  {
    Work wb = (b < Gd && !(p.dbg & 2)) ? make_work_streamk(p.H, p.F, b, Gd) : Work{0, 0, 0, 0, 1, 0};
    const int64_t n_items = wb.left;
    int cur_r = wb.r, c_first = wb.c, c_last = wb.c;
    bool first = true;
    while (wb.left > 0) {
      if (wb.r != cur_r) {
        flush_b(cur_r, c_first, c_last);
        cur_r = wb.r;
        c_first = wb.c;
      }
      const int nch = wb.take(C::kCPS);
      c_last = wb.c + nch - 1;
      consume(nch);
      if (first && threadIdx.x == 0) SS_TRACE_CTA0(3);
      first = false;
      wb.next(nCd, nch);
    }
    if (threadIdx.x == 0) SS_TRACE_MAX(5);
    if (n_items > 0) flush_b(cur_r, c_first, c_last);
  }
  if (p.epi_d.kind == EPI_RESID_NORM && n_fin > 0) {
    if (n_fin > kMaxFin) __trap();   // more finished tiles than a CTA can defer (grid << tiles)
    named_bar(1, nthr);
    for (int i = 0; i < n_fin; ++i)
      norm_finish(p.epi_d, fin[i], norm_target, Mpad, Mpad, threadIdx.x, nthr, scratch, p.trace);
  }
  // ---- exit: the last CTA out clears the flags for the next launch ----
  named_bar(1, nthr);
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.exit_ctr) : "memory");
    if (old == G - 1) {
      for (int t = 0; t < (Ngu >> 7); ++t) p.flags[kFlagStride * t] = 0;
      *p.exit_ctr = 0;
    }
    SS_TRACE_MAX(6);
  }
}

static int env_int_mlp(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <bool Q4, int NT>
static int mlp_setup(int sms, int* stages_out) {   // grid (all resident) and ring depth
  using C = GemvCfg<Q4, NT>;
  static int stages = 0, grid = -1;
  if (grid < 0) {
    const int budget = env_int_mlp("SS_GEMV_RING_KB", 88) * 1024;
    int st = budget / C::kStageBytes;
    if (st < 2) st = 2;
    if (st > C::kMaxStages) st = C::kMaxStages;
    stages = st;
    cudaFuncSetAttribute(mlp_kernel<Q4, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem_for(st));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mlp_kernel<Q4, NT>, kGemvThreads, C::smem_for(st)) !=
        cudaSuccess) {
      cudaGetLastError();
      per_sm = 0;
    }
    const int want = env_int_mlp("SS_GEMV_CTAS_PER_SM", 2);
    grid = sms * (per_sm < want ? per_sm : want);
    if (getenv("SS_VERBOSE")) fprintf(stderr, "mlp<%d,%d>: grid %d stages %d per_sm %d smem %d\n", int(Q4), NT, grid, st, per_sm, C::smem_for(st));
  }
  if (stages_out) *stages_out = stages;
  return grid;
}

int mlp_grid(bool q4, int NT, int sms) {
  switch (NT) {
    case 1: return q4 ? mlp_setup<true, 1>(sms, nullptr) : mlp_setup<false, 1>(sms, nullptr);
    case 2: return q4 ? mlp_setup<true, 2>(sms, nullptr) : mlp_setup<false, 2>(sms, nullptr);
    case 4: return q4 ? mlp_setup<true, 4>(sms, nullptr) : mlp_setup<false, 4>(sms, nullptr);
    default: return 0;
  }
}

template <bool Q4, int NT>
static void launch_t(const MlpParams& p0, int grid, bool pdl, cudaStream_t st) {
  using C = GemvCfg<Q4, NT>;
  int stages = 0;
  mlp_setup<Q4, NT>(0, &stages);   // configured by mlp_grid()
  MlpParams p = p0;
  p.stages = stages;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = C::smem_for(stages);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  static const int as_cluster = env_int_mlp("SS_MLP_CLUSTER1", 1);
  if (as_cluster) {   // a cluster launch of size 1 (the scheduler places clusters GPC-aware)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
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
  cudaLaunchKernelEx(&cfg, mlp_kernel<Q4, NT>, p);
}

void launch_mlp(bool q4, const MlpParams& p, int grid, bool pdl, cudaStream_t st) {
  switch (p.NT) {
    case 1: q4 ? launch_t<true, 1>(p, grid, pdl, st) : launch_t<false, 1>(p, grid, pdl, st); break;
    case 2: q4 ? launch_t<true, 2>(p, grid, pdl, st) : launch_t<false, 2>(p, grid, pdl, st); break;
    case 4: q4 ? launch_t<true, 4>(p, grid, pdl, st) : launch_t<false, 4>(p, grid, pdl, st); break;
    default: break;
  }
}

}  // namespace ss
