// Shared building blocks of the draft GEMVs (gemv_q.cu: K2 on substitutes; gemv.cu: the tcgen05 bf16
// GEMV): pipeline geometry, work lists (cluster tiles / Stream-K), cluster and trace helpers.
#pragma once
#include "common.cuh"

namespace ss {

// The tcgen05 bf16 GEMV of gemv.cu (the head, resident layers), one CTA per SM: warp 0 producer
// (TMA), warp 1 MMA issuer + TMEM owner, warps 2..13 workers (10..13 read the TMEM accumulators, one
// lane quadrant each; all 12 run the split-K reduction and the epilogue).
template <int WF, int MV>
struct GemvShape {
  static_assert(WF == 16, "the tcgen05 GEMV is the bf16 path (substitutes: gemv_q.cu)");
  static constexpr int kMmaWarps = 1;
  static constexpr int kWarps = 14;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kMaxReg = 128;   // <= 4 warps x 128 x 32 per sub-partition
};
constexpr int kGemvWorkers = 384;        // warps 2..13
constexpr int kGemvMaxThreads = 14 * 32; // block of the bf16 GEMV (occupancy proxy)
constexpr int kGemvMaxCluster = 8;       // largest (portable) cluster the split factor may use
constexpr int kGemvSmemBudget = 227 * 1024;

// NT: token groups of 8 (MMA N = 8 NT: 16 or 32).  A stage is one 32 KB bf16 tile-chunk plus the
// matching activation chunk; TMEM holds two tile accumulators of N columns (512 columns allocated:
// the CTA is alone on its SM).
template <int WF, int NT>
struct GemvCfg {
  static_assert(WF == 16, "bf16 only");
  static constexpr int kCPS = 1;                                // tile-chunks per pipeline stage
  static constexpr int kWBytes = kBF16TileBytes;
  static constexpr int kXBytes = NT * kXChunkBytesPerNT;
  static constexpr int kN = NT * 8;                             // MMA N (tokens, padded)
  static constexpr int kSBytes = 0;
  static constexpr int kStageBytes = kCPS * (kWBytes + kXBytes + kSBytes);
  static constexpr int kMaxStages = 16;
  static constexpr int kSlots = 2;
  static constexpr int kDCols = kN;
  static constexpr int kTmemCols = 512;
  static constexpr int kMetaBytes = 0;
  static constexpr int kTileFloats = kTileRows * kN;
  static constexpr int kXPreTokens = 8;
  static constexpr int kXPreFloats = kXPreTokens * kTileRows;
  // cluster reduction staging: [S][ceil(N/S)][128] fp32 partial columns pushed by the ranks
  static constexpr int kStagingFloats = (kN + kGemvMaxCluster - 1) * kTileRows;
  static constexpr int kBars = 2 * kMaxStages + 2 + 2 + 2;     // full, empty, d_full, d_empty, xbar
  static constexpr int kFixed = kTileFloats * 4 + kStagingFloats * 4 + kMetaBytes + kBars * 8 + 64 + 512 + kXPreFloats * 4;
  static constexpr int smem_for(int S) { return S * kStageBytes + kFixed; }
  static constexpr int stages() {
    const int s = (kGemvSmemBudget - kFixed - 1024) / kStageBytes;
    return s > kMaxStages ? kMaxStages : (s < 2 ? 2 : s);
  }
  static_assert(kSlots * kDCols <= kTmemCols, "TMEM columns");
};
SS_HD int64_t owner_of(int64_t t, int64_t T, int G) { return ((t + 1) * G - 1) / T; }

SS_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace events: 0 first CTA entry (min), 1 producer dep-wait done (CTA 0), 2 consumer dep-wait done
// (CTA 0), 3 first stage arrived (CTA 0), 4 main loop done (CTA 0), 5 last flush start (CTA 0),
// 6 kernel end (max over CTAs), 7 main loop done (max over CTAs), 8 cluster reduction done (max),
// 9..12 epilogue steps (see apply_epilogue), 13..15 spare; a record is kTraceEvents u64
#define SS_TRACE_MIN(ev) do { if (p.trace) atomicMin(&p.trace[ev], gtime()); } while (0)
#define SS_TRACE_MAX(ev) do { if (p.trace) atomicMax(&p.trace[ev], gtime()); } while (0)
#define SS_TRACE_CTA0(ev) do { if (p.trace && blockIdx.x == 0) p.trace[ev] = gtime(); } while (0)

SS_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SS_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SS_DEV uint32_t cluster_nrank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
SS_DEV uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
SS_DEV uint32_t cluster_count_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
SS_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
SS_DEV float ld_dsmem_f32(const float* local, uint32_t rank) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
  return v;
}
SS_DEV void st_dsmem_f32x4(float* local, uint32_t rank, float4 v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
SS_DEV float4 ld_dsmem_f32x4(const float* local, uint32_t rank) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra) : "memory");
  return v;
}

// The tile-chunks a CTA processes, in streaming order (identical for producer and consumers).
struct Work {
  int r, c;          // current tile and chunk
  int c_begin, c_end;
  int r_step;
  int64_t left;      // items remaining
  SS_DEV int take(int cps) const {   // chunks of the current tile in the next stage (<= items left)
    int n = c_end - c;
    if (n > cps) n = cps;
    if (n > left) n = int(left);
    return n;
  }
  SS_DEV void next(int nC, int n) {
    c += n;
    if (c == c_end) {
      r += r_step;
      c = c_begin;
      if (r_step == 1 && c_end == nC) c = 0;   // Stream-K: later tiles start at chunk 0
    }
    left -= n;
  }
  SS_DEV int64_t stages(int nC, int cps) const {   // number of stages left (tile-aligned stages)
    Work w = *this;
    int64_t n = 0;
    while (w.left > 0) {
      w.next(nC, w.take(cps));
      ++n;
    }
    return n;
  }
};

// cluster / tile-owner mode: cluster cid of ncl owns row tiles cid, cid + ncl, ...; rank crank of
// csize takes the K chunks [crank*nC/csize, (crank+1)*nC/csize) of each
SS_DEV Work make_work_tiles(int N, int K, int cid, int ncl, uint32_t crank, uint32_t csize) {
  const int nC = K >> 7, n_tiles = N >> 7;
  Work w;
  w.c_begin = int(int64_t(crank) * nC / csize);
  w.c_end = int(int64_t(crank + 1) * nC / csize);
  w.r = cid;
  w.c = w.c_begin;
  w.r_step = ncl;
  const int my_tiles = cid < n_tiles ? (n_tiles - cid + ncl - 1) / ncl : 0;
  w.left = int64_t(my_tiles) * (w.c_end - w.c_begin);
  return w;
}
// Stream-K mode: CTA b of G takes the contiguous tile-chunk range [b*T/G, (b+1)*T/G)
SS_DEV Work make_work_streamk(int N, int K, int b, int G) {
  const int nC = K >> 7, n_tiles = N >> 7;
  const int64_t T = int64_t(n_tiles) * nC;
  const int64_t lo = int64_t(b) * T / G, hi = int64_t(b + 1) * T / G;
  Work w;
  w.r = int(lo / nC);
  w.c = int(lo % nC);
  w.c_begin = w.c;
  w.c_end = nC;
  w.r_step = 1;
  w.left = hi - lo;
  return w;
}
template <bool kCluster>
SS_DEV Work make_work(int N, int K, uint32_t crank, uint32_t csize) {
  if constexpr (kCluster) return make_work_tiles(N, K, int(cluster_id_x()), int(cluster_count_x()), crank, csize);
  else return make_work_streamk(N, K, blockIdx.x, gridDim.x);
}

}  // namespace ss
