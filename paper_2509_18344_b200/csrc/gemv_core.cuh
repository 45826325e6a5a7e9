// K2 building blocks of the dequant-GEMV kernel (gemv.cu): pipeline geometry, work lists, and the
// per-stage tensor-core consumer (see gemv.cu's header for the design).
#pragma once
#include "common.cuh"

namespace ss {

// Warp roles of the tcgen05 K2 kernel (gemv.cu), one CTA per SM: 0 producer (TMA), 1 MMA issuer +
// TMEM owner, 2..9 convert (quadrant w % 4, 64-group (w - 2) / 4 of every tile-chunk: 4-/2-bit codes ->
// bf16 A operand in TMEM), 10..13 accumulate (quadrant w % 4: per-group TMEM accumulators -> fp32
// rows), 14.. further MMA issuers.  Substitutes use 2 (MV = 32) or 4 MMA warps: warp (G, parity)
// issues the MMAs of 64-group G of the tile-chunks of that parity (MMA issue from one thread is ~13
// instructions per tcgen05.mma and shares its sub-partition with three busy warps).  Warps 2..13
// (384 threads) run the split-K reduction and epilogue.
template <int WF, int MV>
struct GemvShape {
  static constexpr int kMmaWarps = WF == 16 ? 1 : (MV <= 16 ? 4 : 2);
  static constexpr int kWarps = 14 + (kMmaWarps > 1 ? kMmaWarps - 1 : 0);
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kMaxReg = kWarps > 16 ? 96 : 128;   // <= 5 warps x 96 x 32 per sub-partition
};
constexpr int kGemvMaxThreads = 17 * 32;
constexpr int kGemvWorkers = 384;        // warps 2..13
constexpr int kGemvMaxCluster = 8;       // largest (portable) cluster the split factor may use
constexpr int kGemvSmemBudget = 227 * 1024;

// WF: weight format, 16 = bf16 (A from shared memory), 4 / 2 = group-64 substitutes (A dequantised
// into TMEM).  NT: token groups of 8 (MMA N = 8 NT: 16 or 32).
template <int WF, int NT>
struct GemvCfg {
  static constexpr bool kQ = WF != 16;
  static constexpr int kCPS = kQ ? 2 : 1;                       // tile-chunks per pipeline stage
  static constexpr int kWBytes = WF == 16 ? kBF16TileBytes : (WF == 2 ? kQ2TileBytes : kQ4TileBytes);
  static constexpr int kCodeBytes = WF == 2 ? kQ2CodeBytes : kQ4CodeBytes;
  static constexpr int kXBytes = NT * kXChunkBytesPerNT;
  static constexpr int kN = NT * 8;                             // MMA N (tokens, padded)
  static constexpr int kSBytes = kQ ? 2 * kN * 4 : 0;           // group sums of x: [2 groups][N] fp32
  static constexpr int kStageBytes = kCPS * (kWBytes + kXBytes + kSBytes);
  static constexpr int kMaxStages = 16;
  // TMEM (all 512 columns): Q: 4 chunk slots of accumulators (2 groups x N columns) then 4 A slots of
  // 64 columns (128 k as bf16 pairs); bf16: 2 tile slots of N columns
  static constexpr int kSlots = kQ ? 4 : 2;
  static constexpr int kDCols = kQ ? 2 * kN : kN;
  static constexpr int kACol0 = kSlots * kDCols;
  static constexpr int kTmemCols = 512;
  static constexpr int kMetaSlots = 8;                          // scale/zero + group-sum side buffer
  static constexpr int kMetaBytes = kQ ? kMetaSlots * (2 * kTileRows * 4 + 2 * kN * 4) : 0;
  static constexpr int kTileFloats = kTileRows * kN;
  static constexpr int kXPreTokens = 8;
  static constexpr int kXPreFloats = kXPreTokens * kTileRows;
  // cluster reduction staging: [S][ceil(N/S)][128] fp32 partial columns pushed by the ranks
  static constexpr int kStagingFloats = (kN + kGemvMaxCluster - 1) * kTileRows;
  static constexpr int kBars = 2 * kMaxStages + 3 * 4 + 2 + 2;   // full, empty, go, a_empty, d_full, d_empty, xbar
  static constexpr int kFixed = kTileFloats * 4 + kStagingFloats * 4 + kMetaBytes + kBars * 8 + 64 + 512 + kXPreFloats * 4;
  static constexpr int smem_for(int S) { return S * kStageBytes + kFixed; }
  static constexpr int stages() {
    const int s = (kGemvSmemBudget - kFixed - 1024) / kStageBytes;
    return s > kMaxStages ? kMaxStages : (s < 2 ? 2 : s);
  }
  static_assert(kACol0 + (kQ ? kSlots * 64 : 0) <= kTmemCols, "TMEM columns");
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
