// K2 building blocks of the dequant-GEMV kernel (gemv.cu): pipeline geometry, work lists, and the
// per-stage tensor-core consumer (see gemv.cu's header for the design).
#pragma once
#include "common.cuh"

namespace ss {

constexpr int kGemvConsumerWarps = 8;
constexpr int kGemvThreads = (kGemvConsumerWarps + 1) * 32;
constexpr int kGemvMaxCluster = 8;   // largest (portable) cluster the split factor may use
#ifndef SS_GEMV_MIN_BLOCKS
#define SS_GEMV_MIN_BLOCKS 2
#endif

template <bool Q4, int NT, int QB = 4>   // QB: code bits of a quantised (Q4 = true) matrix, 4 or 2
struct GemvCfg {
  static constexpr int kCPS = Q4 ? 2 : 1;                       // tile-chunks per pipeline stage
  static constexpr int kWBytes = Q4 ? (QB == 2 ? kQ2TileBytes : kQ4TileBytes) : kBF16TileBytes;
  static constexpr int kCodeBytes = QB == 2 ? kQ2CodeBytes : kQ4CodeBytes;
  static constexpr int kXBytes = NT * kXChunkBytesPerNT;
  static constexpr int kSBytes = Q4 ? 2 * NT * 8 * 4 : 0;       // group sums of x: [2 groups][Mpad] fp32
  static constexpr int kStageBytes = kCPS * (kWBytes + kXBytes + kSBytes);
  static constexpr int kMaxStages = 16;
  static constexpr int kTileFloats = kTileRows * NT * 8;
  // residual rows of a tile's owned tokens (<= 8), TMA-prefetched before the split-K reduction
  static constexpr int kXPreTokens = 8;
  static constexpr int kXPreFloats = kXPreTokens * kTileRows;
  // cluster reduction staging: [S][ceil(Mpad/S)][128] fp32 partial columns pushed by the ranks,
  // S <= kGemvMaxCluster -> at most (Mpad + kGemvMaxCluster - 1) x 128 floats
  static constexpr int kStagingFloats = (NT * 8 + kGemvMaxCluster - 1) * kTileRows;
  // runtime stage count S: ring S*stage + out tile + staging + 2*kMaxStages barriers
  static constexpr int smem_for(int S) {
    return S * kStageBytes + kTileFloats * 4 + kStagingFloats * 4 + 2 * kMaxStages * 8 + 64 + 512 + kXPreFloats * 4;
  }
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

// One pipeline stage (nch tile-chunks of weights + the matching activation chunks + group sums)
// accumulated into this warp's 16 rows x Mpad tokens.
template <bool Q4, int NT, int QB = 4>
SS_DEV void consume_stage(const uint8_t* stage, int nch, float (&acc)[NT][4], int warp, int lane) {
  // warp: row warp (rows 16 warp .. +15 of the tile)
  using C = GemvCfg<Q4, NT, QB>;
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t kMagic = 0x43004300u;   // bf16x2 (128, 128)
#pragma unroll
  for (int ci = 0; ci < C::kCPS; ++ci) {
    if (ci >= nch) break;
    const uint8_t* wst = stage + ci * C::kWBytes;
    const uint8_t* xst = stage + C::kCPS * C::kWBytes + ci * C::kXBytes + ((t4 * 8 + g) * 8);
    if constexpr (Q4) {
      const float* xsum = reinterpret_cast<const float*>(stage + C::kCPS * (C::kWBytes + C::kXBytes) + ci * C::kSBytes);
#pragma unroll
      for (int G = 0; G < 2; ++G) {
        uint4 cw;
        if constexpr (QB == 2) {   // [row g word][row g+8 word], 16 codes each
          const uint2 c2 = *reinterpret_cast<const uint2*>(wst + ((warp * 2 + G) * 32 + lane) * 8);
          cw = make_uint4(c2.x, 0u, c2.y, 0u);
        } else {
          cw = *reinterpret_cast<const uint4*>(wst + ((warp * 2 + G) * 32 + lane) * 16);
        }
        const uint32_t m0 = *reinterpret_cast<const uint32_t*>(wst + C::kCodeBytes + ((warp * 2 + G) * 16 + g) * 4);
        const uint32_t m1 = *reinterpret_cast<const uint32_t*>(wst + C::kCodeBytes + ((warp * 2 + G) * 16 + g + 8) * 4);
        // one accumulator chain per token tile (the 8 consumer warps x 2 CTAs hide the MMA latency;
        // a second chain would cost 4 FADDs per group in an issue-bound loop)
        float cg[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) cg[j][0] = cg[j][1] = cg[j][2] = cg[j][3] = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int st = 4 * G + k4;
          uint32_t a0, a1, a2, a3;
          if constexpr (QB == 2) {   // pairs 2 k4 (a0/a1) and 2 k4 + 1 (a2/a3) at bit 2p
            a0 = lop3_and_or2(cw.x >> (4 * k4), kMagic);
            a1 = lop3_and_or2(cw.z >> (4 * k4), kMagic);
            a2 = lop3_and_or2(cw.x >> (4 * k4 + 2), kMagic);
            a3 = lop3_and_or2(cw.z >> (4 * k4 + 2), kMagic);
          } else {
            const uint32_t wg = (k4 < 2) ? cw.x : cw.y, wg8 = (k4 < 2) ? cw.z : cw.w;
            const int pp = 2 * (k4 & 1);
            a0 = lop3_and_or(wg >> (4 * pp), kMagic);
            a1 = lop3_and_or(wg8 >> (4 * pp), kMagic);
            a2 = lop3_and_or(wg >> (4 * pp + 4), kMagic);
            a3 = lop3_and_or(wg8 >> (4 * pp + 4), kMagic);
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint2 b = *reinterpret_cast<const uint2*>(xst + (j * 8 + st) * 256);
            mma_bf16_16816(cg[j], a0, a1, a2, a3, b.x, b.y);
          }
        }
        // y += s * sum((128 + c) x) + (z - 128 s) * sum(x)      (exact affine dequant, fp32)
        const float s0 = __uint_as_float(m0 << 16), z0 = __uint_as_float(m0 & 0xFFFF0000u);
        const float s1 = __uint_as_float(m1 << 16), z1 = __uint_as_float(m1 & 0xFFFF0000u);
        const float zz0 = fmaf(-128.0f, s0, z0), zz1 = fmaf(-128.0f, s1, z1);   // exact
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const float2 xs = *reinterpret_cast<const float2*>(xsum + G * NT * 8 + j * 8 + 2 * t4);
          acc[j][0] = fmaf(s0, cg[j][0], fmaf(zz0, xs.x, acc[j][0]));
          acc[j][1] = fmaf(s0, cg[j][1], fmaf(zz0, xs.y, acc[j][1]));
          acc[j][2] = fmaf(s1, cg[j][2], fmaf(zz1, xs.x, acc[j][2]));
          acc[j][3] = fmaf(s1, cg[j][3], fmaf(zz1, xs.y, acc[j][3]));
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r0 = *reinterpret_cast<const uint4*>(wst + bf16_piece_off(warp, 0, q, lane));
        const uint4 r1 = *reinterpret_cast<const uint4*>(wst + bf16_piece_off(warp, 1, q, lane));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int st = 2 * q + hh;
          const uint32_t a0 = hh ? r0.z : r0.x, a2 = hh ? r0.w : r0.y;
          const uint32_t a1 = hh ? r1.z : r1.x, a3 = hh ? r1.w : r1.y;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint2 b = *reinterpret_cast<const uint2*>(xst + (j * 8 + st) * 256);
            mma_bf16_16816(acc[j], a0, a1, a2, a3, b.x, b.y);
          }
        }
      }
    }
  }
}

// accumulators -> [128 x Mpad] fp32 tile (row-major in n), then clear
template <int NT>
SS_DEV void stash_acc(float (&acc)[NT][4], float* dst, int warp, int lane) {
  const int g = lane >> 2, t4 = lane & 3, Mpad = NT * 8;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int n0 = warp * 16 + g, m = j * 8 + 2 * t4;
    *reinterpret_cast<float2*>(dst + n0 * Mpad + m) = make_float2(acc[j][0], acc[j][1]);
    *reinterpret_cast<float2*>(dst + (n0 + 8) * Mpad + m) = make_float2(acc[j][2], acc[j][3]);
    acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  }
}

}  // namespace ss
