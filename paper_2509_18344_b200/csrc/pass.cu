// Persistent, warp-specialised draft pass: ONE launch executes a whole draft forward of the frontier
// ("all leaf nodes are input to the draft model"; SURVEY §8(a) A2 + A3):
//   embed -> for every layer: [qkv GEMV (RMSNorm fused) -> tree attention -> o GEMV + residual ->
//   gate_up GEMV (RMSNorm fused) + SiLU*mul -> down GEMV + residual] -> head GEMV (final norm fused)
//   -> sharpened log-softmax partial top-k -> global top-k + tree append.
//
// B200 design: one CTA per SM (cooperative launch).  Warp 8 is a TMA
// producer that streams EVERY weight block of the pass (28 layers x 4 matrices + the head) through an
// S-stage shared-memory ring with cp.async.bulk; it never waits on activations, so HBM streaming
// runs ahead across phase boundaries.  Warps 0..7 consume: they stage each activation chunk into
// shared memory (fusing RMSNorm: h = bf16(x * r * g) with r from per-tile sums of squares written by
// the previous residual epilogue), run the 4-bit dequant MMAs, reduce split tiles deterministically
// (Stream-K fixup in fixed order), apply the fused epilogues, and meet at grid barriers between
// dependent phases.  Attention and top-k run as phases inside the same kernel.
#include <cooperative_groups.h>

#include "attn_warp.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace ss {

constexpr int kPConsumerWarps = 8;
constexpr int kPThreads = (kPConsumerWarps + 1) * 32;
constexpr int kPStageBytes = 2 * kQ4TileBytes;   // 2 Q4 chunks (18 KB) or a bf16 half-chunk (16 KB)
constexpr int kPMaxStages = 8;
constexpr int kPAttnWarps = 4;                    // consumer warps per CTA taking attention tasks
constexpr int kPXBuf = 4 * kXChunkBytesPerNT + 2 * 32 * 4;   // one staged activation chunk (NT <= 4)
constexpr int kPXSlots = 4;                                  // activation ring depth

SS_DEV int attn_warp_bytes(int D) { return 4 * 16 * (D + 8) * 2; }
SS_HD int pass_smem_layout(int D, int stages, int* o_bar, int* o_x, int* o_tile, int* o_misc, int* o_attn) {
  int off = stages * kPStageBytes;
  *o_bar = off;
  off += 2 * kPMaxStages * 8 + 2 * kPXSlots * 8;
  *o_x = off;
  off += kPXSlots * kPXBuf;
  *o_tile = off;
  off += kTileRows * 32 * 4;
  *o_misc = off;
  off += 2048;                                    // rnorm, scratch, flags, top-k lists (512 floats)
  *o_attn = off;
  off += kPAttnWarps * 4 * 16 * (D + 8) * 2;
  return off;
}
int pass_smem_bytes(int head_dim, int stages) {
  int a, b, c, d, e;
  return pass_smem_layout(head_dim, stages, &a, &b, &c, &d, &e);
}

SS_DEV void pbar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }   // consumers only
SS_DEV unsigned long long gclock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
SS_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// all consumer threads of all CTAs; the producer warp never takes part
SS_DEV void grid_sync(unsigned* bar, unsigned target) {
  pbar();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const unsigned long long t0 = gclock();
    while (ld_acquire(bar) < target) {
      __nanosleep(20);
      if (gclock() - t0 > 4000000000ull) __trap();   // watchdog: never hang the GPU
    }
    __threadfence();
  }
  pbar();
}
SS_DEV void mbar_wait_wd(uint64_t* bar, uint32_t parity) {   // mbarrier wait with a watchdog
  const unsigned long long t0 = gclock();
  uint32_t addr = smem_u32(bar);
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (gclock() - t0 > 4000000000ull) __trap();
  }
}

// ---- the weight stream: identical walk for producer and consumers ---------------------------
struct StageIt {
  int64_t t, hi;     // current tile-chunk and end of this CTA's range
  int nC, r, c;      // tile, chunk of t
  int q4, half;      // bf16 chunks are split into two 64-k halves (16 KB stages)
  SS_DEV void init(int64_t lo, int64_t hi_, int nC_, int q4_) {
    t = lo;
    hi = hi_;
    nC = nC_;
    r = int(lo / nC_);
    c = int(lo % nC_);
    q4 = q4_;
    half = 0;
  }
  SS_DEV bool valid() const { return t < hi; }
  SS_DEV int nch() const {   // chunks in this stage (Q4): up to 2, same tile
    if (!q4) return 1;
    const int64_t a = hi - t, b = nC - c;
    return int(a < 2 ? (b < a ? b : a) : (b < 2 ? b : 2));
  }
  SS_DEV uint32_t bytes() const { return q4 ? uint32_t(nch()) * kQ4TileBytes : uint32_t(kBF16TileBytes / 2); }
  SS_DEV const uint8_t* src(const uint8_t* W) const {
    return q4 ? W + t * kQ4TileBytes : W + t * kBF16TileBytes + half * (kBF16TileBytes / 2);
  }
  SS_DEV void next() {
    int n = 1;
    if (q4) {
      n = nch();
    } else if (!half) {
      half = 1;
      return;
    } else {
      half = 0;
    }
    t += n;
    c += n;
    if (c == nC) {
      c = 0;
      ++r;
    }
  }
};
SS_DEV void streamk_range(int64_t T, int G, int b, int64_t* lo, int64_t* hi) {
  const int Ge = int(T < G ? T : G);   // every participating CTA gets >= 1 tile-chunk
  if (b >= Ge) {
    *lo = *hi = 0;
    return;
  }
  *lo = int64_t(b) * T / Ge;
  *hi = int64_t(b + 1) * T / Ge;
}
SS_HD int64_t sk_owner(int64_t t, int64_t T, int G) { return ((t + 1) * G - 1) / T; }

// ---- RMSNorm phase: h = bf16(x * r * g) -> FragX + 64-group sums (one warp per (token, group)) ----
template <int NT>
SS_DEV void norm_phase(const PassParams& p, const PhaseDesc& d) {
  constexpr int Mpad = NT * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nG = p.H / 64, ntask = p.M * nG;
  uint16_t* hf = const_cast<uint16_t*>(d.X);
  float* hs = const_cast<float*>(d.XSUM);
  for (int task = blockIdx.x * kPConsumerWarps + warp; task < ntask; task += gridDim.x * kPConsumerWarps) {
    const int m = task / nG, g64 = task % nG;
    float ssum = 0.f;   // r = 1/sqrt(mean(x^2) + eps) from the per-tile partials, fixed order
    for (int t = 0; t < p.H / 128; ++t) ssum += __ldcg(p.sumsq + int64_t(t) * Mpad + m);
    const float r = 1.0f / sqrtf(ssum / float(p.H) + p.eps);
    float gs = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = g64 * 64 + 32 * u + lane;
      const uint16_t hb = f2bf(__ldcg(p.x + int64_t(m) * p.H + k) * r * bf2f(d.gain[k]));
      hf[fragx_offset(m, k, NT)] = hb;
      gs += bf2f(hb);
    }
    gs = warp_sum(gs);
    if (lane == 0) hs[int64_t(g64) * Mpad + m] = gs;
  }
  __threadfence();
}

// ---- one GEMV phase (consumer side) ---------------------------------------------------------
template <int NT>
SS_DEV void gemv_phase(const PassParams& p, const PhaseDesc& d, uint8_t* ring, uint64_t* full, uint64_t* empty,
                       int& s, uint32_t& ph, uint8_t* xring, uint64_t* xfull, uint64_t* xempty, int& xs,
                       uint32_t& xph, float* otile, float* scratch, int* flag) {
  constexpr int Mpad = NT * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int nC = d.K >> 7;
  const int64_t T = int64_t(d.N >> 7) * nC;
  const int G = int(T < int64_t(gridDim.x) ? T : int64_t(gridDim.x));   // effective Stream-K grid
  int64_t lo, hi;
  streamk_range(T, gridDim.x, blockIdx.x, &lo, &hi);
  EpiParams e = d.epi;
  e.M = p.M;
  e.node_base = p.node_base;
  e.act_nt = NT;
  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  auto stash = [&](float* dst) {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n0 = warp * 16 + g, m = j * 8 + 2 * t4;
      *reinterpret_cast<float2*>(dst + n0 * Mpad + m) = make_float2(acc[j][0], acc[j][1]);
      *reinterpret_cast<float2*>(dst + (n0 + 8) * Mpad + m) = make_float2(acc[j][2], acc[j][3]);
      acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    }
  };
  auto flush = [&](int r, int c_first, int c_last) {
    const bool complete = (c_first == 0 && c_last == nC - 1);
    if (complete) {
      stash(otile);
    } else {
      const int64_t first = sk_owner(int64_t(r) * nC, T, G);
      const int64_t nseg = sk_owner(int64_t(r + 1) * nC - 1, T, G) - first + 1;
      const int64_t slot = blockIdx.x - first;
      float* dst = p.partials + (int64_t(r) * p.max_seg + slot) * int64_t(kTileRows * Mpad);
      stash(dst);
      __threadfence();
      pbar();
      if (threadIdx.x == 0) {
        const int old = atomicAdd(&p.tile_ctr[r], 1);
        *flag = (old == nseg - 1);
      }
      pbar();
      if (!*flag) return;
      __threadfence();
      const float* base = p.partials + int64_t(r) * p.max_seg * int64_t(kTileRows * Mpad);
      for (int q = threadIdx.x; q < kTileRows * Mpad; q += 256) {
        float a = 0.f;
        for (int k = 0; k < nseg; ++k) a += __ldcg(base + k * int64_t(kTileRows * Mpad) + q);
        otile[q] = a;
      }
      if (threadIdx.x == 0) p.tile_ctr[r] = 0;
    }
    pbar();
    apply_epilogue(e, otile, Mpad, r, 0, Mpad, threadIdx.x, 256, scratch);
    __threadfence();
    pbar();
  };

  if (lo >= hi) return;
  StageIt it;
  it.init(lo, hi, nC, d.q4);
  int cur_r = it.r, c_first = it.c, c_last = it.c;
  const uint32_t kMagic = 0x43004300u;
  while (it.valid()) {
    if (it.r != cur_r) {
      flush(cur_r, c_first, c_last);
      cur_r = it.r;
      c_first = it.c;
    }
    const int nch = it.nch();
    c_last = it.c + nch - 1;
    mbar_wait_wd(&full[s], ph);
    const uint8_t* stage = ring + s * kPStageBytes;
    for (int ci = 0; ci < nch; ++ci) {
      // activation chunk it.c + ci arrives in X-ring slot xs (one slot per tile-chunk)
      mbar_wait_wd(&xfull[xs], xph);
      const uint8_t* xb = xring + xs * kPXBuf;
      const uint8_t* xst = xb + ((t4 * 8 + g) * 8);
      if (d.q4) {
        const uint8_t* wst = stage + ci * kQ4TileBytes;
        const float* xsum = reinterpret_cast<const float*>(xb + NT * kXChunkBytesPerNT);
#pragma unroll
        for (int Gq = 0; Gq < 2; ++Gq) {
          const uint4 cw = *reinterpret_cast<const uint4*>(wst + ((warp * 2 + Gq) * 32 + lane) * 16);
          const uint32_t m0 = *reinterpret_cast<const uint32_t*>(wst + kQ4CodeBytes + ((warp * 2 + Gq) * 16 + g) * 4);
          const uint32_t m1 = *reinterpret_cast<const uint32_t*>(wst + kQ4CodeBytes + ((warp * 2 + Gq) * 16 + g + 8) * 4);
          float cg[NT][4];
#pragma unroll
          for (int j = 0; j < NT; ++j) cg[j][0] = cg[j][1] = cg[j][2] = cg[j][3] = 0.f;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int st = 4 * Gq + k4;
            const uint32_t wg = (k4 < 2) ? cw.x : cw.y, wg8 = (k4 < 2) ? cw.z : cw.w;
            const int pp = 2 * (k4 & 1);
            const uint32_t a0 = lop3_and_or(wg >> (4 * pp), kMagic);
            const uint32_t a1 = lop3_and_or(wg8 >> (4 * pp), kMagic);
            const uint32_t a2 = lop3_and_or(wg >> (4 * pp + 4), kMagic);
            const uint32_t a3 = lop3_and_or(wg8 >> (4 * pp + 4), kMagic);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const uint2 b = *reinterpret_cast<const uint2*>(xst + (j * 8 + st) * 256);
              mma_bf16_16816(cg[j], a0, a1, a2, a3, b.x, b.y);
            }
          }
          const float s0 = __uint_as_float(m0 << 16), z0 = __uint_as_float(m0 & 0xFFFF0000u);
          const float s1 = __uint_as_float(m1 << 16), z1 = __uint_as_float(m1 & 0xFFFF0000u);
          const float zz0 = fmaf(-128.0f, s0, z0), zz1 = fmaf(-128.0f, s1, z1);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const float2 xs = *reinterpret_cast<const float2*>(xsum + Gq * Mpad + j * 8 + 2 * t4);
            acc[j][0] = fmaf(s0, cg[j][0], fmaf(zz0, xs.x, acc[j][0]));
            acc[j][1] = fmaf(s0, cg[j][1], fmaf(zz0, xs.y, acc[j][1]));
            acc[j][2] = fmaf(s1, cg[j][2], fmaf(zz1, xs.x, acc[j][2]));
            acc[j][3] = fmaf(s1, cg[j][3], fmaf(zz1, xs.y, acc[j][3]));
          }
        }
      } else {
        // bf16 half-chunk: group Gq = it.half; pieces q = 2*Gq + {0,1} -> k-steps 4*Gq .. 4*Gq+3
        const int Gq = it.half;
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          const int q = 2 * Gq + q2;
          const uint4 r0 = *reinterpret_cast<const uint4*>(stage + bf16_piece_off(warp, 0, q, lane) - Gq * (kBF16TileBytes / 2));
          const uint4 r1 = *reinterpret_cast<const uint4*>(stage + bf16_piece_off(warp, 1, q, lane) - Gq * (kBF16TileBytes / 2));
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
      if (d.q4 || it.half) {   // this activation chunk is done
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[xs]);
        if (++xs == kPXSlots) {
          xs = 0;
          xph ^= 1;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == p.stages) {
      s = 0;
      ph ^= 1;
    }
    it.next();
  }
  flush(cur_r, c_first, c_last);
}

// ---- top-k phases (K5) ----------------------------------------------------------------------
SS_DEV bool tk_better(float va, int ia, float vb, int ib) { return va > vb || (va == vb && ia < ib); }

SS_DEV void topk_block_task(const TopkParams& p, int m, int b, float* red, int* taken, float* wv, int* wi) {
  const int B = p.blocks_per_row;
  const int64_t v0 = int64_t(p.V) * b / B, v1 = int64_t(p.V) * (b + 1) / B;
  const float* l = p.logits + int64_t(m) * p.V;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float mx = -INFINITY;
  for (int64_t v = v0 + tid; v < v1; v += 256) mx = fmaxf(mx, __ldcg(l + v));
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  pbar();
  mx = red[0];
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  pbar();
  float sm = 0.f;
  for (int64_t v = v0 + tid; v < v1; v += 256) sm += expf((__ldcg(l + v) - mx) * p.inv_t);
  sm = warp_sum(sm);
  if (lane == 0) red[warp] = sm;
  pbar();
  const int base = m * B + b;
  if (tid == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    p.blk_max[base] = mx;
    p.blk_sum[base] = t;
  }
  for (int r = 0; r < p.k; ++r) {
    float bv = -INFINITY;
    int bi = INT32_MAX;
    for (int64_t v = v0 + tid; v < v1; v += 256) {
      bool tk = false;
      for (int q = 0; q < r; ++q) tk |= (taken[q] == int(v));
      const float lv = __ldcg(l + v);
      if (!tk && tk_better(lv, int(v), bv, bi)) {
        bv = lv;
        bi = int(v);
      }
    }
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (tk_better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      wv[warp] = bv;
      wi[warp] = bi;
    }
    pbar();
    if (tid == 0) {
      float cv = wv[0];
      int ci = wi[0];
      for (int w = 1; w < 8; ++w)
        if (tk_better(wv[w], wi[w], cv, ci)) {
          cv = wv[w];
          ci = wi[w];
        }
      taken[r] = ci;
      p.blk_val[int64_t(base) * p.k + r] = cv;
      p.blk_idx[int64_t(base) * p.k + r] = ci;
    }
    pbar();
  }
}

SS_DEV void topk_select_task(const TopkParams& p, float* misc) {
  const int B = p.blocks_per_row;
  float* lse = misc;          // [32]
  float* rmax = misc + 32;    // [32]
  float* sel_s = misc + 64;   // [32]
  int* sel_t = reinterpret_cast<int*>(misc + 96);
  int* sel_p = reinterpret_cast<int*>(misc + 128);
  float* wv = misc + 160;     // [8]
  int* wt = reinterpret_cast<int*>(misc + 168);
  int* wp = reinterpret_cast<int*>(misc + 176);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < p.M) {
    const int m = tid;
    float mx = -INFINITY;
    for (int b = 0; b < B; ++b) mx = fmaxf(mx, __ldcg(p.blk_max + m * B + b));
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += __ldcg(p.blk_sum + m * B + b) * expf((__ldcg(p.blk_max + m * B + b) - mx) * p.inv_t);
    rmax[m] = mx;
    lse[m] = logf(s);
  }
  pbar();
  const int ncand = p.M * B * p.k;
  for (int r = 0; r < p.k; ++r) {
    float bs = -INFINITY;
    int bt = INT32_MAX, bp = INT32_MAX;
    for (int c = tid; c < ncand; c += 256) {
      const int m = c / (B * p.k);
      const int tok = __ldcg(p.blk_idx + c);
      bool tk = false;
      for (int q = 0; q < r; ++q) tk |= (sel_t[q] == tok && sel_p[q] == m);
      if (tk) continue;
      const float lp = (__ldcg(p.blk_val + c) - rmax[m]) * p.inv_t - lse[m];
      const float sc = __ldcg(p.score + p.node_base + m) + lp;
      if (sc > bs || (sc == bs && (tok < bt || (tok == bt && m < bp)))) {
        bs = sc;
        bt = tok;
        bp = m;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (os > bs || (os == bs && (ot < bt || (ot == bt && op < bp)))) {
        bs = os;
        bt = ot;
        bp = op;
      }
    }
    if (lane == 0) {
      wv[warp] = bs;
      wt[warp] = bt;
      wp[warp] = bp;
    }
    pbar();
    if (tid == 0) {
      float s = wv[0];
      int t = wt[0], pp = wp[0];
      for (int w = 1; w < 8; ++w)
        if (wv[w] > s || (wv[w] == s && (wt[w] < t || (wt[w] == t && wp[w] < pp)))) {
          s = wv[w];
          t = wt[w];
          pp = wp[w];
        }
      sel_s[r] = s;
      sel_t[r] = t;
      sel_p[r] = pp;
    }
    pbar();
  }
  if (tid == 0) {   // canonical order: parent asc, token asc
    for (int i = 1; i < p.k; ++i) {
      const float s = sel_s[i];
      const int t = sel_t[i], pp = sel_p[i];
      int j = i - 1;
      while (j >= 0 && (sel_p[j] > pp || (sel_p[j] == pp && sel_t[j] > t))) {
        sel_s[j + 1] = sel_s[j];
        sel_t[j + 1] = sel_t[j];
        sel_p[j + 1] = sel_p[j];
        --j;
      }
      sel_s[j + 1] = s;
      sel_t[j + 1] = t;
      sel_p[j + 1] = pp;
    }
  }
  pbar();
  for (int j = warp; j < p.k; j += 8) {
    const int node = p.child_base + j, par = p.node_base + sel_p[j];
    if (lane == 0) {
      p.tok[node] = sel_t[j];
      p.parent[node] = par;
      p.depth[node] = p.child_depth;
      p.score[node] = sel_s[j];
    }
    for (int a = lane; a < p.child_depth; a += 32)
      p.anc[int64_t(node) * p.anc_stride + a] = __ldcg(p.anc + int64_t(par) * p.anc_stride + a);
    if (lane == 0) p.anc[int64_t(node) * p.anc_stride + p.child_depth] = node;
  }
}

int pass_max_segments(int N, int K, int grid) {   // Stream-K segments per tile (host)
  const int64_t nC = K / 128, T = int64_t(N / 128) * nC;
  const int G = int(T < grid ? T : grid);
  int mx = 1;
  for (int64_t r = 0; r < N / 128; ++r) {
    const int64_t a = sk_owner(r * nC, T, G), b = sk_owner((r + 1) * nC - 1, T, G);
    if (b - a + 1 > mx) mx = int(b - a + 1);
  }
  return mx;
}

// ---- the kernel -----------------------------------------------------------------------------
template <int NT, int D>
__global__ void __launch_bounds__(kPThreads, 1) draft_pass_kernel(const PassParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  int o_bar, o_x, o_tile, o_misc, o_attn;
  pass_smem_layout(D, p.stages, &o_bar, &o_x, &o_tile, &o_misc, &o_attn);
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + o_bar);
  uint64_t* empty = full + kPMaxStages;
  uint64_t* xfull = empty + kPMaxStages;
  uint64_t* xempty = xfull + kPXSlots;
  uint8_t* xring = smem + o_x;
  float* otile = reinterpret_cast<float*>(smem + o_tile);
  float* misc = reinterpret_cast<float*>(smem + o_misc);
  float* scratch = misc + 32;       // [128]
  int* flag = reinterpret_cast<int*>(misc + 160);
  float* tkmisc = misc + 256;       // top-k select scratch [184]
  uint16_t* attn_buf = reinterpret_cast<uint16_t*>(smem + o_attn);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kPConsumerWarps);
    }
    for (int i = 0; i < kPXSlots; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], kPConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int G = gridDim.x;

  if (warp == kPConsumerWarps) {
    // ------------------------------ producer: stream all weights -----------------------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      int64_t n_issued = 0;
      for (int i = 0; i < p.n_ph; ++i) {
        const PhaseDesc& d = p.ph[i];
        if (d.kind != PH_GEMV) continue;
        const int nC = d.K >> 7;
        int64_t lo, hi;
        streamk_range(int64_t(d.N >> 7) * nC, G, blockIdx.x, &lo, &hi);
        if (lo >= hi) continue;
        StageIt it;
        it.init(lo, hi, nC, d.q4);
        while (it.valid()) {
          if (n_issued >= S) mbar_wait_wd(&empty[s], ph ^ 1);
          const uint32_t bytes = it.bytes();
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s_hint(ring + s * kPStageBytes, it.src(d.W), bytes, &full[s], pol);
          ++n_issued;
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
          it.next();
        }
      }
    } else if (lane == 1) {
      // -------- activation producer: after the grid barrier that makes phase i's input ready,
      // stream its activation chunks (FragX + group sums) into the X ring
      int xs = 0;
      uint32_t xph = 0;
      int64_t n_issued = 0;
      for (int i = 0; i < p.n_ph; ++i) {
        const PhaseDesc& d = p.ph[i];
        if (d.kind != PH_GEMV) continue;
        const int nC = d.K >> 7;
        int64_t lo, hi;
        streamk_range(int64_t(d.N >> 7) * nC, G, blockIdx.x, &lo, &hi);
        if (lo >= hi) continue;
        {
          const unsigned long long t0 = gclock();
          while (ld_acquire(p.bar) < unsigned(i) * unsigned(G)) {
            __nanosleep(32);
            if (gclock() - t0 > 4000000000ull) __trap();
          }
          asm volatile("fence.proxy.async;" ::: "memory");   // generic-proxy writes -> TMA reads
        }
        constexpr uint32_t xb = NT * kXChunkBytesPerNT, sb = 2 * NT * 8 * 4;
        int c = int(lo % nC);
        for (int64_t t = lo; t < hi; ++t) {
          if (n_issued >= kPXSlots) mbar_wait_wd(&xempty[xs], xph ^ 1);
          uint8_t* dst = xring + xs * kPXBuf;
          mbar_arrive_expect_tx(&xfull[xs], xb + sb);
          bulk_g2s(dst, d.X + int64_t(c) * NT * 1024, xb, &xfull[xs]);
          bulk_g2s(dst + NT * kXChunkBytesPerNT, d.XSUM + int64_t(c) * 2 * NT * 8, sb, &xfull[xs]);
          ++n_issued;
          if (++xs == kPXSlots) {
            xs = 0;
            xph ^= 1;
          }
          if (++c == nC) c = 0;
        }
      }
    }
    return;
  }

  // -------------------------------- consumers ------------------------------------------------
  int s = 0, xs = 0;
  uint32_t ph = 0, xph = 0;
  unsigned nbar = 0;
  const int P = *p.attn.committed_len;
  for (int i = 0; i < p.n_ph; ++i) {
    const PhaseDesc& d = p.ph[i];
    if (i > 0) grid_sync(p.bar, (++nbar) * unsigned(G));
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[2 * i] = gclock();
    switch (d.kind) {
      case PH_EMBED: {
        // x[m] = embed[token], and per 128-column tile sums of squares (fixed order)
        const int nt = p.H / 128, ntask = p.M * nt;
        for (int task = blockIdx.x; task < ntask; task += G) {
          const int m = task / nt, t = task % nt;
          const int tokm = p.tok[p.node_base + m];
          float v2 = 0.f;
          if (threadIdx.x < 128) {
            const float v = bf2f(p.embed[int64_t(tokm) * p.H + t * 128 + threadIdx.x]);
            p.x[int64_t(m) * p.H + t * 128 + threadIdx.x] = v;
            v2 = v * v;
          }
          v2 = warp_sum(v2);
          if (lane == 0) scratch[warp] = v2;
          pbar();
          if (threadIdx.x == 0) p.sumsq[int64_t(t) * (NT * 8) + m] = ((scratch[0] + scratch[1]) + scratch[2]) + scratch[3];
          pbar();
        }
        __threadfence();
        break;
      }
      case PH_GEMV:
        gemv_phase<NT>(p, d, ring, full, empty, s, ph, xring, xfull, xempty, xs, xph, otile, scratch, flag);
        break;
      case PH_NORM:
        norm_phase<NT>(p, d);
        break;
      case PH_COMBINE: {
        AttnParams a = p.attn;
        a.n_q = p.M;
        a.node_base = p.node_base;
        a.out_nt = NT;
        const int dep = a.depth[p.node_base];
        const int nseg = (P + dep + 1 + a.split - 1) / a.split;
        if (nseg > 1) {
          const int nrow = p.M * a.n_heads;
          for (int row = blockIdx.x * kPConsumerWarps + warp; row < nrow; row += G * kPConsumerWarps)
            attn_combine_row<D>(a, P, row / a.n_heads, row % a.n_heads, lane);
        }
        __threadfence();
        break;
      }
      case PH_ATTN: {
        AttnParams a = p.attn;
        a.k_cache += d.layer * p.kc_layer;
        a.v_cache += d.layer * p.kc_layer;
        a.k_tree += d.layer * p.kt_layer;
        a.v_tree += d.layer * p.kt_layer;
        a.n_q = p.M;
        a.node_base = p.node_base;
        a.out_nt = NT;
        const int dep = a.depth[p.node_base];
        const int nseg = (P + dep + 1 + a.split - 1) / a.split;
        const int ntask = p.M * a.n_kv * nseg;
        if (warp < kPAttnWarps) {
          uint16_t* wb = attn_buf + warp * 4 * 16 * (D + 8);
          for (int task = blockIdx.x * kPAttnWarps + warp; task < ntask; task += G * kPAttnWarps) {
            const int qi = task / (a.n_kv * nseg), kvh = (task / nseg) % a.n_kv, seg = task % nseg;
            attn_task<D>(a, P, kvh, seg, qi, wb, nseg == 1);
          }
        }
        __threadfence();
        break;
      }
      case PH_TOPK1: {
        if (p.skip_topk) break;
        const int B = p.topk.blocks_per_row, ntask = p.M * B;
        int* taken = reinterpret_cast<int*>(misc + 192);
        for (int task = blockIdx.x; task < ntask; task += G)
          topk_block_task(p.topk, task / B, task % B, scratch, taken, misc + 224, reinterpret_cast<int*>(misc + 232));
        __threadfence();
        break;
      }
      case PH_TOPK2:
        if (blockIdx.x == 0 && !p.skip_topk) topk_select_task(p.topk, tkmisc);
        break;
    }
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[2 * i + 1] = gclock();
  }
}

template <int NT, int D>
static cudaError_t launch_t(const PassParams& p, int grid, cudaStream_t st) {
  const int smem = pass_smem_bytes(D, p.stages);
  static int done = 0;
  if (!done) {
    cudaFuncSetAttribute(draft_pass_kernel<NT, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    done = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: grid barriers are safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, draft_pass_kernel<NT, D>, p);
}

void launch_draft_pass(const PassParams& p, int grid, int head_dim, cudaStream_t st) {
  if (head_dim == 128) {
    switch (p.NT) {
      case 1: launch_t<1, 128>(p, grid, st); break;
      case 2: launch_t<2, 128>(p, grid, st); break;
      case 4: launch_t<4, 128>(p, grid, st); break;
    }
  } else {
    switch (p.NT) {
      case 1: launch_t<1, 64>(p, grid, st); break;
      case 2: launch_t<2, 64>(p, grid, st); break;
      case 4: launch_t<4, 64>(p, grid, st); break;
    }
  }
}

int pass_max_grid(int head_dim, int stages) {
  int sms = 148, blocks = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = pass_smem_bytes(head_dim, stages);
  if (head_dim == 128) {
    cudaFuncSetAttribute(draft_pass_kernel<1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, draft_pass_kernel<1, 128>, kPThreads, smem);
  } else {
    cudaFuncSetAttribute(draft_pass_kernel<1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, draft_pass_kernel<1, 64>, kPThreads, smem);
  }
  return blocks * sms;
}

}  // namespace ss
