// Epilogues applied to a complete [128 weight rows x ncols tokens] fp32 tile held in shared memory.
// out_tile[n * ld + m] = sum_k W[128*r + n, k] * X[m0 + m, k].
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace ss {

// Fused RMSNorm, second half: wait until the norm barrier counter reaches `target` (all tiles'
// residual rows and sums of squares are published), then write h = bf16(x * r_m * gain) for the
// 128 columns of tile r and tokens [0, nn) in FragX, plus the 64-group sums.  Threads [0, nthreads)
// cooperate; scratch needs 32 floats (scratch[126..127] must stay untouched).
SS_DEV void norm_finish(const EpiParams& e, int r, unsigned long long target, int nn, int ssld_tile, int tid,
                        int nthreads, float* scratch, unsigned long long* trace) {
  const int row0 = r * kTileRows;
  const int64_t ssld = e.sumsq_ld > 0 ? e.sumsq_ld : ssld_tile;
  if (tid == 0) {
    unsigned long long v, t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(e.norm_ctr) : "memory");
      if (v >= target) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 4000000000ull) __trap();   // watchdog: never hang the GPU
    }
  }
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
  if (trace && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&trace[10], t);
  }
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthreads >> 5;
  const int npairs = nn * 2;   // (token, 64-group) pairs; a warp takes 64 columns of one token
  float xv[8][2];              // x_new prefetched for this warp's pairs (<= 8 per warp)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int pr = warp + i * nwarps, m = pr >> 1, G = pr & 1;
#pragma unroll
    for (int u = 0; u < 2; ++u)
      xv[i][u] = (pr < npairs && m < e.M) ? __ldcg(e.x + int64_t(m) * e.ldx + row0 + 64 * G + 32 * u + lane) : 0.f;
  }
  // r_m = 1/sqrt(mean(x_m^2) + eps): warp m loads the per-tile partials (lane t, t + 32, ...) and
  // reduces them with a fixed shuffle tree (independent of M)
  for (int m = warp; m < nn; m += nwarps) {
    float ssum = 0.f;
    if (m < e.M)
      for (int t = lane; t < e.n_tiles; t += 32) ssum += __ldcg(e.sumsq + int64_t(t) * ssld + m);
    ssum = warp_sum(ssum);
    if (lane == 0) scratch[m] = 1.0f / sqrtf(ssum / float(e.ldx) + e.eps);
  }
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
  if (trace && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&trace[11], t);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int pr = warp + i * nwarps, m = pr >> 1, G = pr & 1;
    if (pr >= npairs) break;
    float gs = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = row0 + 64 * G + 32 * u + lane;
      uint16_t hb = 0;
      if (m < e.M) hb = f2bf(xv[i][u] * scratch[m] * bf2f(e.norm_gain[k]));
      e.norm_out[fragx_offset(m, k, e.act_nt)] = hb;
      gs += bf2f(hb);
    }
    gs = warp_sum(gs);
    if (lane == 0) e.norm_xs[int64_t(row0 / 64 + G) * (e.act_nt * 8) + m] = gs;
  }
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");   // scratch is reused by the caller
  if (trace && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&trace[12], t);
  }
}

// threads [0, nthreads) cooperate; caller syncs before and after.  Token columns [m0, m0 + ncols)
// of the tile are processed (a cluster GEMV splits a tile's tokens over its ranks).  EPI_RESID_NORM:
// every call arrives once at the norm barrier, which completes after n_tiles * arrive_per_tile
// arrivals; the norm_wait caller of a tile then writes the normalised activations of tokens
// [0, norm_ncols).
SS_DEV void apply_epilogue(const EpiParams& e, const float* tile, int ld, int r, int m0, int ncols, int tid,
                           int nthreads, float* scratch = nullptr, unsigned long long* trace = nullptr,
                           int arrive_per_tile = 1, bool norm_wait = true, int norm_ncols = 0,
                           unsigned long long* arrive_target = nullptr, const float* xpre = nullptr) {
  // xpre (optional): the residual rows x[m0 + m][128 r .. 128 r + 127] already in shared memory,
  // [ncols][128], for EPI_RESID / EPI_RESID_SS / EPI_RESID_NORM
  // debug trace (max over CTAs of %globaltimer): 9 residual stored, 10 norm barrier passed,
  // 11 r computed, 12 epilogue done
  auto tr = [&](int ev) {
    if (trace && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&trace[ev], t);
    }
  };
  const int row0 = r * kTileRows;
  switch (e.kind) {
    case EPI_QKV: {
      // item = (RoPE pair u, token m): rows (lo, lo + d/2) of one head; bias + rotate-half RoPE at
      // pos = P + depth(node) on (acc + bias) in fp32, then one bf16 rounding (reading R3).
      const int d = e.head_dim, half = d >> 1;
      const int P0 = e.committed_len[e.rq.req0];
      const int nitems = (kTileRows / 2) * ncols;
      for (int it = tid; it < nitems; it += nthreads) {
        const int u = it / ncols, m = it % ncols;
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        const int lo = (u / half) * d + (u % half), hi = lo + half;   // rows within the tile
        const int rlo = row0 + lo, rhi = row0 + hi;
        float vlo = tile[lo * ld + m], vhi = tile[hi * ld + m];
        if (e.bias) {
          vlo += bf2f(e.bias[rlo]);
          vhi += bf2f(e.bias[rhi]);
        }
        const int rb = rq_req(e.rq, mg);   // batched requests: request rb's local node, strided slot
        const int node = rb * e.rq.node_stride + e.node_base + rq_loc(e.rq, mg);
        const int P = e.rq.rows > 0 ? e.committed_len[rb] : P0;
        const int i = u % half;
        if (rlo < e.q_dim + e.kv_dim) {   // q or k head: rotate
          const float2 cs = e.rope[(P + e.depth[node]) * half + i];
          const float a = vlo * cs.x - vhi * cs.y, b = vhi * cs.x + vlo * cs.y;
          vlo = a;
          vhi = b;
        }
        const uint16_t blo = f2bf(vlo), bhi = f2bf(vhi);
        if (rlo < e.q_dim) {
          e.q_out[int64_t(mg) * e.q_dim + rlo] = blo;
          e.q_out[int64_t(mg) * e.q_dim + rhi] = bhi;
        } else if (rlo < e.q_dim + e.kv_dim) {
          const int kvh = (rlo - e.q_dim) / d, j = (rlo - e.q_dim) % d;
          uint16_t* dst = e.k_tree + (int64_t(kvh) * e.max_nodes + node) * d;
          dst[j] = blo;
          dst[j + half] = bhi;
        } else {
          const int kvh = (rlo - e.q_dim - e.kv_dim) / d, j = (rlo - e.q_dim - e.kv_dim) % d;
          uint16_t* dst = e.v_tree + (int64_t(kvh) * e.max_nodes + node) * d;
          dst[j] = blo;
          dst[j + half] = bhi;
        }
      }
      break;
    }
    case EPI_RESID: {
      for (int idx = tid; idx < kTileRows * ncols; idx += nthreads) {
        const int m = idx / kTileRows, n = idx % kTileRows;   // coalesced along n
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        float* xp = e.x + int64_t(mg) * e.ldx + row0 + n;
        *xp = (xpre ? xpre[m * kTileRows + n] : *xp) + tile[n * ld + m];
      }
      break;
    }
    case EPI_RESID_NORM: {
      // x[m, row] += y; then sum over the tile's 128 rows of x_new^2 per token, in a fixed order:
      // a warp covers 32 consecutive rows of one token -> 4 warp sums per token -> scratch -> ordered add
      const int64_t ssld = e.sumsq_ld > 0 ? e.sumsq_ld : ld;
      const int nitems = kTileRows * ncols;
      for (int base = (tid & ~31); base < nitems; base += nthreads) {
        const int it = base + (tid & 31);
        const int m = it / kTileRows, n = it % kTileRows;
        const int mg = m0 + m;
        float v2 = 0.f;
        if (it < nitems && mg < e.M) {
          float* xp = e.x + int64_t(mg) * e.ldx + row0 + n;
          const float xn = (xpre ? xpre[m * kTileRows + n] : __ldcg(xp)) + tile[n * ld + m];
          *xp = xn;
          v2 = xn * xn;
        }
        const float s = warp_sum(v2);
        if ((tid & 31) == 0 && it < nitems) scratch[m * 4 + n / 32] = s;
        __syncwarp();
      }
      asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
      for (int m = tid; m < ncols; m += nthreads) {
        const int mg = m0 + m;
        if (mg < e.M) e.sumsq[int64_t(r) * ssld + mg] = ((scratch[m * 4] + scratch[m * 4 + 1]) + scratch[m * 4 + 2]) + scratch[m * 4 + 3];
      }
      tr(9);
      // ---- fused RMSNorm ----
      // Every caller arrives at a barrier on a monotonic 64-bit counter (release add; never reset).
      // The norm_wait caller of each tile (one CTA per tile, so the waiters are few enough to be
      // co-resident) then waits for this launch's generation and normalises the tile's 128 columns
      // (norm_finish); a caller that still has other work passes norm_wait = false, keeps the
      // generation target (*arrive_target) and calls norm_finish itself later.
      asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
      if (tid == 0) {
        const unsigned long long n_arr = (unsigned long long)e.n_tiles * (unsigned long long)arrive_per_tile;
        unsigned long long old;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(e.norm_ctr) : "memory");
        const unsigned long long target = (old / n_arr + 1) * n_arr;
        if (arrive_target) *arrive_target = target;
        reinterpret_cast<unsigned long long*>(scratch)[63] = target;   // scratch[126..127]
      }
      if (!norm_wait) break;
      asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
      norm_finish(e, r, reinterpret_cast<unsigned long long*>(scratch)[63], norm_ncols > 0 ? norm_ncols : m0 + ncols, ld, tid,
                  nthreads, scratch, trace);
      break;
    }
    case EPI_SILU: {
      // tile rows 0..63 gate, 64..127 up, for ffn index f = 64 r + u (exactly one 64-group).
      // item = (token m, u); a warp covers 32 consecutive u of one token, so the group sum of the
      // bf16 activations is two warp sums combined in fixed order by the lane-0 of the first half.
      const int nitems = 64 * ncols;
      for (int base = (tid & ~31); base < nitems; base += nthreads) {
        const int it = base + (tid & 31);
        const int m = it / 64, u = it % 64;
        const int mg = m0 + m;
        const bool ok = it < nitems && mg < e.M;
        float a = 0.f;
        if (ok) {
          const float gte = tile[u * ld + m], up = tile[(64 + u) * ld + m];
          const uint16_t ab = f2bf(gte / (1.0f + expf(-gte)) * up);
          e.act[fragx_offset(mg, int64_t(r) * 64 + u, e.act_nt)] = ab;
          a = bf2f(ab);
        }
        const float s = warp_sum(a);   // u in [0,32) or [32,64) of token m
        if (e.act_xs && ok && (u == 0 || u == 32)) {
          if (scratch && ncols <= 32) {
            scratch[2 * m + (u >> 5)] = s;   // both halves in shared memory, combined below
          } else {
            float* dst = e.act_xs + int64_t(r) * (e.act_nt * 8) + mg;
            if (u == 0) *dst = s;        // first half; the second half adds after the barrier below
          }
        }
        __syncwarp();
      }
      if (e.act_xs && scratch && ncols <= 32) {
        // group sum = first half + second half (the same fixed order as the two-pass form below)
        asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
        for (int m = tid; m < ncols; m += nthreads)
          if (m0 + m < e.M) e.act_xs[int64_t(r) * (e.act_nt * 8) + m0 + m] = scratch[2 * m] + scratch[2 * m + 1];
      } else if (e.act_xs) {
        // second halves: add the u in [32, 64) sums after the first halves are stored
        asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
        for (int base = (tid & ~31); base < nitems; base += nthreads) {
          const int it = base + (tid & 31);
          const int m = it / 64, u = it % 64;
          const int mg = m0 + m;
          const bool ok = it < nitems && mg < e.M && u >= 32;
          float a = 0.f;
          if (ok) {   // recompute (bitwise identical) instead of re-reading the global store
            const float gte = tile[u * ld + m], up = tile[(64 + u) * ld + m];
            a = bf2f(f2bf(gte / (1.0f + expf(-gte)) * up));
          }
          const float s = warp_sum(a);
          if (ok && u == 32) e.act_xs[int64_t(r) * (e.act_nt * 8) + mg] += s;
          __syncwarp();
        }
      }
      break;
    }
    case EPI_LOGITS:
    case EPI_STORE: {
      for (int idx = tid; idx < kTileRows * ncols; idx += nthreads) {
        const int m = idx / kTileRows, n = idx % kTileRows;
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        e.out[int64_t(mg) * e.ldo + row0 + n] = tile[n * ld + m];
      }
      break;
    }
    case EPI_TOPK: {
      // sharpened top-k statistics of one 128-logit vocab tile per token (reading R13:
      // fp32 logits from the accumulator): warp w takes tokens w, w + nwarps, ...; lane holds rows
      // lane + 32 i; max, sum exp((l - max) / T) in a fixed shuffle order, then tk_k rounds of warp argmax
      // (value desc, index asc) with the picked row excluded
      const int warp = tid >> 5, lane = tid & 31, nwarps = nthreads >> 5;
      for (int m = warp; m < ncols; m += nwarps) {
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = tile[(lane + 32 * i) * ld + m];
        float mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
        mx = warp_max(mx);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) s += expf((v[i] - mx) * e.tk_inv_t);
        s = warp_sum(s);
        const int64_t base = int64_t(mg) * e.tk_tiles + r;
        if (lane == 0) {
          e.tk_max[base] = mx;
          e.tk_sum[base] = s;
        }
        for (int q = 0; q < e.tk_k; ++q) {
          float bv = -INFINITY;
          int bi = 0x7fffffff;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (v[i] > bv) {   // i ascending: the first of equal values has the smaller row
              bv = v[i];
              bi = lane + 32 * i;
            }
          for (int o = 16; o; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
              bv = ov;
              bi = oi;
            }
          }
          if (lane == 0) {
            e.tk_val[base * e.tk_k + q] = bv;
            e.tk_idx[base * e.tk_k + q] = row0 + bi;
          }
          if ((bi & 31) == lane) v[bi >> 5] = -INFINITY;   // excluded from the next rounds
        }
      }
      break;
    }
    case EPI_ARGMAX: {   // one thread per token column: max, first argmax, second max over the 128 rows
      for (int m = tid; m < ncols; m += nthreads) {
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        float best = -INFINITY, second = -INFINITY;
        int bi = 0;
        for (int n = 0; n < kTileRows; ++n) {
          const float v = tile[n * ld + m];
          if (v > best) {
            second = best;
            best = v;
            bi = n;
          } else if (v > second) {
            second = v;
          }
        }
        e.am_val[int64_t(mg) * e.am_tiles + r] = best;
        e.am_idx[int64_t(mg) * e.am_tiles + r] = row0 + bi;
        e.am_second[int64_t(mg) * e.am_tiles + r] = second;
      }
      break;
    }
  }
}

}  // namespace ss
