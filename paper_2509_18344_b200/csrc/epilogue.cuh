// Epilogues applied to a complete [128 weight rows x ncols tokens] fp32 tile held in shared memory.
// out_tile[n * ld + m] = sum_k W[128*r + n, k] * X[m0 + m, k].
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace ss {

// threads [0, nthreads) cooperate; caller syncs before and after.
SS_DEV void apply_epilogue(const EpiParams& e, const float* tile, int ld, int r, int m0, int ncols, int tid,
                           int nthreads) {
  const int row0 = r * kTileRows;
  switch (e.kind) {
    case EPI_QKV: {
      // item = (RoPE pair u, token m): rows (lo, lo + d/2) of one head; bias + rotate-half RoPE at
      // pos = P + depth(node) on (acc + bias) in fp32, then one bf16 rounding (reading R3).
      const int d = e.head_dim, half = d >> 1;
      const int P = *e.committed_len;
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
        const int node = e.node_base + mg;
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
        e.x[int64_t(mg) * e.ldx + row0 + n] += tile[n * ld + m];
      }
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
          float* dst = e.act_xs + int64_t(r) * (e.act_nt * 8) + mg;
          if (u == 0) *dst = s;        // first half; the second half adds after the barrier below
        }
        __syncwarp();
      }
      if (e.act_xs) {
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
