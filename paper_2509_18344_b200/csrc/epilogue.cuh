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
      const int d = e.head_dim, half = d >> 1;
      const int P = *e.committed_len;
      for (int idx = tid; idx < kTileRows * ncols; idx += nthreads) {
        const int n = idx / ncols, m = idx % ncols;
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        const int row = row0 + n;
        float v = tile[n * ld + m];
        if (e.bias) v += bf2f(e.bias[row]);
        const int i = row % d;
        const int node = e.node_base + mg;
        if (row < e.q_dim + e.kv_dim) {   // q or k: rotate-half RoPE at pos = P + depth(node)
          const int partner_row = i < half ? row + half : row - half;
          float pv = tile[(partner_row - row0) * ld + m];
          if (e.bias) pv += bf2f(e.bias[partner_row]);
          const int pos = P + e.depth[node];
          const float2 cs = e.rope[pos * half + (i % half)];
          v = i < half ? (v * cs.x - pv * cs.y) : (v * cs.x + pv * cs.y);
        }
        const uint16_t b = f2bf(v);
        if (row < e.q_dim) {
          e.q_out[int64_t(mg) * e.q_dim + row] = b;
        } else if (row < e.q_dim + e.kv_dim) {
          const int kvh = (row - e.q_dim) / d;
          e.k_tree[(int64_t(kvh) * e.max_nodes + node) * d + i] = b;
        } else {
          const int kvh = (row - e.q_dim - e.kv_dim) / d;
          e.v_tree[(int64_t(kvh) * e.max_nodes + node) * d + i] = b;
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
    case EPI_SILU: {   // tile rows 0..63 gate, 64..127 up, for ffn index f = 64 r + i
      for (int idx = tid; idx < 64 * ncols; idx += nthreads) {
        const int m = idx / 64, i = idx % 64;
        const int mg = m0 + m;
        if (mg >= e.M) continue;
        const float gte = tile[i * ld + m], up = tile[(64 + i) * ld + m];
        const float a = gte / (1.0f + expf(-gte)) * up;
        e.act[fragx_offset(mg, int64_t(r) * 64 + i, e.act_nt)] = f2bf(a);
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
