// K3 tree-attention building blocks (the per-(kv head, node) CTA of attn_node_kernel).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace ss {

SS_DEV void cp_async16(void* dst_smem, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst_smem)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
SS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
SS_DEV uint32_t pack_bf16(float lo, float hi) {
  return uint32_t(f2bf(lo)) | (uint32_t(f2bf(hi)) << 16);
}
SS_DEV void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}

// ---------------------------------------------------------------------------------------------
// K3 v2: a cluster of S CTAs per (kv head, query node); warp w of rank q processes the node's logical
// 16-key tiles t = w + 8q, w + 8q + 8S, ... (online softmax, tensor-core QK^T / PV).  Each CTA merges
// its 8 per-warp partials in shared memory in warp order, then rank q finalises head rows q, q + S, ...
// by merging the S rank partials read through distributed shared memory in rank order (fixed).  No
// combine kernel.  The reduction order depends only on the node's logical key count (S is fixed), so
// a node's output is bitwise the same in a tree (verify) and as an AR step (batch invariance).
// smem: 8 warps x 2 buffers x (K, V) x 16 x (D+8) bf16 + merge area 8 x 16 x (D+2) fp32 + the
// rank partial 16 x (D+4) fp32.
template <int D>
SS_DEV void attn_node_cta(const AttnParams& p, int kvh, int qi, uint8_t* sm, int rank = 0, int S = 1) {
  constexpr int RS = D + 8;
  constexpr int TILE = 16 * RS;
  constexpr int PIECES = 16 * D * 2 / 16;
  const int grp = p.n_heads / p.n_kv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int req = rq_req(p.rq, qi);   // batched requests: request req, local node, strided state
  const int node = req * p.rq.node_stride + p.node_base + rq_loc(p.rq, qi);
  auto trace_max = [&](int ev) {
    if (p.trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&p.trace[ev], t);
    }
  };
  // prologue: the group's query rows (16 rows x D, one coalesced 16-byte load per thread), P and the
  // node's depth are independent loads issued together; the first K/V stage goes out before the
  // query fragments are read back with ldmatrix
  constexpr int QRS = D + 8;   // padded smem row (conflict-free ldmatrix)
  uint4 qv = make_uint4(0u, 0u, 0u, 0u);
  const int q_row = threadIdx.x / (D / 8), q_col = (threadIdx.x % (D / 8)) * 8;
  if (q_row < grp && q_row < 16)
    qv = __ldcg(reinterpret_cast<const uint4*>(p.q + (int64_t(qi) * p.n_heads + kvh * grp + q_row) * D + q_col));
  const int P = __ldcg(p.committed_len + req);
  const int dep = __ldcg(p.depth + node);
  const int nkeys = P + dep + 1;
  const int ntiles = (nkeys + 15) / 16;
  uint16_t* ks = reinterpret_cast<uint16_t*>(sm) + warp * 4 * TILE;
  float* mrg = reinterpret_cast<float*>(sm + 8 * 4 * TILE * 2);   // [8 warps][16 rows][D + 2]
  float* cm = mrg + 8 * 16 * (D + 2);   // this rank's partial [16][D + 4] (16-byte aligned rows)
  uint16_t* qs = reinterpret_cast<uint16_t*>(mrg);                 // query rows [16][QRS] (before the merge)
  const int* an = p.anc + int64_t(node) * p.anc_stride;   // ancestor slots are request-local
  const uint16_t* kc = p.k_cache + (int64_t(kvh) * p.max_ctx + int64_t(req) * p.rq.ctx_stride) * D;
  const uint16_t* vc = p.v_cache + (int64_t(kvh) * p.max_ctx + int64_t(req) * p.rq.ctx_stride) * D;
  const uint16_t* kt = p.k_tree + (int64_t(kvh) * p.max_nodes + int64_t(req) * p.rq.node_stride) * D;
  const uint16_t* vt = p.v_tree + (int64_t(kvh) * p.max_nodes + int64_t(req) * p.rq.node_stride) * D;
  auto stage = [&](int t, int buf) {
    uint16_t* kd = ks + buf * 2 * TILE;
    uint16_t* vd = kd + TILE;
#pragma unroll
    for (int i = 0; i < PIECES / 32; ++i) {
      const int pc = lane + 32 * i;
      const int r = pc / (D / 8), col = (pc % (D / 8)) * 8;
      const int kl = t * 16 + r;
      const bool valid = kl < nkeys;
      const int64_t row = !valid ? 0 : (kl < P ? int64_t(kl) : int64_t(an[kl - P]));
      const uint16_t* ksrc = (kl < P || !valid) ? kc : kt;
      const uint16_t* vsrc = (kl < P || !valid) ? vc : vt;
      cp_async16(kd + r * RS + col, ksrc + row * D + col, valid);
      cp_async16(vd + r * RS + col, vsrc + row * D + col, valid);
    }
    cp_async_commit();
  };
  const int t_first0 = warp + 8 * rank;
  if (t_first0 < ntiles) stage(t_first0, 0);
  if (q_row < 16) *reinterpret_cast<uint4*>(qs + q_row * QRS + q_col) = qv;
  __syncthreads();
  uint32_t qa[D / 16][4];
  {
    const int lr = (lane & 7) + ((lane >> 3) & 1) * 8, lc = (lane >> 4) * 8;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t addr = smem_u32(qs + lr * QRS + kk * 16 + lc);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(qa[kk][0]), "=r"(qa[kk][1]), "=r"(qa[kk][2]), "=r"(qa[kk][3])
                   : "r"(addr));
    }
  }
  int buf = 0;
  const int t_first = t_first0, t_step = 8 * S;
  trace_max(2);
  const float sl2 = rsqrtf(float(D)) * 1.4426950408889634f;
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  for (int t = t_first; t < ntiles; t += t_step) {
    if (t + t_step < ntiles) {
      stage(t + t_step, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const uint16_t* kd = ks + buf * 2 * TILE;
    const uint16_t* vd = kd + TILE;
    float sc[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
      const uint16_t* kr = kd + (j * 8 + g) * RS + 2 * t4;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + kk * 16);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + kk * 16 + 8);
        mma_bf16_16816(sc[j], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool ok = t * 16 + j * 8 + 2 * t4 + e < nkeys;
        sc[j][e] = ok ? sc[j][e] * sl2 : -INFINITY;
        sc[j][2 + e] = ok ? sc[j][2 + e] * sl2 : -INFINITY;
        mx0 = fmaxf(mx0, sc[j][e]);
        mx1 = fmaxf(mx1, sc[j][2 + e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - nm0), a1 = exp2f(m1 - nm1);
    m0 = nm0;
    m1 = nm1;
    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sc[j][e] = exp2f(sc[j][e] - m0);
        sc[j][2 + e] = exp2f(sc[j][2 + e] - m1);
        ps0 += sc[j][e];
        ps1 += sc[j][2 + e];
      }
    l0 = l0 * a0 + ps0;
    l1 = l1 * a1 + ps1;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      o[j][0] *= a0;
      o[j][1] *= a0;
      o[j][2] *= a1;
      o[j][3] *= a1;
    }
    const uint32_t pa0 = pack_bf16(sc[0][0], sc[0][1]), pa1 = pack_bf16(sc[0][2], sc[0][3]);
    const uint32_t pa2 = pack_bf16(sc[1][0], sc[1][1]), pa3 = pack_bf16(sc[1][2], sc[1][3]);
    const int lr = lane & 15, ld_off = (lane >> 4) * 8;
#pragma unroll
    for (int nd = 0; nd < D / 8; nd += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_trans(b0, b1, b2, b3, vd + lr * RS + nd * 8 + ld_off);
      mma_bf16_16816(o[nd], pa0, pa1, pa2, pa3, b0, b1);
      mma_bf16_16816(o[nd + 1], pa0, pa1, pa2, pa3, b2, b3);
    }
    __syncwarp();
    buf ^= 1;
  }
  trace_max(3);
  __syncthreads();   // qs (aliasing the merge area) is no longer read
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  // per-warp partial (rows = head rows 0..15 of this kv group) -> merge area
  float* mw = mrg + warp * 16 * (D + 2);
#pragma unroll
  for (int nd = 0; nd < D / 8; ++nd) {
    *reinterpret_cast<float2*>(mw + g * (D + 2) + nd * 8 + 2 * t4) = make_float2(o[nd][0], o[nd][1]);
    *reinterpret_cast<float2*>(mw + (g + 8) * (D + 2) + nd * 8 + 2 * t4) = make_float2(o[nd][2], o[nd][3]);
  }
  if (t4 == 0) {
    mw[g * (D + 2) + D] = m0;
    mw[g * (D + 2) + D + 1] = l0;
    mw[(g + 8) * (D + 2) + D] = m1;
    mw[(g + 8) * (D + 2) + D + 1] = l1;
  }
  __syncthreads();
  constexpr int DPL = D / 32;
  constexpr int LPG = 64 / DPL;   // lanes per 64-group: 16 (D = 128) or 32 (D = 64)
  const int nw = ntiles - 8 * rank < 8 ? (ntiles - 8 * rank > 0 ? ntiles - 8 * rank : 0) : 8;
  // merge 1 (this CTA): warp w takes head rows w, w+8; lane holds D/32 dims; warps in order (fixed)
  auto merge_warps = [&](int row, float& mm, float& l, float (&acc)[DPL]) {
    mm = -INFINITY;
    for (int w = 0; w < nw; ++w) mm = fmaxf(mm, mrg[(w * 16 + row) * (D + 2) + D]);
    l = 0.f;
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
    for (int w = 0; w < nw; ++w) {
      const float* r = mrg + (w * 16 + row) * (D + 2);
      const float wgt = exp2f(r[D] - mm);
      l += wgt * r[D + 1];
#pragma unroll
      for (int t = 0; t < DPL; ++t) acc[t] += wgt * r[lane * DPL + t];
    }
  };
  auto write_row = [&](int row, float l, const float (&acc)[DPL]) {
    const float inv = 1.0f / l;
    const int hq = kvh * grp + row;
    float gs = 0.f;
#pragma unroll
    for (int t = 0; t < DPL; ++t) {
      const uint16_t ob = f2bf(acc[t] * inv);
      p.out_fragx[fragx_offset(qi, int64_t(hq) * D + lane * DPL + t, p.out_nt)] = ob;
      gs += bf2f(ob);
    }
#pragma unroll
    for (int o2 = LPG / 2; o2; o2 >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o2);
    if (p.out_xs && (lane % LPG) == 0) p.out_xs[(int64_t(hq) * D / 64 + lane / LPG) * (p.out_nt * 8) + qi] = gs;
  };
  if (S == 1) {   // single CTA: finalise directly
    for (int row = warp; row < grp; row += 8) {
      float mm, l, acc[DPL];
      merge_warps(row, mm, l, acc);
      write_row(row, l, acc);
    }
    trace_max(4);
    return;
  }
  for (int row = warp; row < grp; row += 8) {   // unnormalised rank partial -> cm
    float mm, l, acc[DPL];
    merge_warps(row, mm, l, acc);
    float* c = cm + row * (D + 4);
#pragma unroll
    for (int t = 0; t < DPL; ++t) c[lane * DPL + t] = acc[t];
    if (lane == 0) {
      c[D] = mm;
      c[D + 1] = l;
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  trace_max(4);
  // merge 2 (cluster): rank q finalises rows q + S*w (warp w); every rank's partial is loaded
  // (vector DSMEM loads) before the rank-ordered merge
  const int row = rank + S * warp;
  if (row < grp) {
    float mr[8], lr[8], ar[8][DPL];
    const uint32_t base = smem_u32(cm + row * (D + 4));
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < S) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(q));
        asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(mr[q]), "=f"(lr[q]) : "r"(ra + D * 4));
        if constexpr (DPL == 4) {
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(ar[q][0]), "=f"(ar[q][1]), "=f"(ar[q][2]), "=f"(ar[q][3])
                       : "r"(ra + lane * DPL * 4));
        } else {
#pragma unroll
          for (int t = 0; t < DPL; ++t)
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(ar[q][t]) : "r"(ra + (lane * DPL + t) * 4));
        }
      }
    }
    float mm = -INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < S) mm = fmaxf(mm, mr[q]);
    float acc[DPL], l = 0.f;
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < S) {
        const float wgt = exp2f(mr[q] - mm);
        l += wgt * lr[q];
#pragma unroll
        for (int t = 0; t < DPL; ++t) acc[t] += wgt * ar[q][t];
      }
    write_row(row, l, acc);
  }
  // peers read this CTA's partial: stay resident until every rank is done
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace ss
