// K3 tree attention, K4 RMSNorm/embedding, K5 sharpened top-k tree growth, K8 argmax merge,
// K9 greedy acceptance + KV commit.  All reductions use fixed orders (bitwise reproducible).
#include "common.cuh"
#include "kernels.h"
#include "attn_warp.cuh"

namespace ss {

static void launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, bool pdl, cudaStream_t st, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelExC(&cfg, fn, args);
}

// block-wide fixed-order sum (256 threads)
SS_DEV float block_sum_256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = (l < 8) ? red[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) red[8] = t;
  }
  __syncthreads();
  return red[8];
}

// ---------------------------------------------------------------------------
// K4: h = bf16(x * 1/sqrt(mean(x^2) + eps) * g) -> FragX.  Optionally x = embed[token] first.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rmsnorm_kernel(const int* tokens, int tok_offset, const uint16_t* embed,
                                                      float* x, int H, const uint16_t* gain, float eps,
                                                      uint16_t* out, float* xs, int nt, ReqMap rq) {
  __shared__ float red[9];
  const int m = blockIdx.x;
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  float* xr = x + int64_t(m) * H;
  if (embed) {
    const int node = rq_req(rq, m) * rq.node_stride + tok_offset + rq_loc(rq, m);   // batched requests
    const uint16_t* er = embed + int64_t(tokens[node]) * H;
    for (int i = threadIdx.x; i < H; i += 256) xr[i] = bf2f(er[i]);
    __syncthreads();
  }
  float ss = 0.f;
  for (int i = threadIdx.x; i < H; i += 256) ss += xr[i] * xr[i];
  ss = block_sum_256(ss, red);
  const float r = 1.0f / sqrtf(ss / float(H) + eps);
  // warp w handles 64-groups w, w+8, ...: 2 elements per lane, group sum of the bf16 values
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g64 = warp; g64 < H / 64; g64 += 8) {
    float gs = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = g64 * 64 + u * 32 + lane;
      const uint16_t hb = f2bf(xr[i] * r * bf2f(gain[i]));
      out[fragx_offset(m, i, nt)] = hb;
      gs += bf2f(hb);
    }
    gs = warp_sum(gs);
    if (lane == 0 && xs) xs[int64_t(g64) * (nt * 8) + m] = gs;
  }
}

void launch_embed_rmsnorm(const int* tokens_dev, int tok_offset, int M, const uint16_t* embed, float* x, int H,
                          const uint16_t* gain, float eps, uint16_t* h_fragx, float* h_xs, int nt, bool pdl,
                          cudaStream_t st, ReqMap rq) {
  void* args[] = {&tokens_dev, &tok_offset, &embed, &x, &H, &gain, &eps, &h_fragx, &h_xs, &nt, &rq};
  launch_pdl((const void*)rmsnorm_kernel, dim3(M), dim3(256), 0, pdl, st, args);
}
void launch_rmsnorm(const float* x, int M, int H, const uint16_t* gain, float eps, uint16_t* h_fragx, float* h_xs,
                    int nt, bool pdl, cudaStream_t st) {
  const int* tokens = nullptr;
  int off = 0;
  const uint16_t* embed = nullptr;
  float* xx = const_cast<float*>(x);
  ReqMap rq{0, 0, 0, 0};
  void* args[] = {&tokens, &off, &embed, &xx, &H, &gain, &eps, &h_fragx, &h_xs, &nt, &rq};
  launch_pdl((const void*)rmsnorm_kernel, dim3(M), dim3(256), 0, pdl, st, args);
}

// ---------------------------------------------------------------------------
// K3: tree attention.  Row = (query node, head).  The keys of node i
// form one LOGICAL sequence: committed prefix [0, P) followed by its ancestors root..i (tree
// slots), i.e. exactly the keys an AR step at that position would see, in the same order.
// One CTA per (kv head, node) walks the node's logical keys in 16-key tiles (attn_warp.cuh).
// Because the blocking depends only on the logical key index, a node's attention is bitwise
// identical whether computed in a tree (verify) or as an AR step.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256, 1) attn_node_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  if (p.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&p.trace[0], t);
  }
  griddep_launch();
  griddep_wait();
  if (p.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.trace[1], t);
  }
  const int S = p.cluster;   // grid.x = n_kv * S, clusters of S along x
  attn_node_cta<D>(p, blockIdx.x / S, blockIdx.y, sm, blockIdx.x % S, S);
  if (p.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.trace[5], t);
  }
}

void launch_attention(const AttnParams& p, bool pdl, cudaStream_t st) {
  // cluster of S = 1 CTA per (kv head, node): the S > 1 DSMEM key split measured no gain
  const int S = 1;
  const size_t smem = size_t(8) * 4 * 16 * (p.head_dim + 8) * 2 + size_t(8) * 16 * (p.head_dim + 2) * 4 +
                      size_t(16) * (p.head_dim + 4) * 4;
  AttnParams pp = p;
  pp.cluster = S;
  const void* fn = p.head_dim == 128 ? (const void*)attn_node_kernel<128> : (const void*)attn_node_kernel<64>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_kv * S, p.n_q);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = S;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (p.head_dim == 128) cudaLaunchKernelEx(&cfg, attn_node_kernel<128>, pp);
  else cudaLaunchKernelEx(&cfg, attn_node_kernel<64>, pp);
}

// ---------------------------------------------------------------------------
// K5: sharpened log-softmax scores and global top-k tree growth.
// Stage A (grid M x B): per block max, sum exp((l - max)/T), and the block's top-k logits.
// Stage B (1 CTA): lse per row, candidate score = parent + (l - max_m)/T - lse_m, global
// top-k by (score desc, token asc, parent asc), canonical order (parent asc, token asc).
// ---------------------------------------------------------------------------
struct Cand {
  float v;
  int idx;
};
SS_DEV bool better(float va, int ia, float vb, int ib) { return va > vb || (va == vb && ia < ib); }

__global__ void __launch_bounds__(256) topk_block_kernel(const TopkParams p) {
  __shared__ float red[9];
  __shared__ Cand wbest[8];
  __shared__ int taken[32];
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  const int m = blockIdx.x, b = blockIdx.y, B = gridDim.y;
  const int64_t v0 = int64_t(p.V) * b / B, v1 = int64_t(p.V) * (b + 1) / B;
  const float* l = p.logits + int64_t(m) * p.V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // max
  float mx = -INFINITY;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += 256) mx = fmaxf(mx, l[v]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += 256) s += expf((l[v] - mx) * p.inv_t);
  s = block_sum_256(s, red);
  const int base = (m * B + b);
  if (threadIdx.x == 0) {
    p.blk_max[base] = mx;
    p.blk_sum[base] = s;
  }
  // k rounds of block argmax with exclusion
  for (int r = 0; r < p.k; ++r) {
    float bv = -INFINITY;
    int bi = INT32_MAX;
    for (int64_t v = v0 + threadIdx.x; v < v1; v += 256) {
      bool tk = false;
      for (int q = 0; q < r; ++q) tk |= (taken[q] == int(v));
      if (!tk && better(l[v], int(v), bv, bi)) {
        bv = l[v];
        bi = int(v);
      }
    }
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) wbest[warp] = {bv, bi};
    __syncthreads();
    if (threadIdx.x == 0) {
      Cand c = wbest[0];
      for (int w = 1; w < 8; ++w)
        if (better(wbest[w].v, wbest[w].idx, c.v, c.idx)) c = wbest[w];
      taken[r] = c.idx;
      p.blk_val[int64_t(base) * p.k + r] = c.v;
      p.blk_idx[int64_t(base) * p.k + r] = c.idx;
    }
    __syncthreads();
  }
}

constexpr int kSelRegK = 8;   // topk_select: per-lane register top-k up to this k (the paper's k = 6)
// the selection order of R12: score desc, then token asc, then parent (frontier row) asc
SS_DEV bool sel_before(float s, int t, int m, float s2, int t2, int m2) {
  return s > s2 || (s == s2 && (t < t2 || (t == t2 && m < m2)));
}
__global__ void __launch_bounds__(512) topk_select_kernel(const TopkParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int B = p.blocks_per_row;
  float* sel_s = reinterpret_cast<float*>(sm);      // [k]
  int* sel_t = reinterpret_cast<int*>(sel_s + 32);  // [k] token
  int* sel_p = sel_t + 32;                          // [k] parent row m
  __shared__ float cs[32][32];                      // per frontier row: its k best (score, token)
  __shared__ int ct[32][32];
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // batched requests: CTA q selects request q's children from its own frontier rows [r0, r0 + Mr)
  const int q = blockIdx.x;
  const int Mr = p.req_rows > 0 ? p.req_rows : p.M, r0 = q * Mr;
  const int64_t nofs = int64_t(q) * p.node_stride;
  const float* score = p.score + nofs;
  for (int m = warp; m < Mr; m += int(blockDim.x >> 5)) {
    // warp per row m: the row's max and sum exp((l - max) / T) merged over its B vocab tiles (fixed
    // lane order + fixed shuffle tree: deterministic), then its k best children in selection order
    const int mg = r0 + m;
    // one pass, 8 independent loads in flight per lane: a running (max, sum) per lane in its fixed
    // tile order, then the lanes merged by a fixed shuffle tree
    float lm = -INFINITY, lsum = 0.f;
    const float* bmx = p.blk_max + int64_t(mg) * B;
    const float* bsm = p.blk_sum + int64_t(mg) * B;
    for (int b0 = lane; b0 < B; b0 += 32 * 8) {
      float vm[8], vs[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = b0 + 32 * j;
        vm[j] = b < B ? bmx[b] : -INFINITY;
        vs[j] = b < B ? bsm[b] : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (vm[j] > -INFINITY) {
          const float nm = fmaxf(lm, vm[j]);
          lsum = lsum * expf((lm - nm) * p.inv_t) + vs[j] * expf((vm[j] - nm) * p.inv_t);
          lm = nm;
        }
    }
    const float mx = warp_max(lm);
    const float lse = logf(warp_sum(lm > -INFINITY ? lsum * expf((lm - mx) * p.inv_t) : 0.f));
    const int nc = B * p.k;
    const int* bi = p.blk_idx + int64_t(mg) * nc;
    const float* bv = p.blk_val + int64_t(mg) * nc;
    const float base = score[p.node_base + m];
    const bool fast = p.k <= kSelRegK && B >= p.k;
    if (fast) {
      // Every vocab tile's list is sorted in selection order (value desc, token asc; the candidate
      // score is monotone in the value), so the row's k best lie in the k tiles with the best heads:
      // (1) each lane keeps the k best tile heads it scans, in registers; (2) k rounds of a warp
      // merge pick the k best heads; (3) the k x k candidates of those tiles -> the row's k best.
      float ls[kSelRegK];
      int lt[kSelRegK], lb[kSelRegK];
#pragma unroll
      for (int i = 0; i < kSelRegK; ++i) {
        ls[i] = -INFINITY;
        lt[i] = INT32_MAX;
        lb[i] = 0;
      }
      for (int t0 = lane; t0 < B; t0 += 32 * 8) {
        int ht[8];
        float hv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // 8 independent head loads in flight
          const int t = t0 + 32 * j;
          ht[j] = t < B ? bi[int64_t(t) * p.k] : INT32_MAX;
          hv[j] = t < B ? bv[int64_t(t) * p.k] : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
        const int t = t0 + 32 * j, tok = ht[j];
        if (t >= B) continue;
        const float sc = base + ((hv[j] - mx) * p.inv_t - lse);
        if (sel_before(sc, tok, 0, ls[kSelRegK - 1], lt[kSelRegK - 1], 0)) {
          float cs_ = sc;
          int ct_ = tok, cb_ = t;
#pragma unroll
          for (int i = 0; i < kSelRegK; ++i)
            if (sel_before(cs_, ct_, 0, ls[i], lt[i], 0)) {
              const float ts = ls[i];
              const int tt = lt[i], tb = lb[i];
              ls[i] = cs_;
              lt[i] = ct_;
              lb[i] = cb_;
              cs_ = ts;
              ct_ = tt;
              cb_ = tb;
            }
        }
        }
      }
      int mytile = -1;   // lane r < k: the r-th best tile
      for (int r = 0; r < p.k; ++r) {
        float bs = ls[0];
        int bt = lt[0], bb = lb[0];
        for (int o = 16; o; o >>= 1) {
          const float os = __shfl_xor_sync(0xffffffffu, bs, o);
          const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
          const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
          if (sel_before(os, ot, 0, bs, bt, 0)) {
            bs = os;
            bt = ot;
            bb = ob;
          }
        }
        if (lane == r) mytile = bb;
        if (lt[0] == bt && ls[0] == bs) {   // the winner's lane pops its head (tokens are distinct)
#pragma unroll
          for (int i = 0; i + 1 < kSelRegK; ++i) {
            ls[i] = ls[i + 1];
            lt[i] = lt[i + 1];
            lb[i] = lb[i + 1];
          }
          ls[kSelRegK - 1] = -INFINITY;
          lt[kSelRegK - 1] = INT32_MAX;
        }
      }
      // candidates of the k chosen tiles: c = r * k + j -> tile of lane r, entry j (k * k <= 64)
      const int ncand = p.k * p.k;
      float c_s[2];
      int c_t[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        const int tile = __shfl_sync(0xffffffffu, mytile, (c / p.k) & 31);
        c_s[h] = -INFINITY;
        c_t[h] = INT32_MAX;
        if (c < ncand) {
          const int64_t e = int64_t(tile) * p.k + c % p.k;
          c_t[h] = bi[e];
          c_s[h] = base + ((bv[e] - mx) * p.inv_t - lse);
        }
      }
      float ps = INFINITY;
      int pt = -1;
      for (int r = 0; r < p.k; ++r) {
        float bs = -INFINITY;
        int bt = INT32_MAX;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (sel_before(ps, pt, 0, c_s[h], c_t[h], 0) && sel_before(c_s[h], c_t[h], 0, bs, bt, 0)) {
            bs = c_s[h];
            bt = c_t[h];
          }
        for (int o = 16; o; o >>= 1) {
          const float os = __shfl_xor_sync(0xffffffffu, bs, o);
          const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
          if (sel_before(os, ot, 0, bs, bt, 0)) {
            bs = os;
            bt = ot;
          }
        }
        if (lane == 0) {
          cs[m][r] = bs;
          ct[m][r] = bt;
        }
        ps = bs;
        pt = bt;
      }
    }
    float ps = INFINITY;   // the previous pick (candidates are distinct tokens within a row)
    int pt = -1;
    for (int r = 0; r < p.k && !fast; ++r) {   // otherwise: k scans of all the candidates
      float bs = -INFINITY;
      int bt = INT32_MAX;
      for (int c = lane; c < nc; c += 32) {
        const int tok = bi[c];
        const float sc = base + ((bv[c] - mx) * p.inv_t - lse);
        if (sel_before(ps, pt, 0, sc, tok, 0) && sel_before(sc, tok, 0, bs, bt, 0)) {
          bs = sc;
          bt = tok;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const float os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        if (sel_before(os, ot, 0, bs, bt, 0)) {
          bs = os;
          bt = ot;
        }
      }
      if (lane == 0) {
        cs[m][r] = bs;
        ct[m][r] = bt;
      }
      ps = bs;
      pt = bt;
    }
  }
  __syncthreads();
  if (warp == 0) {
    // the k best of the Mr x k row candidates, in selection order (key (score, token, row) is unique)
    float ps = INFINITY;
    int pt = -1, pm = -1;
    for (int r = 0; r < p.k; ++r) {
      float bs = -INFINITY;
      int bt = INT32_MAX, bm = INT32_MAX;
      for (int c = lane; c < Mr * p.k; c += 32) {
        const int m = c / p.k, j = c % p.k;
        const float sc = cs[m][j];
        const int tok = ct[m][j];
        if (sel_before(ps, pt, pm, sc, tok, m) && sel_before(sc, tok, m, bs, bt, bm)) {
          bs = sc;
          bt = tok;
          bm = m;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const float os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        const int om = __shfl_xor_sync(0xffffffffu, bm, o);
        if (sel_before(os, ot, om, bs, bt, bm)) {
          bs = os;
          bt = ot;
          bm = om;
        }
      }
      if (lane == 0) {
        sel_s[r] = bs;
        sel_t[r] = bt;
        sel_p[r] = bm;
      }
      ps = bs;
      pt = bt;
      pm = bm;
    }
    __syncwarp();
    if (lane == 0) {
      // canonical order: parent asc, token asc (insertion sort, k <= 32)
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
  }
  __syncthreads();
  int* anc = p.anc + nofs * p.anc_stride;   // slots, parents and ancestors are request-local
  for (int j = warp; j < p.k; j += blockDim.x >> 5) {
    const int node = p.child_base + j, par = p.node_base + sel_p[j];
    if (lane == 0) {
      p.tok[nofs + node] = sel_t[j];
      p.parent[nofs + node] = par;
      p.depth[nofs + node] = p.child_depth;
      p.score[nofs + node] = sel_s[j];
    }
    for (int a = lane; a < p.child_depth; a += 32)
      anc[int64_t(node) * p.anc_stride + a] = anc[int64_t(par) * p.anc_stride + a];
    if (lane == 0) anc[int64_t(node) * p.anc_stride + p.child_depth] = node;
  }
}

void launch_topk_select(const TopkParams& p, bool pdl, cudaStream_t st) {
  void* args[] = {const_cast<TopkParams*>(&p)};
  const int nreq = p.req_rows > 0 ? p.M / p.req_rows : 1;
  launch_pdl((const void*)topk_select_kernel, dim3(nreq), dim3(512), 3 * 32 * 4, pdl, st, args);
}

void launch_topk(const TopkParams& p, bool pdl, cudaStream_t st) {
  TopkParams pp = p;
  void* args[] = {&pp};
  launch_pdl((const void*)topk_block_kernel, dim3(p.M, p.blocks_per_row), dim3(256), 0, pdl, st, args);
  const int n_req = p.req_rows > 0 ? p.M / p.req_rows : 1;
  launch_pdl((const void*)topk_select_kernel, dim3(n_req), dim3(512), 3 * 32 * 4, pdl, st, args);
}

// ---------------------------------------------------------------------------
// K8: merge per-tile (max, argmax, second) into per-node argmax (ties -> smallest id) and gap.
// ---------------------------------------------------------------------------
__global__ void argmax_merge_kernel(const float* am_val, const int* am_idx, const float* am_second, int M, int tiles,
                                    int* argmax, float* gap) {
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * 8 + warp;
  if (m >= M) return;
  float bv = -INFINITY, sv = -INFINITY;
  int bi = INT32_MAX;
  for (int t = lane; t < tiles; t += 32) {
    const float v = am_val[int64_t(m) * tiles + t], s2 = am_second[int64_t(m) * tiles + t];
    const int i = am_idx[int64_t(m) * tiles + t];
    if (better(v, i, bv, bi)) {
      sv = fmaxf(bv, s2);
      bv = v;
      bi = i;
    } else {
      sv = fmaxf(sv, v);
    }
  }
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const float os = __shfl_xor_sync(0xffffffffu, sv, o);
    if (better(ov, oi, bv, bi)) {
      sv = fmaxf(bv, os);
      bv = ov;
      bi = oi;
    } else {
      sv = fmaxf(sv, ov);
    }
  }
  if (lane == 0) {
    argmax[m] = bi;
    gap[m] = bv - sv;
  }
}
void launch_argmax_merge(const float* am_val, const int* am_idx, const float* am_second, int M, int tiles,
                         int* argmax, float* gap, bool pdl, cudaStream_t st) {
  void* args[] = {&am_val, &am_idx, &am_second, &M, &tiles, &argmax, &gap};
  launch_pdl((const void*)argmax_merge_kernel, dim3((M + 7) / 8), dim3(256), 0, pdl, st, args);
}

// ---------------------------------------------------------------------------
// K9: greedy acceptance (one warp, ballot over the <= 32 children of each depth) and the
// KV commit/compaction of root + accepted path into committed positions P..P+a.
// ---------------------------------------------------------------------------
__global__ void accept_kernel(const AcceptParams p0) {
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  // batched requests: one warp per request, every per-request array offset by its stride
  const int q = p0.req0 + blockIdx.x;
  AcceptParams p = p0;
  p.argmax += int64_t(blockIdx.x) * p0.n_nodes;
  p.tok += int64_t(q) * p0.node_stride;
  p.parent += int64_t(q) * p0.node_stride;
  p.commit_meta += 2 * q;
  p.committed_len += q;
  p.root_tok += q;
  p.out_tokens += int64_t(q) * p0.out_stride;
  p.out_n += q;
  p.out_path += int64_t(q) * p0.out_stride;
  const int lane = threadIdx.x;
  int n = 1, cur = 0;
  if (p.chain) {
    for (int i = lane; i < p.n_nodes; i += 32) p.out_path[i] = i;
    n = p.n_nodes;
    cur = p.n_nodes - 1;
  } else {
    if (lane == 0) p.out_path[0] = 0;
    for (int d = 0; d < p.depth_max; ++d) {
      const int y = p.argmax[cur];
      const int c = 1 + d * p.k + lane;
      const bool hit = lane < p.k && c < p.n_nodes && p.parent[c] == cur && p.tok[c] == y;
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (b == 0) break;
      cur = 1 + d * p.k + (__ffs(b) - 1);
      if (lane == 0) {
        p.out_path[n] = cur;
        p.out_tokens[n - 1] = p.tok[cur];
      }
      ++n;
    }
  }
  if (lane == 0) {
    const int bonus = p.argmax[cur];
    const int P = *p.committed_len;
    if (p.chain) {
      p.out_tokens[0] = bonus;
      *p.out_n = 1;
    } else {
      p.out_tokens[n - 1] = bonus;
      *p.out_n = n;
    }
    p.commit_meta[0] = P;   // base position
    p.commit_meta[1] = n;   // rows committed (root + accepted)
    *p.committed_len = P + n;
    *p.root_tok = bonus;
  }
}

__global__ void __launch_bounds__(256) commit_kernel(const AcceptParams p) {
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  const int l = blockIdx.x, h = blockIdx.y, which = blockIdx.z & 1, q = p.req0 + (blockIdx.z >> 1);
  const int base = p.commit_meta[2 * q], n = p.commit_meta[2 * q + 1];
  uint16_t* cache = (which ? p.v_cache : p.k_cache) + l * p.cache_layer_stride +
                    (int64_t(h) * p.max_ctx + int64_t(q) * p.ctx_stride) * p.head_dim;
  const uint16_t* tree = (which ? p.v_tree : p.k_tree) + l * p.tree_layer_stride +
                         (int64_t(h) * p.max_nodes + int64_t(q) * p.node_stride) * p.head_dim;
  const int* path = p.out_path + int64_t(q) * p.out_stride;
  const int dw = p.head_dim / 2;
  for (int e = threadIdx.x; e < n * dw; e += 256) {
    const int j = e / dw, i = e % dw;
    const int slot = path[j];
    reinterpret_cast<uint32_t*>(cache + int64_t(base + j) * p.head_dim)[i] =
        reinterpret_cast<const uint32_t*>(tree + int64_t(slot) * p.head_dim)[i];
  }
}

void launch_commit(const AcceptParams& p, bool pdl, cudaStream_t st) {
  AcceptParams pp = p;
  void* args[] = {&pp};
  const int n_req = p.n_req > 0 ? p.n_req : 1;
  launch_pdl((const void*)commit_kernel, dim3(p.n_layers, p.n_kv, 2 * n_req), dim3(256), 0, pdl, st, args);
}

void launch_accept_commit(const AcceptParams& p, bool pdl, cudaStream_t st) {
  AcceptParams pp = p;
  void* args[] = {&pp};
  const int n_req = p.n_req > 0 ? p.n_req : 1;
  launch_pdl((const void*)accept_kernel, dim3(n_req), dim3(32), 0, pdl, st, args);
  launch_pdl((const void*)commit_kernel, dim3(p.n_layers, p.n_kv, 2 * n_req), dim3(256), 0, pdl, st, args);
}

__global__ void tree_init_kernel(const int* root_tok, int* tok, int* parent, int* depth, float* score, int* anc,
                                 int node_stride, int anc_stride) {
  griddep_launch();   // small grid: let the next kernel start its prologue (weight prefetch) now
  griddep_wait();
  const int q = threadIdx.x;   // request q's root at its slot 0
  const int64_t o = int64_t(q) * node_stride;
  tok[o] = root_tok[q];
  parent[o] = -1;
  depth[o] = 0;
  score[o] = 0.f;
  anc[o * anc_stride] = 0;
}
void launch_tree_init(const int* root_tok, int* tok, int* parent, int* depth, float* score, int* anc, bool pdl,
                      cudaStream_t st, int n_req, int node_stride, int anc_stride) {
  void* args[] = {&root_tok, &tok, &parent, &depth, &score, &anc, &node_stride, &anc_stride};
  launch_pdl((const void*)tree_init_kernel, dim3(1), dim3(n_req < 1 ? 1 : n_req), 0, pdl, st, args);
}

__global__ void chain_init_kernel(const int* tokens, int n, int* tok, int* parent, int* depth, float* score, int* anc,
                                  int anc_stride) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    if (threadIdx.x == 0) {
      tok[i] = tokens[i];
      parent[i] = i - 1;
      depth[i] = i;
      score[i] = 0.f;
    }
    for (int j = threadIdx.x; j <= i; j += blockDim.x) anc[int64_t(i) * anc_stride + j] = j;
  }
}
void launch_chain_init(const int* tokens, int n, int* tok, int* parent, int* depth, float* score, int* anc,
                       int anc_stride, cudaStream_t st) {
  chain_init_kernel<<<n < 256 ? n : 256, 128, 0, st>>>(tokens, n, tok, parent, depth, score, anc, anc_stride);
}

}  // namespace ss
