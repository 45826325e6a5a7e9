// SS_FP32 precision mode (SURVEY.md §8(b) `precision`; BASELINE.json north_star "1e-4 in fp32 mode"):
// the same forward with every activation, q/k/v, the KV cache and the attention
// kept in fp32 (no bf16 rounding points), on plain CUDA-core kernels.  The weights are the same bf16
// values (exact in fp32) and the substitutes the same code*s + z (exact in fp32).  It exists for parity
// (1e-4 x logit scale against the fp64 oracle), not speed: one thread per output, K-loops in order.
#include "common.cuh"
#include "kernels.h"

namespace ss {

// ---- K4f: x = embed[token] (optional), h = x * rsqrt(mean(x^2) + eps) * g ----------------------
__global__ void __launch_bounds__(256) rmsnorm_f32_kernel(const int* tokens, int tok_offset, const uint16_t* embed,
                                                          float* x, int H, const uint16_t* gain, float eps, float* h) {
  __shared__ float red[8];
  const int m = blockIdx.x;
  float* xr = x + int64_t(m) * H;
  if (embed) {
    const uint16_t* er = embed + int64_t(tokens[tok_offset + m]) * H;
    for (int i = threadIdx.x; i < H; i += 256) xr[i] = bf2f(er[i]);
    __syncthreads();
  }
  float ss = 0.f;
  for (int i = threadIdx.x; i < H; i += 256) ss += xr[i] * xr[i];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < 8; ++w) t += red[w];
  const float r = 1.0f / sqrtf(t / float(H) + eps);
  for (int i = threadIdx.x; i < H; i += 256) h[int64_t(m) * H + i] = xr[i] * r * bf2f(gain[i]);
}

// ---- K2f / K6f: Y[M x N] = X[M x K] * W^T, W tiled bf16 (fmt 0) or a 4-/3-/2-bit substitute (fmt 4 / 3 / 2:
// W_hat = code * s + z, exact in fp32).  Block: 128 output columns x 8 rows; X tiles staged in smem.
__device__ __forceinline__ float wval(const uint8_t* W, int fmt, int64_t n, int64_t k, int64_t K) {
  if (fmt == 0) return bf2f(*reinterpret_cast<const uint16_t*>(W + bf16_tiled_offset(n, k, K)));
  uint64_t off, moff;
  int sh;
  uint32_t code;
  if (fmt == 3) {
    uint64_t hoff;
    int hbit;
    q3_code_pos(n, k, K, &off, &sh, &hoff, &hbit);
    moff = q3_meta_offset(n, k, K);
    code = ((W[off] >> sh) & 3u) | (((W[hoff] >> hbit) & 1u) << 2);
  } else {
    if (fmt == 2) {
      q2_code_pos(n, k, K, &off, &sh);
      moff = q2_meta_offset(n, k, K);
    } else {
      q4_code_pos(n, k, K, &off, &sh);
      moff = q4_meta_offset(n, k, K);
    }
    code = (W[off] >> sh) & (fmt == 2 ? 3u : 15u);
  }
  const uint32_t m = *reinterpret_cast<const uint32_t*>(W + moff);
  return fmaf(float(code), __uint_as_float(m << 16), __uint_as_float(m & 0xFFFF0000u));   // exact
}

constexpr int kF32Rows = 8, kF32KTile = 256;
__global__ void __launch_bounds__(128) linear_f32_kernel(const float* X, int M, int K, const uint8_t* W, int fmt, int N,
                                                         float* Y) {
  __shared__ float xs[kF32Rows][kF32KTile];
  const int n = blockIdx.x * 128 + threadIdx.x, m0 = blockIdx.y * kF32Rows;
  float acc[kF32Rows];
#pragma unroll
  for (int r = 0; r < kF32Rows; ++r) acc[r] = 0.f;
  for (int k0 = 0; k0 < K; k0 += kF32KTile) {
    __syncthreads();
    for (int i = threadIdx.x; i < kF32Rows * kF32KTile; i += 128) {
      const int r = i / kF32KTile, kk = i % kF32KTile;
      xs[r][kk] = (m0 + r < M && k0 + kk < K) ? X[int64_t(m0 + r) * K + k0 + kk] : 0.f;
    }
    __syncthreads();
    const int kn = min(kF32KTile, K - k0);
    for (int kk = 0; kk < kn; ++kk) {
      const float w = wval(W, fmt, n, k0 + kk, K);
#pragma unroll
      for (int r = 0; r < kF32Rows; ++r) acc[r] = fmaf(xs[r][kk], w, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < kF32Rows; ++r)
    if (m0 + r < M) Y[int64_t(m0 + r) * N + n] = acc[r];
}

// ---- qkv epilogue: + bias, rotate-half RoPE at pos = P + depth, q out, K/V into the tree slots ----
__global__ void qkv_post_f32_kernel(const float* Y, int M, const uint16_t* bias, int qd, int kvd, int d,
                                    const float2* rope, const int* committed_len, const int* depth, int node_base,
                                    float* q_out, float* k_tree, float* v_tree, int max_nodes) {
  const int m = blockIdx.x;
  const int rows = qd + 2 * kvd, half = d / 2;
  const int P = *committed_len, node = node_base + m;
  const int pos = P + depth[node];
  for (int u = threadIdx.x; u < rows / 2; u += blockDim.x) {
    const int hd = u / half, i = u % half;     // head (over q, k, v heads), rotation pair i
    const int lo = hd * d + i, hi = lo + half;
    float vlo = Y[int64_t(m) * rows + lo], vhi = Y[int64_t(m) * rows + hi];
    if (bias) {
      vlo += bf2f(bias[lo]);
      vhi += bf2f(bias[hi]);
    }
    if (lo < qd + kvd) {
      const float2 cs = rope[int64_t(pos) * half + i];
      const float a = vlo * cs.x - vhi * cs.y, b = vhi * cs.x + vlo * cs.y;
      vlo = a;
      vhi = b;
    }
    if (lo < qd) {
      q_out[int64_t(m) * qd + lo] = vlo;
      q_out[int64_t(m) * qd + hi] = vhi;
    } else {
      const bool isk = lo < qd + kvd;
      const int r = lo - (isk ? qd : qd + kvd), kvh = r / d, j = r % d;
      float* dst = (isk ? k_tree : v_tree) + (int64_t(kvh) * max_nodes + node) * d;
      dst[j] = vlo;
      dst[j + half] = vhi;
    }
  }
}

// ---- tree attention: node m, head h; keys = committed prefix [0, P) ++ ancestors root..self --------
__global__ void attention_f32_kernel(const float* q, const float* k_cache, const float* v_cache, const float* k_tree,
                                     const float* v_tree, const int* committed_len, const int* anc, const int* depth,
                                     int anc_stride, int max_ctx, int max_nodes, int node_base, int n_heads, int n_kv,
                                     int d, float* out) {
  extern __shared__ float sc[];   // [keys]
  __shared__ float red[32];
  const int m = blockIdx.x, h = blockIdx.y;
  const int node = node_base + m, kvh = h / (n_heads / n_kv);
  const int P = *committed_len, nk = P + depth[node] + 1;
  const float* qv = q + (int64_t(m) * n_heads + h) * d;
  const float inv = 1.0f / sqrtf(float(d));
  auto key = [&](int j) -> const float* {
    return j < P ? k_cache + (int64_t(kvh) * max_ctx + j) * d
                 : k_tree + (int64_t(kvh) * max_nodes + anc[int64_t(node) * anc_stride + (j - P)]) * d;
  };
  auto val = [&](int j) -> const float* {
    return j < P ? v_cache + (int64_t(kvh) * max_ctx + j) * d
                 : v_tree + (int64_t(kvh) * max_nodes + anc[int64_t(node) * anc_stride + (j - P)]) * d;
  };
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const float* kr = key(j);
    float s = 0.f;
    for (int t = 0; t < d; ++t) s = fmaf(qv[t], kr[t], s);
    s *= inv;
    sc[j] = s;
    mx = fmaxf(mx, s);
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) sum += red[w];
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float o = 0.f;
    for (int j = 0; j < nk; ++j) o = fmaf(sc[j], val(j)[t], o);
    out[(int64_t(m) * n_heads + h) * d + t] = o / sum;
  }
}

__global__ void add_f32_kernel(float* x, const float* y, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) x[i] += y[i];
}

// gate/up rows interleaved per 64 (gate 64, up 64): act[m][64 b + u] = silu(gate) * up
__global__ void silu_mul_f32_kernel(const float* Y, int M, int F, float* act) {
  const int64_t n = int64_t(M) * F;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / F;
    const int f = int(i % F), b = f / 64, u = f % 64;
    const float g = Y[m * 2 * F + 128 * b + u], up = Y[m * 2 * F + 128 * b + 64 + u];
    act[i] = g / (1.0f + expf(-g)) * up;
  }
}

// per row: argmax (first index of the max) and top-1 minus top-2 (fixed-order block reduction)
__global__ void __launch_bounds__(256) argmax_f32_kernel(const float* logits, int V, int* argmax, float* gap) {
  __shared__ float bv[256], b2[256];
  __shared__ int bi[256];
  const int m = blockIdx.x;
  const float* l = logits + int64_t(m) * V;
  float v1 = -INFINITY, v2 = -INFINITY;
  int i1 = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += 256) {
    const float v = l[i];
    if (v > v1) {
      v2 = v1;
      v1 = v;
      i1 = i;
    } else if (v > v2) {
      v2 = v;
    }
  }
  bv[threadIdx.x] = v1;
  b2[threadIdx.x] = v2;
  bi[threadIdx.x] = i1;
  __syncthreads();
  if (threadIdx.x == 0) {
    float best = -INFINITY, second = -INFINITY;
    int idx = 0x7fffffff;
    for (int t = 0; t < 256; ++t) {
      const float v = bv[t];
      if (v > best || (v == best && bi[t] < idx)) {
        second = fmaxf(second, best);
        best = v;
        idx = bi[t];
      } else {
        second = fmaxf(second, v);
      }
      second = fmaxf(second, b2[t]);
    }
    argmax[m] = idx;
    gap[m] = best - second;
  }
}

// ---- launchers ---------------------------------------------------------------------------------
void launch_rmsnorm_f32(const int* tokens, int tok_offset, const uint16_t* embed, float* x, int M, int H,
                        const uint16_t* gain, float eps, float* h, cudaStream_t st) {
  rmsnorm_f32_kernel<<<M, 256, 0, st>>>(tokens, tok_offset, embed, x, H, gain, eps, h);
}
void launch_linear_f32(const float* X, int M, int K, const uint8_t* W, int fmt, int N, float* Y, cudaStream_t st) {
  linear_f32_kernel<<<dim3(N / 128, (M + kF32Rows - 1) / kF32Rows), 128, 0, st>>>(X, M, K, W, fmt, N, Y);
}
void launch_qkv_post_f32(const float* Y, int M, const uint16_t* bias, int qd, int kvd, int d, const float2* rope,
                         const int* committed_len, const int* depth, int node_base, float* q_out, float* k_tree,
                         float* v_tree, int max_nodes, cudaStream_t st) {
  qkv_post_f32_kernel<<<M, 128, 0, st>>>(Y, M, bias, qd, kvd, d, rope, committed_len, depth, node_base, q_out, k_tree,
                                         v_tree, max_nodes);
}
void launch_attention_f32(const float* q, const float* k_cache, const float* v_cache, const float* k_tree,
                          const float* v_tree, const int* committed_len, const int* anc, const int* depth, int anc_stride,
                          int max_ctx, int max_nodes, int node_base, int M, int n_heads, int n_kv, int d, float* out,
                          cudaStream_t st) {
  attention_f32_kernel<<<dim3(M, n_heads), 128, size_t(max_ctx) * 4, st>>>(q, k_cache, v_cache, k_tree, v_tree,
                                                                        committed_len, anc, depth, anc_stride, max_ctx,
                                                                        max_nodes, node_base, n_heads, n_kv, d, out);
}
void launch_add_f32(float* x, const float* y, int64_t n, cudaStream_t st) {
  add_f32_kernel<<<int((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(x, y, n);
}
void launch_silu_mul_f32(const float* Y, int M, int F, float* act, cudaStream_t st) {
  const int64_t n = int64_t(M) * F;
  silu_mul_f32_kernel<<<int((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(Y, M, F, act);
}
void launch_argmax_f32(const float* logits, int M, int V, int* argmax, float* gap, cudaStream_t st) {
  argmax_f32_kernel<<<M, 256, 0, st>>>(logits, V, argmax, gap);
}

}  // namespace ss
