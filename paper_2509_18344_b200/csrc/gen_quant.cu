// Weight generator (independent re-implementation of synth/weights.py),
// K1 substitute quantizer (SURVEY O.2 / PAPER.md:133-136, :278) and layout debug readbacks.
#include "common.cuh"
#include "kernels.h"

namespace ss {

SS_DEV uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// element value for row-major index idx: Irwin-Hall(4) integer, one fp32 multiply, (gain: + 1.0f), RNE bf16
SS_DEV uint16_t gen_value(uint64_t key, uint64_t idx, float c32, int gain) {
  uint64_t r = splitmix64(key ^ idx);
  int32_t s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += int32_t((r >> (16 * j)) & 0xFFFFu);
  int32_t s2 = 2 * s - 4 * 65535;
  float w = __fmul_rn(float(s2), c32);   // s2 exact in fp32 (|s2| < 2^18)
  if (gain) w = __fadd_rn(1.0f, w);
  return f2bf(w);
}

// natural row-major destination (embedding, norm gains, biases)
__global__ void gen_natural_kernel(uint16_t* __restrict__ dst, uint64_t key, uint64_t first, uint64_t count, float c32,
                                   int gain) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = gen_value(key, first + i, c32, gain);
}

// tiled destination: src [rows x K] row-major index space, dst row = map(src row)
// map: 0 -> dst = row_off + r ; 1 -> gate rows (r/64)*128 + r%64 ; 2 -> up rows (r/64)*128 + 64 + r%64
__global__ void gen_tiled_kernel(uint8_t* __restrict__ dst, uint64_t key, int64_t rows, int64_t K, float c32,
                                 int map, int64_t row_off) {
  int64_t n8 = rows * (K / 8);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n8; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = t / (K / 8), k0 = (t % (K / 8)) * 8;
    int64_t dr = map == 0 ? row_off + r : (map == 1 ? (r / 64) * 128 + (r % 64) : (r / 64) * 128 + 64 + (r % 64));
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint16_t lo = gen_value(key, uint64_t(r * K + k0 + 2 * e), c32, 0);
      uint16_t hi = gen_value(key, uint64_t(r * K + k0 + 2 * e + 1), c32, 0);
      v[e] = uint32_t(lo) | (uint32_t(hi) << 16);
    }
    *reinterpret_cast<uint4*>(dst + bf16_tiled_offset(dr, k0, K)) = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// caller weights: natural row-major bf16 source [rows x K] (device copy) -> tiled destination, with
// the same row map as gen_tiled_kernel
__global__ void tile_from_natural_kernel(uint8_t* __restrict__ dst, const uint16_t* __restrict__ src, int64_t rows,
                                         int64_t K, int map, int64_t row_off) {
  int64_t n8 = rows * (K / 8);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n8; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = t / (K / 8), k0 = (t % (K / 8)) * 8;
    int64_t dr = map == 0 ? row_off + r : (map == 1 ? (r / 64) * 128 + (r % 64) : (r / 64) * 128 + 64 + (r % 64));
    *reinterpret_cast<uint4*>(dst + bf16_tiled_offset(dr, k0, K)) = *reinterpret_cast<const uint4*>(src + r * K + k0);
  }
}

void launch_tile_from_natural(uint8_t* dst, const uint16_t* src, int64_t rows, int64_t K, int map, int64_t row_off,
                              cudaStream_t st) {
  int64_t n8 = rows * (K / 8);
  int blocks = int((n8 + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  tile_from_natural_kernel<<<blocks, 256, 0, st>>>(dst, src, rows, K, map, row_off);
}

void launch_gen_natural(uint16_t* dst, uint64_t key, uint64_t count, float c32, int gain, cudaStream_t st,
                        uint64_t first) {
  int blocks = int((count + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  gen_natural_kernel<<<blocks, 256, 0, st>>>(dst, key, first, count, c32, gain);
}
void launch_gen_tiled(uint8_t* dst, uint64_t key, int64_t rows, int64_t K, float c32, int map, int64_t row_off,
                      cudaStream_t st) {
  int64_t n8 = rows * (K / 8);
  int blocks = int((n8 + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  gen_tiled_kernel<<<blocks, 256, 0, st>>>(dst, key, rows, K, c32, map, row_off);
}

// ---------------------------------------------------------------------------
// K1: RTN min/max group-64 quantizer, bf16 tiled -> Q4 (or Q2) tiled (layouts in
// common.cuh).  One thread per (row, 64-group) of a tile-chunk (256 threads per chunk):
//   s = (M == m) ? 1 : RNE_bf16(fp32(M - m) / (2^BITS - 1)) ; z = m   (HQQ: z = RNE_bf16(refined zero))
//   code = clamp(rint_even(fp32(x - z) / s), 0, 2^BITS - 1)       (IEEE div.rn; built without fast-math)
// ---------------------------------------------------------------------------
// HQQ zero refinement (reading R28; oracle/quant.py hqq_refine_zero): the
// min/max scale is kept, the zero is refined by half-quadratic splitting of min_z ||x - W_r(z)||_0.7,
//   code = clamp(rint((x - z)/s)), e = x - (code*s + z), err = mean|e|  (stop once err stops falling,
//   keep the zero of the lowest err), W_e = sign(e)*max(|e| - |e|^(p-1)/beta, 0),
//   z <- mean(x - W_e - code*s), beta *= kappa,
// in fp64 with index-order sums, per 64-group (one thread).  Explicit _rn intrinsics: no contraction
// (code*s is exact, so a contracted form would round identically, but the sums must not reassociate).
constexpr double kHqqP = 0.7, kHqqBeta0 = 10.0, kHqqKappa = 1.01;
template <int BITS>
SS_DEV double hqq_refine_zero(const float (&x)[64], double s, double z0, int iters) {
  const double qmax = double((1 << BITS) - 1), pm1 = kHqqP - 1.0;
  double z = z0, best_z = z0, best_err = __longlong_as_double(0x7FF0000000000000ll), beta = kHqqBeta0;
  for (int it = 0; it < iters; ++it) {
    double err = 0.0;
    for (int i = 0; i < 64; ++i) {
      const double c = fmin(fmax(rint(__ddiv_rn(__dsub_rn(double(x[i]), z), s)), 0.0), qmax);
      err = __dadd_rn(err, fabs(__dsub_rn(double(x[i]), __dadd_rn(__dmul_rn(c, s), z))));
    }
    err = __dmul_rn(err, 1.0 / 64.0);
    if (!(err < best_err)) break;
    best_err = err;
    best_z = z;
    double acc = 0.0;
    for (int i = 0; i < 64; ++i) {
      const double xi = double(x[i]);
      const double c = fmin(fmax(rint(__ddiv_rn(__dsub_rn(xi, z), s)), 0.0), qmax);
      const double cs = __dmul_rn(c, s);
      const double e = __dsub_rn(xi, __dadd_rn(cs, z));
      const double a = fabs(e);
      const double t = __dsub_rn(a, __ddiv_rn(pow(a, pm1), beta));
      const double we = t > 0.0 ? copysign(t, e) : 0.0;
      acc = __dadd_rn(acc, __dsub_rn(__dsub_rn(xi, we), cs));
    }
    z = __dmul_rn(acc, 1.0 / 64.0);
    beta = __dmul_rn(beta, kHqqKappa);
  }
  return best_z;
}
// fp64 -> bf16 bits, round to nearest even, in one step (normal range)
SS_DEV uint16_t f64_to_bf16_rne(double v) {
  const unsigned long long u = __double_as_longlong(v);
  const unsigned long long r = (u + ((1ull << 44) - 1) + ((u >> 45) & 1ull)) & ~((1ull << 45) - 1);
  return f2bf(float(__longlong_as_double(r)));   // exact: r has 8 significant bits
}

template <int BITS>
__global__ void __launch_bounds__(256) quantize_q_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                         int64_t n_tc, int hqq_iters) {
  constexpr float kLevels = float((1 << BITS) - 1);
  constexpr int kTile = BITS == 2 ? kQ2TileBytes : (BITS == 3 ? kQ3TileBytes : kQ4TileBytes);
  constexpr int kCode = BITS == 2 ? kQ2CodeBytes : (BITS == 3 ? kQ3CodeBytes : kQ4CodeBytes);
  const int row = threadIdx.x & 127, G = threadIdx.x >> 7;
  for (int64_t tc = blockIdx.x; tc < n_tc; tc += gridDim.x) {
    const uint8_t* s_tile = src + tc * kBF16TileBytes;
    uint8_t* d_tile = dst + tc * kTile;
    float x[64];
#pragma unroll
    for (int q = 0; q < 8; ++q) {   // core matrices kg = 8G + q: k = 64G + 8q .. +7 of this row
      const uint4 v = *reinterpret_cast<const uint4*>(s_tile + core_off(row >> 3, 8 * G + q, row & 7, 0));
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        x[8 * q + 2 * e] = __uint_as_float(w4[e] << 16);
        x[8 * q + 2 * e + 1] = __uint_as_float(w4[e] & 0xFFFF0000u);
      }
    }
    float mn = x[0], mx = x[0];
#pragma unroll
    for (int i = 1; i < 64; ++i) {
      mn = fminf(mn, x[i]);
      mx = fmaxf(mx, x[i]);
    }
    const float sc = (mx == mn) ? 1.0f : __uint_as_float(uint32_t(f2bf(__fdiv_rn(__fsub_rn(mx, mn), kLevels))) << 16);
    float z = mn;
    if (hqq_iters > 0) z = __uint_as_float(uint32_t(f64_to_bf16_rne(hqq_refine_zero<BITS>(x, sc, mn, hqq_iters))) << 16);
    // codes in A-fragment order (common.cuh): lane t4 of this row's 8-row group takes the k with
    // (k % 16) / 2 % 4 == t4; word h of lane t4 holds k-steps 2h, 2h+1
    const int w = row >> 4, h = (row & 15) >> 3, g = row & 7;
    uint32_t words[4][2];
    uint32_t hib[4][2];   // Q3 high-bit bytes of this row: [t4][d]
#pragma unroll
    for (int t = 0; t < 4; ++t) words[t][0] = words[t][1] = hib[t][0] = hib[t][1] = 0u;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float t = __fdiv_rn(__fsub_rn(x[i], z), sc);
      const uint32_t r = uint32_t(fminf(fmaxf(rintf(t), 0.0f), kLevels));
      const int k4 = i >> 4, r16 = i & 15, t4 = (r16 & 7) >> 1, e = r16 >> 3, d = r16 & 1;
      if constexpr (BITS == 2) {
        words[t4][0] |= r << (d * 16 + 2 * (2 * k4 + e));
      } else if constexpr (BITS == 3) {
        words[t4][0] |= (r & 3u) << (d * 16 + 2 * (2 * k4 + e));
        hib[t4][d] |= (r >> 2) << (2 * k4 + e);
      } else {
        words[t4][k4 >> 1] |= r << (d * 16 + 4 * (2 * (k4 & 1) + e));
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int lane = g * 4 + t;
      if constexpr (BITS == 2 || BITS == 3)
        *reinterpret_cast<uint32_t*>(d_tile + ((w * 2 + G) * 32 + lane) * 8 + h * 4) = words[t][0];
      else
        *reinterpret_cast<uint2*>(d_tile + ((w * 2 + G) * 32 + lane) * 16 + h * 8) = make_uint2(words[t][0], words[t][1]);
      if constexpr (BITS == 3) {   // this row owns bytes h (d = 0) and 2 + h (d = 1) of the lane's high word
        uint8_t* hw = d_tile + kQ2CodeBytes + ((w * 2 + G) * 32 + lane) * 4;
        hw[h] = uint8_t(hib[t][0]);
        hw[2 + h] = uint8_t(hib[t][1]);
      }
    }
    *reinterpret_cast<uint32_t*>(d_tile + kCode + G * 512 + row * 4) = uint32_t(f2bf(sc)) | (uint32_t(f2bf(z)) << 16);
  }
}

void launch_quantize(const uint8_t* src_bf16_tiled, uint8_t* dst_q, int64_t N, int64_t K, int bits, int hqq_iters,
                     cudaStream_t st) {
  int64_t n_tc = (N / 128) * (K / 128);
  int blocks = int(n_tc < 148 * 8 ? n_tc : 148 * 8);
  if (bits == 2)
    quantize_q_kernel<2><<<blocks, 256, 0, st>>>(src_bf16_tiled, dst_q, n_tc, hqq_iters);
  else if (bits == 3)
    quantize_q_kernel<3><<<blocks, 256, 0, st>>>(src_bf16_tiled, dst_q, n_tc, hqq_iters);
  else
    quantize_q_kernel<4><<<blocks, 256, 0, st>>>(src_bf16_tiled, dst_q, n_tc, hqq_iters);
}

// ---- debug readbacks --------------------------------------------------------
__global__ void q4_to_canonical_kernel(const uint8_t* __restrict__ q4, uint8_t* codes, uint16_t* s, uint16_t* z,
                                       int64_t N, int64_t K) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < N * K; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t n = t / K, k = t % K;
    uint64_t off;
    int sh;
    q4_code_pos(n, k, K, &off, &sh);
    codes[t] = (q4[off] >> sh) & 15;
    if ((k & 63) == 0) {
      uint32_t m = *reinterpret_cast<const uint32_t*>(q4 + q4_meta_offset(n, k, K));
      s[n * (K / 64) + k / 64] = uint16_t(m & 0xFFFF);
      z[n * (K / 64) + k / 64] = uint16_t(m >> 16);
    }
  }
}
__global__ void tiled_to_natural_kernel(const uint8_t* __restrict__ t, uint16_t* out, int64_t N, int64_t K) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N * K; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = *reinterpret_cast<const uint16_t*>(t + bf16_tiled_offset(i / K, i % K, K));
}
void launch_q4_to_canonical(const uint8_t* q4, uint8_t* codes, uint16_t* s, uint16_t* z, int64_t N, int64_t K,
                            cudaStream_t st) {
  q4_to_canonical_kernel<<<1024, 256, 0, st>>>(q4, codes, s, z, N, K);
}
void launch_tiled_to_natural(const uint8_t* t, uint16_t* out, int64_t N, int64_t K, cudaStream_t st) {
  tiled_to_natural_kernel<<<1024, 256, 0, st>>>(t, out, N, K);
}

}  // namespace ss
