// Shared device helpers for libsubspec (sm_100a).  No method arithmetic lives here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define SS_DEV __device__ __forceinline__
#define SS_HD __host__ __device__ __forceinline__

namespace ss {

constexpr int kTileRows = 128;      // weight rows per tile (one head at d_h = 128)
constexpr int kChunkK = 128;        // K elements per tile-chunk
constexpr int kQ4CodeBytes = 8192;  // 128 x 128 x 4 bit
constexpr int kQ4MetaBytes = 1024;  // 128 rows x 2 groups x (s,z) bf16
constexpr int kQ4TileBytes = kQ4CodeBytes + kQ4MetaBytes;   // 9216
constexpr int kBF16TileBytes = kTileRows * kChunkK * 2;     // 32768
constexpr int kXChunkBytesPerNT = 8 * kChunkK * 2;          // 2048: 8 tokens x 128 k bf16
constexpr int kTraceEvents = 16;   // u64 %globaltimer events per traced launch (debug)

// ---------------------------------------------------------------------------
// Weight "tiled fragment" layout.
// Matrix W [N x K] (N % 128 == 0, K % 128 == 0) is stored as tile-chunks
// (r = n/128, c = k/128), index tc = r * (K/128) + c, each contiguous.
// Inside a tile-chunk warp w (0..7) owns rows 16w..16w+15; lane = g*4 + t4 owns rows
// 16w+g (h=0) and 16w+g+8 (h=1).  Within the chunk, k = 64*G + 16*t4 + i16 (G = 64-group,
// i16 = 0..15), so every mma.m16n8k16 k-step st = 4*G + i16/4 stays inside one quant group.
// ---------------------------------------------------------------------------
struct KPos {
  int G, t4, i16, st, j;
};
SS_HD KPos kpos(int64_t k) {
  const int kk = int(k & 127);
  KPos p;
  p.G = kk >> 6;
  p.t4 = (kk & 63) >> 4;
  p.i16 = kk & 15;
  p.st = 4 * p.G + (p.i16 >> 2);
  p.j = p.i16 & 3;
  return p;
}
// byte offset, inside a bf16 tile-chunk, of the 16-byte piece q (= 2*G + half) of (warp w, row half h,
// lane): group-major, so each 64-k half of a tile-chunk (16 KB) is contiguous.
SS_HD int bf16_piece_off(int w, int h, int q, int lane) {
  return (((((q >> 1) * 8 + w) * 2 + h) * 2 + (q & 1)) * 32 + lane) * 16;
}
SS_HD uint64_t bf16_tiled_offset(int64_t n, int64_t k, int64_t K) {   // in bytes
  const int64_t tc = (n >> 7) * (K >> 7) + (k >> 7);
  const int nn = int(n & 127);
  const int w = nn >> 4, rr = nn & 15, h = rr >> 3, g = rr & 7;
  const KPos p = kpos(k);
  const int q = 2 * p.G + (p.i16 >> 3), e = p.i16 & 7;
  const int lane = g * 4 + p.t4;
  return uint64_t(tc) * kBF16TileBytes + uint64_t(bf16_piece_off(w, h, q, lane) + e * 2);
}

// Q4: per (warp w, group G, lane) 16 bytes = [row g: word0, word1][row g+8: word0, word1];
// word holds i16 = 8*word .. +7; code c8 = i16 % 8 lives in nibble slot (c8%2)*4 + c8/2, so
// (word >> 4p) & 0x000F000F yields the bf16x2 pair (c_2p, c_2p+1).
// Meta (4 B: s bf16 lo, z bf16 hi) at 8192 + ((w*2 + G)*16 + row_in_warp) * 4.
SS_HD uint64_t q4_tile_base(int64_t n, int64_t k, int64_t K) {
  return uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ4TileBytes;
}
SS_HD void q4_code_pos(int64_t n, int64_t k, int64_t K, uint64_t* byte_off, int* shift) {
  const int nn = int(n & 127);
  const int w = nn >> 4, rr = nn & 15, h = rr >> 3, g = rr & 7;
  const KPos p = kpos(k);
  const int lane = g * 4 + p.t4;
  const int word = p.i16 >> 3, c8 = p.i16 & 7;
  const int slot = (c8 & 1) * 4 + (c8 >> 1);
  const uint64_t wordoff = q4_tile_base(n, k, K) + uint64_t(((w * 2 + p.G) * 32 + lane) * 16 + h * 8 + word * 4);
  *byte_off = wordoff + (slot >> 1);
  *shift = (slot & 1) * 4;
}
SS_HD uint64_t q4_meta_offset(int64_t n, int64_t k, int64_t K) {     // bytes; 4 B (s lo16, z hi16)
  const int nn = int(n & 127);
  const int w = nn >> 4, rr = nn & 15;
  return q4_tile_base(n, k, K) + kQ4CodeBytes + uint64_t(((w * 2 + kpos(k).G) * 16 + rr) * 4);
}

// Q2 (NEXT-3, 2-bit substitutes): per (warp w, group G, lane) 8 bytes = [row g word][row g+8 word];
// the word holds i16 = 0..15 of the lane's 16 k of group G: code i16 lives in bits
// (i16 % 2) * 16 + 2 * (i16 / 2), so (word >> 2p) & 0x00030003 yields the bf16x2 pair
// (c_2p, c_2p+1) — k-step k4 uses pairs 2 k4 (a0/a1) and 2 k4 + 1 (a2/a3).
// Meta as Q4, at kQ2CodeBytes + ((w*2 + G)*16 + row_in_warp) * 4.
constexpr int kQ2CodeBytes = 4096;  // 128 x 128 x 2 bit
constexpr int kQ2TileBytes = kQ2CodeBytes + kQ4MetaBytes;   // 5120
SS_HD int qtile_bytes(int bits) { return bits == 2 ? kQ2TileBytes : kQ4TileBytes; }
SS_HD int qcode_bytes(int bits) { return bits == 2 ? kQ2CodeBytes : kQ4CodeBytes; }
SS_HD void q2_code_pos(int64_t n, int64_t k, int64_t K, uint64_t* byte_off, int* shift) {
  const int nn = int(n & 127);
  const int w = nn >> 4, rr = nn & 15, h = rr >> 3, g = rr & 7;
  const KPos p = kpos(k);
  const int lane = g * 4 + p.t4;
  const int bit = (p.i16 & 1) * 16 + 2 * (p.i16 >> 1);
  const uint64_t wordoff = uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ2TileBytes +
                           uint64_t(((w * 2 + p.G) * 32 + lane) * 8 + h * 4);
  *byte_off = wordoff + (bit >> 3);
  *shift = bit & 7;
}
SS_HD uint64_t q2_meta_offset(int64_t n, int64_t k, int64_t K) {
  const int nn = int(n & 127);
  const int w = nn >> 4, rr = nn & 15;
  return uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ2TileBytes + kQ2CodeBytes +
         uint64_t(((w * 2 + kpos(k).G) * 16 + rr) * 4);
}

// ---------------------------------------------------------------------------
// FragX activation layout: X [Mpad x K] bf16, Mpad % 8 == 0, NT = Mpad/8.
// Chunk c (128 k) of all NT n-tiles is contiguous (NT * 2 KB); within it
// offset(m,k) = ((((c*NT + nt)*8 + st)*4 + t4)*8 + g)*4 + j  with (st, t4, j) = kpos(k),
// nt = m/8, g = m%8: the 8 bytes lane (g, t4) needs for k-step st are contiguous.
// ---------------------------------------------------------------------------
SS_HD int64_t fragx_offset(int64_t m, int64_t k, int NT) {
  const int64_t c = k >> 7;
  const KPos p = kpos(k);
  const int nt = int(m >> 3), g = int(m & 7);
  return ((((c * NT + nt) * 8 + p.st) * 4 + p.t4) * 8 + g) * 4 + p.j;
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
SS_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SS_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

SS_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

SS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SS_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
SS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// (x & 0x000F000F) | magic in ONE lop3 (C++ "(x & a) | b" becomes two LOP3s with immediates)
SS_DEV uint32_t lop3_and_or(uint32_t x, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(d) : "r"(x), "r"(magic));
  return d;
}
SS_DEV uint32_t lop3_and_or2(uint32_t x, uint32_t magic) {   // 2-bit codes: (x & 0x00030003) | magic
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x00030003, %2, 0xEA;" : "=r"(d) : "r"(x), "r"(magic));
  return d;
}
// 1-D bulk async copy global -> shared, completion counted on an mbarrier (TMA engine; SASS UBLKCP)
SS_DEV void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
SS_DEV void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// TMA-engine prefetch of a global range into L2 (no shared memory involved)
SS_DEV void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
SS_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

SS_DEV void mma_bf16_16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                           uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

SS_DEV float bf2f(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }
SS_DEV uint16_t f2bf(float f) {   // RNE (finite inputs)
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
SS_DEV float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SS_DEV float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace ss
