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
constexpr int kQ4MetaBytes = 1024;  // 2 groups x 128 rows x (s,z) bf16
constexpr int kQ4TileBytes = kQ4CodeBytes + kQ4MetaBytes;   // 9216
constexpr int kBF16TileBytes = kTileRows * kChunkK * 2;     // 32768
constexpr int kXChunkBytesPerNT = 8 * kChunkK * 2;          // 2048: 8 tokens x 128 k bf16
constexpr int kTraceEvents = 16;   // u64 %globaltimer events per traced launch (debug)

// ---------------------------------------------------------------------------
// Core-matrix layouts.  A core matrix is 8 rows x 8 consecutive k
// (bf16, 16 B per row, 128 B contiguous): the unit of both `ldmatrix` (one 8-lane phase) and the
// tcgen05 K-major SWIZZLE_NONE shared-memory descriptor (LBO = K-direction core stride, SBO =
// row-group stride).  A 128-k chunk of 8*R rows holds core (rg, kg) at ((rg * 16 + kg) * 128) bytes,
// so LBO = 128 B and SBO = 2048 B for every operand below, and advancing K by 16 is +256 B.
// ---------------------------------------------------------------------------
SS_HD uint32_t core_off(int rg, int kg, int r, int e) { return uint32_t(((rg * 16 + kg) * 64 + r * 8 + e) * 2); }

// bf16 weights W [N x K] (N % 128 == 0, K % 128 == 0): tile-chunks (row tile n/128, chunk k/128),
// index tc = (n/128) * (K/128) + k/128, 32 KB each, core matrices inside as above.
SS_HD uint64_t bf16_tiled_offset(int64_t n, int64_t k, int64_t K) {   // in bytes
  const int64_t tc = (n >> 7) * (K >> 7) + (k >> 7);
  const int nn = int(n & 127), kk = int(k & 127);
  return uint64_t(tc) * kBF16TileBytes + core_off(nn >> 3, kk >> 3, nn & 7, kk & 7);
}

// Q4 substitutes: codes in mma.m16n8k16 A-fragment order with natural k.  Per tile-chunk, for warp
// w (rows 16w .. 16w+15), 64-group G and lane (g = lane / 4, t4 = lane % 4): 16 bytes at
// ((w * 2 + G) * 32 + lane) * 16 = [row 16w+g: word0, word1][row 16w+g+8: word0, word1].  Word h
// holds the k-steps k4 = 2h, 2h+1 of the group; pair p = 2 (k4 % 2) + e (e = 0: k = 16 k4 + 2 t4,
// +1; e = 1: k + 8, +9) has its first code at bits 4p .. 4p+3 and its second at bits 16 + 4p, so
// (word >> 4p) & 0x000F000F is the pair's bf16x2 mantissa bits (the A registers a0..a3 of the
// k-step).  Then meta (s bf16 lo16, z bf16 hi16) at 8192 + G * 512 + row * 4.
SS_HD uint64_t q4_tile_base(int64_t n, int64_t k, int64_t K) {
  return uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ4TileBytes;
}
SS_HD void q4_code_pos(int64_t n, int64_t k, int64_t K, uint64_t* byte_off, int* shift) {
  const int row = int(n & 127), kk = int(k & 127);
  const int w = row >> 4, h = (row & 15) >> 3, g = row & 7;
  const int G = kk >> 6, kl = kk & 63, k4 = kl >> 4, r16 = kl & 15;
  const int t4 = (r16 & 7) >> 1, e = r16 >> 3, d = r16 & 1;
  const int lane = g * 4 + t4, p = 2 * (k4 & 1) + e, bit = d * 16 + 4 * p;
  *byte_off = q4_tile_base(n, k, K) + uint64_t(((w * 2 + G) * 32 + lane) * 16 + h * 8 + (k4 >> 1) * 4 + (bit >> 3));
  *shift = bit & 7;
}
SS_HD uint64_t q4_meta_offset(int64_t n, int64_t k, int64_t K) {     // bytes; 4 B (s lo16, z hi16)
  return q4_tile_base(n, k, K) + kQ4CodeBytes + uint64_t(((k & 127) >> 6) * 512 + (n & 127) * 4);
}

// Q2 (NEXT-3, 2-bit substitutes): per (w, G, lane) 8 bytes = [row g word][row g+8 word]; pair
// p = 2 k4 + e (k as for Q4) at bits 2p (first) and 16 + 2p (second), so (word >> 2p) & 0x00030003
// is a pair; meta as Q4 at kQ2CodeBytes + G * 512 + row * 4.
constexpr int kQ2CodeBytes = 4096;  // 128 x 128 x 2 bit
constexpr int kQ2TileBytes = kQ2CodeBytes + kQ4MetaBytes;   // 5120
// Q3 (NEXT-3, 3-bit substitutes): the low two bits of every code in the Q2 layout
// (4096 B), then a plane of the high bits: per (w, G, lane) one 32-bit word at 4096 +
// ((w * 2 + G) * 32 + lane) * 4 whose bit d * 16 + h * 8 + p is the high bit of pair p's code d of
// row g + 8h, so (word >> (8h + p - 2)) & 0x00040004 (a left shift for 8h + p < 2) puts the pair's
// high bits at bf16 mantissa bit 2; meta as Q4 at kQ3CodeBytes + G * 512 + row * 4.
constexpr int kQ3CodeBytes = 6144;  // 128 x 128 x 3 bit
constexpr int kQ3TileBytes = kQ3CodeBytes + kQ4MetaBytes;   // 7168
SS_HD int qtile_bytes(int bits) { return bits == 2 ? kQ2TileBytes : (bits == 3 ? kQ3TileBytes : kQ4TileBytes); }
SS_HD int qcode_bytes(int bits) { return bits == 2 ? kQ2CodeBytes : (bits == 3 ? kQ3CodeBytes : kQ4CodeBytes); }
SS_HD void q2_code_pos(int64_t n, int64_t k, int64_t K, uint64_t* byte_off, int* shift) {
  const int row = int(n & 127), kk = int(k & 127);
  const int w = row >> 4, h = (row & 15) >> 3, g = row & 7;
  const int G = kk >> 6, kl = kk & 63, k4 = kl >> 4, r16 = kl & 15;
  const int t4 = (r16 & 7) >> 1, e = r16 >> 3, d = r16 & 1;
  const int lane = g * 4 + t4, p = 2 * k4 + e, bit = d * 16 + 2 * p;
  *byte_off = uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ2TileBytes +
              uint64_t(((w * 2 + G) * 32 + lane) * 8 + h * 4 + (bit >> 3));
  *shift = bit & 7;
}
SS_HD uint64_t q2_meta_offset(int64_t n, int64_t k, int64_t K) {
  return uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ2TileBytes + kQ2CodeBytes +
         uint64_t(((k & 127) >> 6) * 512 + (n & 127) * 4);
}
// Q3: low two bits at (*lo_off, *lo_shift) (the Q2 position inside the Q3 tile), high bit at
// (*hi_off, *hi_bit)
SS_HD void q3_code_pos(int64_t n, int64_t k, int64_t K, uint64_t* lo_off, int* lo_shift, uint64_t* hi_off,
                       int* hi_bit) {
  const int row = int(n & 127), kk = int(k & 127);
  const int w = row >> 4, h = (row & 15) >> 3, g = row & 7;
  const int G = kk >> 6, kl = kk & 63, k4 = kl >> 4, r16 = kl & 15;
  const int t4 = (r16 & 7) >> 1, e = r16 >> 3, d = r16 & 1;
  const int lane = g * 4 + t4, p = 2 * k4 + e, bit = d * 16 + 2 * p, hb = d * 16 + h * 8 + p;
  const uint64_t base = uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ3TileBytes;
  *lo_off = base + uint64_t(((w * 2 + G) * 32 + lane) * 8 + h * 4 + (bit >> 3));
  *lo_shift = bit & 7;
  *hi_off = base + kQ2CodeBytes + uint64_t(((w * 2 + G) * 32 + lane) * 4 + (hb >> 3));
  *hi_bit = hb & 7;
}
SS_HD uint64_t q3_meta_offset(int64_t n, int64_t k, int64_t K) {
  return uint64_t((n >> 7) * (K >> 7) + (k >> 7)) * kQ3TileBytes + kQ3CodeBytes +
         uint64_t(((k & 127) >> 6) * 512 + (n & 127) * 4);
}

// ---------------------------------------------------------------------------
// Activation layout ("FragX", now core-matrix): X [Mpad x K] bf16, Mpad % 8 == 0, NT = Mpad / 8 token
// groups.  Chunk c (128 k) of all NT token groups is contiguous (NT * 2 KB); inside it token group tg
// holds core (tg, kg) at ((tg * 16 + kg) * 64) elements, so the B operand of a tcgen05 MMA (N = 8 NT
// tokens, K-major) and the mma.sync B fragments (ldmatrix) read it directly.  offset in elements.
// ---------------------------------------------------------------------------
SS_HD int64_t fragx_offset(int64_t m, int64_t k, int NT) {
  const int64_t c = k >> 7;
  const int kk = int(k & 127);
  return ((c * NT + (m >> 3)) * 16 + (kk >> 3)) * 64 + (m & 7) * 8 + (kk & 7);
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
SS_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(addr), "r"(parity)
      : "memory");
  return done != 0;
}
// wait for the phase with this parity; a watchdog traps after ~4 s instead of hanging the GPU
SS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(addr, parity)) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 4000000000ull) __trap();
  }
}
// (x & 0x000F000F) | magic in ONE lop3 (C++ "(x & a) | b" becomes two LOP3s with immediates)
SS_DEV uint32_t lop3_and_or(uint32_t x, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(d) : "r"(x), "r"(magic));
  return d;
}
SS_DEV uint32_t lop3_and_or_hi(uint32_t x, uint32_t pair) {   // 3-bit codes: (x & 0x00040004) | pair
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x00040004, %2, 0xEA;" : "=r"(d) : "r"(x), "r"(pair));
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

// ldmatrix: four 8x8 b16 core matrices; lane L supplies the row address of matrix L / 8
SS_DEV void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}

// ---- tcgen05 (5th-generation tensor core, TMEM) --------------------------------------------
// shared-memory matrix descriptor, K-major, SWIZZLE_NONE (canonical core-matrix layout above)
SS_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);   // version 1 (sm_100), layout 0
}
// instruction descriptor: kind::f16, A = B = bf16, D = f32, both K-major, M = 128, N
SS_HD constexpr uint32_t umma_idesc_bf16(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
// D[tmem] (+)= A[tmem] * B[smem]   (A: 128 lanes = rows, K = 16 bf16 in 8 columns)
SS_DEV void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[smem] * B[smem]
SS_DEV void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on an mbarrier when every tcgen05.mma issued so far by this thread has completed
SS_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// warp-wide forms: the whole (converged) warp executes them, one elected lane issues, so the
// operands stay warp-uniform (uniform registers, no per-MMA broadcast loop)
SS_DEV void umma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
SS_DEV void umma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
SS_DEV void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
SS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SS_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {   // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
SS_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {   // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// this warp's 32 TMEM lanes, 32 consecutive 32-bit columns from taddr
SS_DEV void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
SS_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
SS_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
SS_DEV void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
SS_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
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
