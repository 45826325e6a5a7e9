// Microbenchmark of tcgen05 issue costs on this part (one CTA): cycles per tcgen05.mma (A from
// TMEM or shared memory, M = 128, N = 16/32, K = 16), per tcgen05.commit, per mbarrier try_wait on a
// completed phase, and per tcgen05.st (32x32b.x32) + wait::st.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2509_18344_b200/csrc \
//        tools/probes/tc_probe.cu -o tools/probes/tc_probe
#include <cstdio>
#include "common.cuh"
using namespace ss;

__global__ void probe(unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[40 * 1024];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (warp == 0) tmem_alloc(&tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 0) {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = 0x3f803f80u;
    tmem_st32(tb + 128, v);
    tmem_wait_st();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t sb = smem_u32(sm);
    long long t0, t1;
    // 1) 32 x umma_ts N=16
    t0 = clock64();
    for (int i = 0; i < 32; ++i) umma_ts(tb, tb + 128 + (i & 3) * 8, umma_desc(sb + (i & 3) * 256, 128, 2048), umma_idesc_bf16(16), i > 0);
    t1 = clock64();
    out[0] = t1 - t0;
    umma_commit(&bar[0]);
    t0 = clock64();
    mbar_wait(&bar[0], 0);
    t1 = clock64();
    out[1] = t1 - t0;   // drain of the 32 MMAs after issue
    // 2) 32 x umma_ss N=16
    t0 = clock64();
    for (int i = 0; i < 32; ++i)
      umma_ss(tb, umma_desc(sb + (i & 7) * 256, 128, 2048), umma_desc(sb + 32768 + (i & 3) * 256, 128, 2048), umma_idesc_bf16(16), i > 0);
    t1 = clock64();
    out[2] = t1 - t0;
    umma_commit(&bar[1]);
    mbar_wait(&bar[1], 0);
    // 3) 32 x umma_ts N=32
    t0 = clock64();
    for (int i = 0; i < 32; ++i) umma_ts(tb, tb + 128 + (i & 3) * 8, umma_desc(sb + (i & 3) * 256, 128, 2048), umma_idesc_bf16(32), i > 0);
    t1 = clock64();
    out[3] = t1 - t0;
    umma_commit(&bar[2]);
    mbar_wait(&bar[2], 0);
    // 4) commit cost: 16 commits
    t0 = clock64();
    for (int i = 0; i < 16; ++i) umma_commit(&bar[3]);
    t1 = clock64();
    out[4] = t1 - t0;
    // 5) try_wait on a completed phase (bar[0] phase 0 done)
    t0 = clock64();
    for (int i = 0; i < 16; ++i) mbar_wait(&bar[0], 0);
    t1 = clock64();
    out[5] = t1 - t0;
    // 6) one MMA + commit + wait round trip
    t0 = clock64();
    umma_ts(tb, tb + 128, umma_desc(sb, 128, 2048), umma_idesc_bf16(16), 0);
    umma_commit(&bar[1]);
    mbar_wait(&bar[1], 1);
    t1 = clock64();
    out[6] = t1 - t0;
    // 7) 4 MMA + commit + wait round trip
    t0 = clock64();
    for (int i = 0; i < 4; ++i) umma_ts(tb, tb + 128 + i * 8, umma_desc(sb + i * 256, 128, 2048), umma_idesc_bf16(16), i > 0);
    umma_commit(&bar[2]);
    mbar_wait(&bar[2], 1);
    t1 = clock64();
    out[7] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) {   // 10) whole-warp issue, descriptors advanced by adds
    const uint32_t sb = smem_u32(sm);
    const uint64_t b0 = umma_desc(sb, 128, 2048), a0 = umma_desc(sb, 128, 2048), bb = umma_desc(sb + 32768, 128, 2048);
    long long t0 = clock64();
    for (int i = 0; i < 32; ++i) umma_ts_w(tb, tb + 128 + (i & 3) * 8, b0 + uint64_t((i & 3) * 16), umma_idesc_bf16(16), i > 0);
    long long t1 = clock64();
    if (lane == 0) out[10] = t1 - t0;
    umma_commit_w(&bar[3]);
    t0 = clock64();
    for (int i = 0; i < 32; ++i) umma_ss_w(tb, a0 + uint64_t((i & 7) * 16), bb + uint64_t((i & 3) * 16), umma_idesc_bf16(16), i > 0);
    t1 = clock64();
    if (lane == 0) out[11] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < 16; ++i) umma_commit_w(&bar[3]);
    t1 = clock64();
    if (lane == 0) out[12] = t1 - t0;
  }
  __syncthreads();
  if (warp == 1) {   // 8) tcgen05.st x32 + wait::st (warp 1 -> lanes 32..63)
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = i;
    long long t0 = clock64();
    for (int r = 0; r < 8; ++r) {
      tmem_st32(tb + (32u << 16) + 128 + (r & 1) * 32, v);
      tmem_wait_st();
    }
    long long t1 = clock64();
    if (lane == 0) out[8] = t1 - t0;
    uint32_t d[16];
    t0 = clock64();
    for (int r = 0; r < 8; ++r) {
      tmem_ld16(tb + (32u << 16) + (r & 1) * 16, d);
      tmem_wait_ld();
    }
    t1 = clock64();
    if (lane == 0) out[9] = t1 - t0 + (d[0] == 12345);
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64 * 8);
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 128>>>(d);
  unsigned long long h[16];
  cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  const char* names[] = {"32x umma_ts N16 issue", "drain after issue", "32x umma_ss N16 issue", "32x umma_ts N32 issue",
                         "16x commit", "16x try_wait completed", "1 mma+commit+wait", "4 mma+commit+wait",
                         "8x sttm32+wait (warp)", "8x ldtm16+wait (warp)", "32x umma_ts warp-elect", "32x umma_ss warp-elect",
                         "16x commit warp-elect"};
  for (int i = 0; i < 13; ++i) printf("%-28s %llu cycles\n", names[i], h[i]);
  return 0;
}
