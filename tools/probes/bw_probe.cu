// Memory-system probe for the K2 design: how fast can 148 persistent CTAs stream N bytes with
// (a) cp.async.bulk into an smem ring (stage bytes B, S stages), (b) plain LDG.128 unrolled?
// Back-to-back launches over a 4 GB buffer so nothing is L2-resident.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(288, 1) bulk_stream(const uint8_t* src, int64_t bytes, int stage_bytes, int stages, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + stages * stage_bytes);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" :: "r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t per = bytes / gridDim.x / stage_bytes;   // stages per CTA
  const uint8_t* base = src + int64_t(blockIdx.x) * per * stage_bytes;
  if (warp == 8) {
    if (lane == 0) {
      for (int64_t i = 0; i < per; ++i) {
        int s = i % stages;
        if (i >= stages) {
          uint32_t ph = ((i / stages) - 1) & 1;
          asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(su(&empty[s])), "r"(ph));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(stage_bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su(sm + s * stage_bytes)), "l"(base + i * stage_bytes), "r"(stage_bytes), "r"(su(&full[s])));
      }
    }
    return;
  }
  float acc = 0.f;
  for (int64_t i = 0; i < per; ++i) {
    int s = i % stages;
    uint32_t ph = (i / stages) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(su(&full[s])), "r"(ph));
    acc += ((const float*)(sm + s * stage_bytes))[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[s])));
  }
  if (acc == 12345.f) *sink = acc;
}
__global__ void __launch_bounds__(288, 1) bulk_stream_pdl(const uint8_t* src, int64_t bytes, int stage_bytes, int stages, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + stages * stage_bytes);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" :: "r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t per = bytes / gridDim.x / stage_bytes;
  const uint8_t* base = src + int64_t(blockIdx.x) * per * stage_bytes;
  if (warp == 8) {
    if (lane == 0) {
      for (int64_t i = 0; i < per; ++i) {
        int s = i % stages;
        if (i >= stages) {
          uint32_t ph = ((i / stages) - 1) & 1;
          asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(su(&empty[s])), "r"(ph));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(stage_bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su(sm + s * stage_bytes)), "l"(base + i * stage_bytes), "r"(stage_bytes), "r"(su(&full[s])));
      }
    }
    return;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float acc = 0.f;
  for (int64_t i = 0; i < per; ++i) {
    int s = i % stages;
    uint32_t ph = (i / stages) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(su(&full[s])), "r"(ph));
    acc += ((const float*)(sm + s * stage_bytes))[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[s])));
  }
  if (acc == 12345.f) *sink = acc;
}
__global__ void ldg_stream(const uint4* src, int64_t n16, float* sink) {
  uint32_t acc = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc ^= src[i].x;
  if (acc == 0x12345) *sink = 1.f;
}
int main() {
  const int64_t pool = 4ll << 30;
  uint8_t* buf; float* sink;
  CK(cudaMalloc(&buf, pool)); CK(cudaMalloc(&sink, 4)); CK(cudaMemset(buf, 1, pool));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(bulk_stream_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  // PDL chain: 4 matrix sizes of a Qwen-7B layer in pass order, repeated over 28 "layers"
  {
    const int64_t lay[4] = {9289728, 7225344, 76382208, 38191104};
    for (int st : {4, 8}) for (int sb : {9216, 18432}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.blockDim = dim3(288); cfg.dynamicSmemBytes = sb * st + 256; cfg.attrs = at; cfg.numAttrs = 1; cfg.stream = 0;
      for (int pdl = 0; pdl < 2; ++pdl) {
        cfg.numAttrs = pdl;
        double tot_bytes = 0;
        int64_t off = 0;
        for (int w = 0; w < 2; ++w) {
          if (w == 1) cudaEventRecord(e0);
          off = 0; tot_bytes = 0;
          for (int l = 0; l < 28; ++l) for (int g = 0; g < 4; ++g) {
            int64_t per = lay[g] / sms / sb; if (per < 1) per = 1;
            int64_t nb = per * sb * sms;
            cfg.gridDim = dim3(sms);
            cudaLaunchKernelEx(&cfg, bulk_stream_pdl, (const uint8_t*)(buf + off), nb, sb, st, sink);
            off += nb; tot_bytes += nb;
          }
        }
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("layer-chain pdl=%d stage=%d stages=%d: %.1f us per layer (4 kernels), %.1f GB/s\n", pdl, sb, st, ms * 1000 / 28, tot_bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  const int64_t sizes[] = {9437184, 76546048};
  for (int64_t bytes : sizes) {
    for (int sb : {9216, 18432, 36864}) for (int st : {2, 4, 8}) {
      if (sb * st > 200 * 1024) continue;
      for (int cps : {1, 2}) {
        int grid = sms * cps;
        if (sb * st * cps > 220 * 1024) continue;
        int64_t per = bytes / grid / sb; if (per < 1) continue;
        int64_t nb = per * sb * grid;
        int reps = int(std::min<int64_t>(40, pool / nb));
        bulk_stream<<<grid, 288, sb * st + 256>>>(buf, nb, sb, st, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) bulk_stream<<<grid, 288, sb * st + 256>>>(buf + r * nb, nb, sb, st, sink);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("bulk bytes=%10lld stage=%6d stages=%d ctas/sm=%d : %8.2f us  %7.1f GB/s\n", (long long)nb, sb, st, cps, ms * 1000 / reps, nb * reps / (ms * 1e-3) / 1e9);
      }
    }
    for (int bpsm : {4, 8, 16}) {
      int64_t n16 = bytes / 16;
      int reps = int(std::min<int64_t>(40, pool / bytes));
      ldg_stream<<<sms * bpsm, 256>>>((const uint4*)buf, n16, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) ldg_stream<<<sms * bpsm, 256>>>((const uint4*)(buf + r * bytes), n16, sink);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg  bytes=%10lld blocks/sm=%d : %8.2f us  %7.1f GB/s\n", (long long)bytes, bpsm, ms * 1000 / reps, bytes * reps / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
