// Does the hardware co-schedule two CTAs of a TMEM-allocating kernel on one SM (the occupancy
// calculator says 1)?  296 CTAs that each hold TMEM for ~20 us: count the CTAs alive at once.
#include <cstdio>
#include <vector>
#include <algorithm>
#include "common.cuh"
using namespace ss;
__global__ void __launch_bounds__(320) tmem_k(unsigned long long* o, int ncols) {
  __shared__ uint32_t slot;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x < 32) tmem_alloc(&slot, ncols);
  __syncthreads();
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < 20000);
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(slot, ncols);
  if (threadIdx.x == 0) { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); o[3 * blockIdx.x] = sm; o[3 * blockIdx.x + 1] = t0; o[3 * blockIdx.x + 2] = t1; }
}
__global__ void __launch_bounds__(320) plain_k(unsigned long long* o, int) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < 20000);
  if (threadIdx.x == 0) { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); o[3 * blockIdx.x] = sm; o[3 * blockIdx.x + 1] = t0; o[3 * blockIdx.x + 2] = t1; }
}
static void report(const char* name, unsigned long long* d, int n) {
  std::vector<unsigned long long> h(3 * n);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, tend = 0;
  for (int i = 0; i < n; ++i) { t0 = std::min(t0, h[3 * i + 1]); tend = std::max(tend, h[3 * i + 2]); }
  int late = 0;
  for (int i = 0; i < n; ++i) late += (h[3 * i + 1] - t0) > 10000;
  printf("%s: %d CTAs, started >10us late: %d, span %.1f us\n", name, n, late, (tend - t0) / 1e3);
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 3 * 600 * 8);
  for (int ncols : {128, 256}) {
    tmem_k<<<296, 320>>>(d, ncols);
    cudaDeviceSynchronize();
    char nm[64];
    snprintf(nm, 64, "tmem %d cols", ncols);
    report(nm, d, 296);
  }
  plain_k<<<296, 320>>>(d, 0);
  cudaDeviceSynchronize();
  report("plain", d, 296);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
