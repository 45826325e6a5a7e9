// Occupancy-calculator probe: does tcgen05 TMEM allocation limit resident CTAs per SM?
#include <cstdio>
#include "common.cuh"
using namespace ss;
__global__ void __launch_bounds__(320) plain_k(int* o) { if (threadIdx.x == 0 && o) o[0] = 1; }
__global__ void __launch_bounds__(320) tmem_k(int* o) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc(&slot, 128);
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(slot, 128);
  if (threadIdx.x == 0 && o) o[0] = 1;
}
__global__ void __launch_bounds__(320) tmem_noperm_k(int* o) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(128) : "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(slot, 128);
  if (threadIdx.x == 0 && o) o[0] = 1;
}
int main() {
  int a = 0, b = 0, c = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, plain_k, 320, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tmem_k, 320, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, tmem_noperm_k, 320, 0);
  printf("plain %d tmem %d tmem_noperm %d\n", a, b, c);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tmem_k);
  printf("tmem_k regs %d\n", fa.numRegs);
  return 0;
}
