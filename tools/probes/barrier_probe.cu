// Grid-barrier latency on B200 with 148 co-resident CTAs (cooperative launch), 288 threads each.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
template <int MODE>
__global__ void __launch_bounds__(288, 1) bar_kernel(unsigned* ctr, unsigned* flag, int iters, int sleep_ns) {
  if (threadIdx.x >= 256) return;   // the producer warp never takes part
  for (int i = 1; i <= iters; ++i) {
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (threadIdx.x == 0) {
      if (MODE == 0) {          // fence + atomicAdd + poll counter (current implementation)
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acq(ctr) < unsigned(i) * gridDim.x) { if (sleep_ns) __nanosleep(sleep_ns); }
        __threadfence();
      } else if (MODE == 1) {   // red.release + poll counter with ld.acquire, no extra fences
        red_rel(ctr, 1u);
        while (ld_acq(ctr) < unsigned(i) * gridDim.x) { if (sleep_ns) __nanosleep(sleep_ns); }
      } else {                  // arrive with atom; last arriver releases a generation flag
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        if (old == unsigned(i) * gridDim.x - 1) {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(flag), "r"(unsigned(i)) : "memory");
        } else {
          while (ld_acq(flag) < unsigned(i)) { if (sleep_ns) __nanosleep(sleep_ns); }
        }
      }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
}
int main() {
  unsigned *ctr, *flag; cudaMalloc(&ctr, 4); cudaMalloc(&flag, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  void (*ks[3])(unsigned*, unsigned*, int, int) = {bar_kernel<0>, bar_kernel<1>, bar_kernel<2>};
  for (int mode = 0; mode < 3; ++mode) for (int sl : {0, 20, 100}) {
    int iters = 2000;
    cudaMemset(ctr, 0, 4); cudaMemset(flag, 0, 4);
    void* args[] = {&ctr, &flag, &iters, &sl};
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)ks[mode], dim3(sms), dim3(288), args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d sleep %3d: %s %.3f us per barrier\n", mode, sl, cudaGetErrorString(e), ms * 1000 / iters);
    fflush(stdout);
  }
  return 0;
}
