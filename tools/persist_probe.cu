// persist_probe.cu -- can a small kernel run beside a persistent kernel that
// holds one CTA per SM?  Variants: dynamic smem, threads, TMEM allocation.
// A spinner (grid = #SMs) polls a flag until a helper kernel on another
// stream sets it (or 1 s passes); prints how long the helper took to start.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void spinner(volatile unsigned* flag, int use_tmem, unsigned long long* t_out) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned holder;
  if (use_tmem && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((unsigned)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  sm[threadIdx.x] = 1;
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) {
    while (*flag == 0 && gt() - t0 < 1000000000ull) __nanosleep(200);
    if (blockIdx.x == 0) t_out[0] = gt() - t0;
  }
  __syncthreads();
  if (use_tmem && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(holder));
}

__global__ void helper(volatile unsigned* flag) { if (threadIdx.x == 0) *flag = 1; }

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = argc > 1 ? atoi(argv[1]) : 200000, threads = argc > 2 ? atoi(argv[2]) : 544;
  const int tmem = argc > 3 ? atoi(argv[3]) : 0, carve = argc > 4 ? atoi(argv[4]) : 1;
  cudaFuncSetAttribute(spinner, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // carve bits: 1 spinner prefers max smem, 2 helper prefers max smem, 4 helper preloaded (attributes query)
  if (carve & 1) cudaFuncSetAttribute(spinner, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (carve & 2) cudaFuncSetAttribute(helper, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (carve & 4) { cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, helper); }
  unsigned* flag; unsigned long long* t;
  cudaMalloc(&flag, 4); cudaMalloc(&t, 8); cudaMemset(flag, 0, 4); cudaMemset(t, 0, 8);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  spinner<<<sms, threads, smem, a>>>(flag, tmem, t);
  cudaError_t e = cudaGetLastError();
  helper<<<1, 32, 0, b>>>(flag);
  cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("smem=%d threads=%d tmem=%d carve=%d launch=%s : helper released the spinner after %.3f ms%s\n", smem, threads,
         tmem, carve, cudaGetErrorString(e), h / 1e6, h >= 999000000ull ? "  (BLOCKED)" : "");
  return 0;
}
