// Throwaway probe: TMA 1-D bulk-copy throughput vs op size, random 16B-aligned
// sources in an 18 GB buffer, W issuing warps, NS x 32 KB stages, consumer
// releases immediately.  Tells whether the gather is op-rate or byte-rate bound.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) { asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) { asm volatile("{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra LAB_WAIT;}" ::"r"(su32(b)), "r"(ph) : "memory"); }
template <int W, int NS>
__global__ void __launch_bounds__((W + 1) * 32, 1)
k(const uint8_t* __restrict__ base, uint64_t span, uint32_t op_bytes, uint32_t stages, uint64_t seed, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mbar_init(&full[i], W); mbar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint32_t ops = 32768 / op_bytes;  // per stage
  if (warp < W) {
    uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (uint32_t st = 0; st < stages; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      uint32_t mine = 0;
      for (uint32_t o = warp * 32 + lane; o < ops; o += W * 32) ++mine;
      uint32_t tot = mine * op_bytes;
      for (int x = 16; x; x >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, x);
      if (lane == 0) mbar_arrive_tx(&full[s], tot);
      __syncwarp();
      for (uint32_t o = warp * 32 + lane; o < ops; o += W * 32) {
        uint64_t h = (seed + blockIdx.x) * 0x9E3779B97F4A7C15ull + (uint64_t)st * 1315423911ull + o * 2654435761ull;
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        const uint64_t off = (h % (span / 64 - 1024)) * 64;
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(sm + s * 32768 + o * op_bytes)), "l"(base + off), "r"(op_bytes), "r"(su32(&full[s])), "l"(pol) : "memory");
      }
    }
  } else if (warp == W && lane == 0) {
    uint32_t acc = 0;
    for (uint32_t st = 0; st < stages; ++st) { const uint32_t s = st % NS; mbar_wait(&full[s], (st / NS) & 1); acc ^= sm[s * 32768 + (st & 1023)]; mbar_arrive(&empty[s]); }
    if (acc == 0x7F) sink[0] = acc;
  }
}
int main() {
  const uint64_t span = 18ull << 30;
  uint8_t* d; CK(cudaMalloc(&d, span)); CK(cudaMemset(d, 1, span));
  uint32_t* sink; CK(cudaMalloc(&sink, 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int W, uint32_t ob) {
    const uint32_t stages = 200;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    kern<<<sms, 32 * (W + 1), 4 * 32768>>>(d, span, ob, stages, 1, sink); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) kern<<<sms, 32 * (W + 1), 4 * 32768>>>(d, span, ob, stages, 2 + r, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    const double bytes = (double)sms * stages * 32768;
    printf("W=%d op=%5u B  %7.3f ms  %6.0f GB/s  %6.1f ns/op/SM\n", W, ob, ms, bytes / ms / 1e6, ms * 1e6 / (stages * (32768.0 / ob)));
  };
  for (uint32_t ob : {256u, 512u, 1024u, 2048u, 4096u, 8192u, 16384u}) run(k<1, 4>, 1, ob);
  for (uint32_t ob : {512u, 1024u, 2048u, 4096u}) run(k<2, 4>, 2, ob);
  for (uint32_t ob : {512u, 1024u, 2048u}) run(k<4, 4>, 4, ob);
  return 0;
}
