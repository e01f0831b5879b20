// Throwaway probe: does compute-sanitizer racecheck model mbarrier-based
// producer/consumer synchronisation (the MaxSim kernel's only intra-CTA sync)?
// Each variant is a CORRECT program under the PTX memory model:
//   A  warp 0: 32 lanes write smem, __syncwarp, lane 0 mbarrier.arrive (count 1);
//      warp 1: mbarrier.try_wait.parity, then reads       (the kernel's pattern)
//   B  as A, but all 32 lanes arrive (count 32)
//   C  as A, but __syncthreads instead of the mbarrier     (control)
//   D  warp 0 lane 0: cp.async.bulk global -> smem completing on the mbarrier
//      (expect_tx); warp 1 waits, reads                    (the TMA landing)
//   E  WAR through the tensor-core proxy: warp 1 reads smem, then releases it
//      with tcgen05.commit (arrive::one, nothing pending); warp 0 waits, writes
//      (how the MMA warp frees a stage / TMEM buffer)
//   F  as E with a plain mbarrier.arrive by every lane of warp 1 (control)
// Run: compute-sanitizer --tool racecheck ./racecheck_probe
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(su32(b)), "r"(ph) : "memory");
}
template <int V>
__global__ void k(const uint4* g, uint32_t* out) {
  __shared__ __align__(128) uint4 buf[32];
  __shared__ uint64_t bar;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(V == 1 || V == 5 ? 32 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (V == 4 || V == 5) {  // WAR: warp 1 reads first, warp 0 writes after the release
    if (w == 1) {
      out[l] = buf[31 - l].x;
      __syncwarp();
      if (V == 4) {
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su32(&bar)) : "memory");
      } else {
        arrive(&bar);
      }
    } else {
      wait(&bar, 0);
      buf[l] = make_uint4(l, l, l, l);
    }
    return;
  }
  if (V == 2) {
    if (w == 0) buf[l] = make_uint4(l, l, l, l);
    __syncthreads();
    if (w == 1) out[l] = buf[31 - l].x;
    return;
  }
  if (w == 0) {
    if (V == 3) {
      if (l == 0) {
        asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(su32(&bar)), "r"(512) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(buf)), "l"(g), "r"(512), "r"(su32(&bar)) : "memory");
      }
    } else {
      buf[l] = make_uint4(l, l, l, l);
      __syncwarp();
      if (V == 1 || l == 0) arrive(&bar);
    }
  } else {
    wait(&bar, 0);
    out[l] = buf[31 - l].x;
  }
}
int main() {
  uint4* g; uint32_t* o;
  cudaMalloc(&g, 512); cudaMemset(g, 1, 512); cudaMalloc(&o, 128);
  k<0><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("A done\n");
  k<1><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("B done\n");
  k<2><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("C done\n");
  k<3><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("D done\n");
  k<4><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("E done\n");
  k<5><<<1, 64>>>(g, o); cudaDeviceSynchronize(); printf("F done\n");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
