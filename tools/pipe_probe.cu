// Throwaway probe: the MaxSim kernel's copy pipeline without MMA/epilogue.
// W copy warps fill a ring of NS stages (32 KB, 512 slots x 64 B) from a slot
// table of random docs; one consumer warp waits "full" and releases "empty".
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra LAB_WAIT;}" ::"r"(su32(b)), "r"(ph) : "memory");
}

// MODE 0: cp.async 16B + arrive.noinc ; MODE 1: LDG.128 -> STS (regs), unroll 4
template <int W, int NS, int MODE>
__global__ void __launch_bounds__((W + 1) * 32, 1)
pipe(const uint4* __restrict__ rows, const uint2* __restrict__ grp, uint64_t n_groups_total, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], W * 32); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // each CTA streams its contiguous share of the group table, 64 groups (512 slots) per stage
  const uint64_t per_cta = n_groups_total / gridDim.x;
  const uint64_t g_begin = blockIdx.x * per_cta;
  const uint32_t n_st = (uint32_t)(per_cta / 64);
  if (warp < W) {
    for (uint32_t st = 0; st < n_st; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      const uint32_t sbase = su32(sm + s * 32768);
      const uint2* g = grp + g_begin + (uint64_t)st * 64;
      if (MODE == 0) {
#pragma unroll 4
        for (uint32_t e = warp * 32 + lane; e < 2048; e += W * 32) {
          const uint32_t rel = e >> 2, c = e & 3;
          const uint2 gr = g[rel >> 3];
          const uint32_t row = min(gr.x + (rel & 7u), gr.y);
          const uint32_t dst = sbase + ((rel >> 7) * 8192) + ((rel & 127) >> 3) * 512 + c * 128 + (rel & 7) * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(rows + (size_t)row * 4 + c) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
      } else {
        constexpr int PER = 2048 / (W * 32);
        uint4 v[PER];
        uint32_t d[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const uint32_t e = warp * 32 + lane + i * W * 32;
          const uint32_t rel = e >> 2, c = e & 3;
          const uint2 gr = g[rel >> 3];
          const uint32_t row = min(gr.x + (rel & 7u), gr.y);
          d[i] = ((rel >> 7) * 8192) + ((rel & 127) >> 3) * 512 + c * 128 + (rel & 7) * 16;
          v[i] = __ldcs(rows + (size_t)row * 4 + c);
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) *reinterpret_cast<uint4*>(sm + s * 32768 + d[i]) = v[i];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[s]);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (lane == 0) {
    uint32_t acc = 0;
    for (uint32_t st = 0; st < n_st; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&full[s], (st / NS) & 1);
      acc ^= *reinterpret_cast<uint32_t*>(sm + s * 32768 + (st & 1023) * 4);
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

int main() {
  const uint64_t N = 8800000;
  std::mt19937_64 rng(1);
  std::vector<uint64_t> rp(N + 1, 0);
  for (uint64_t i = 0; i < N; ++i) rp[i + 1] = rp[i] + 1 + rng() % 63;
  const uint64_t T = rp[N];
  // group table for ~8 batches of 64 x 1000 random docs (8-aligned slot packing)
  std::vector<uint2> grp;
  uint64_t bytes = 0;
  for (int i = 0; i < 512000; ++i) {
    uint64_t id = rng() % N;
    uint32_t r0 = (uint32_t)rp[id], t = (uint32_t)(rp[id + 1] - rp[id]);
    for (uint32_t g = 0; g < (t + 7) / 8; ++g) grp.push_back(make_uint2(r0 + 8 * g, r0 + t - 1));
    bytes += t * 64ull;
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t ng = grp.size() / (sms * 64) * (sms * 64);
  double slot_bytes = ng * 8 * 64.0;  // incl. pad slots (re-reads of the last row hit L2)
  printf("groups %llu, doc bytes %.1f MB, slot bytes %.1f MB\n", (unsigned long long)ng, bytes / 1e6, slot_bytes / 1e6);
  uint4* d_rows; uint2* d_grp; uint32_t* sink;
  CK(cudaMalloc(&d_rows, T * 64)); CK(cudaMemset(d_rows, 1, T * 64));
  CK(cudaMalloc(&d_grp, ng * 8)); CK(cudaMemcpy(d_grp, grp.data(), ng * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double doc_frac = (double)bytes / (grp.size() * 512.0);
  auto run = [&](const char* name, auto kern, int threads, int ns) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768));
    for (int w = 0; w < 2; ++w) kern<<<sms, threads, ns * 32768>>>(d_rows, d_grp, ng, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<sms, threads, ns * 32768>>>(d_rows, d_grp, ng, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-36s %7.3f ms  unique-row %6.0f GB/s\n", name, ms, slot_bytes * doc_frac / ms / 1e6);
  };
  run("cp.async W=4 NS=4", pipe<4, 4, 0>, 5 * 32, 4);
  run("cp.async W=8 NS=4", pipe<8, 4, 0>, 9 * 32, 4);
  run("cp.async W=16 NS=4", pipe<16, 4, 0>, 17 * 32, 4);
  run("cp.async W=8 NS=6", pipe<8, 6, 0>, 9 * 32, 6);
  run("cp.async W=16 NS=6", pipe<16, 6, 0>, 17 * 32, 6);
  run("LDG->STS W=4 NS=4", pipe<4, 4, 1>, 5 * 32, 4);
  run("LDG->STS W=8 NS=4", pipe<8, 4, 1>, 9 * 32, 4);
  run("LDG->STS W=16 NS=4", pipe<16, 4, 1>, 17 * 32, 4);
  run("LDG->STS W=16 NS=6", pipe<16, 6, 1>, 17 * 32, 6);
  run("LDG->STS W=32 NS=4", pipe<32, 4, 1>, 33 * 32, 4);
  run("cp.async W=32 NS=4", pipe<32, 4, 0>, 33 * 32, 4);
  return 0;
}
