// Throwaway probe: DRAM bytes read per random-document read, to explain the
// MaxSim kernel's and the K1 gather's ~1.10x DRAM over-read on C2.
// 64,000 random docs from a 4 GB region; per variant: doc start alignment
// (64 / 128 / 256 B), doc length (fixed 2048 B or 64 B x U{1..63}), reader
// (LDG warp per doc, or one cp.async.bulk per doc into shared memory) and the
// context's L2 fetch granularity limit.  Run under
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv
// and compare dram bytes with the printed payload bytes.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_read(const uint8_t* __restrict__ base, const uint2* __restrict__ docs, uint32_t n, uint32_t* sink) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint2 d = docs[w];  // byte offset / 16, bytes
  const uint4* p = reinterpret_cast<const uint4*>(base) + d.x;
  uint32_t acc = 0;
  for (uint32_t i = lane; i < d.y / 16; i += 32) {
    const uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc == 0x12345678u) sink[0] = acc;
}

// one CTA of 32 threads, lanes issue one bulk copy per doc into 8 KB slots
__global__ void bulk_read(const uint8_t* __restrict__ base, const uint2* __restrict__ docs, uint32_t n, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  const uint32_t lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t ph = 0;
  for (uint32_t d0 = blockIdx.x * 8; d0 < n; d0 += gridDim.x * 8) {
    uint32_t bytes = 0;
    const uint32_t k = d0 + lane;
    uint2 d = make_uint2(0, 0);
    if (lane < 8 && k < n) d = docs[k];
    bytes = d.y;
    for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    if (lane == 0)
      asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    __syncwarp();
    if (d.y)
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + lane * 4096)), "l"(base + (uint64_t)d.x * 16), "r"(d.y), "r"(su32(&bar)) : "memory");
    asm volatile("{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra LAB_WAIT;}" ::"r"(su32(&bar)), "r"(ph) : "memory");
    ph ^= 1;
  }
  if (lane == 0 && sm[5] == 0x7f && sm[77] == 0x11) sink[0] = 1;
}

int main() {
  const size_t region = 4ull << 30;
  uint8_t* base;
  CK(cudaMalloc(&base, region));
  CK(cudaMemset(base, 1, region));
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4));
  const uint32_t n = 64000;
  uint2* ddocs;
  CK(cudaMalloc(&ddocs, n * sizeof(uint2)));
  uint8_t* flush;
  CK(cudaMalloc(&flush, 512ull << 20));
  CK(cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
  std::mt19937_64 rng(1);
  const int aligns[3] = {64, 128, 256};
  const int grans[3] = {32, 64, 128};
  size_t def = 0;
  CK(cudaDeviceGetLimit(&def, cudaLimitMaxL2FetchGranularity));
  printf("default L2 fetch granularity limit: %zu\n", def);
  int launch = 0;
  for (int gi = 0; gi < 4; ++gi) {
    if (gi < 3) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, grans[gi]));
    else CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, def));
    size_t g = 0;
    CK(cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity));
    for (int lenmode = 0; lenmode < 2; ++lenmode)
      for (int ai = 0; ai < 3; ++ai) {
        std::vector<uint2> docs(n);
        uint64_t payload = 0;
        for (uint32_t i = 0; i < n; ++i) {
          const uint32_t bytes = lenmode == 0 ? 2048u : 64u * (1u + (uint32_t)(rng() % 63));
          const uint64_t off = (rng() % ((region - 8192) / aligns[ai])) * aligns[ai];
          docs[i] = make_uint2((uint32_t)(off / 16), bytes);
          payload += bytes;
        }
        CK(cudaMemcpy(ddocs, docs.data(), n * sizeof(uint2), cudaMemcpyHostToDevice));
        for (int reader = 0; reader < 2; ++reader) {
          CK(cudaMemset(flush, reader, 512ull << 20));  // evict L2
          CK(cudaDeviceSynchronize());
          if (reader == 0) ldg_read<<<(n * 32 + 255) / 256, 256>>>(base, ddocs, n, sink);
          else bulk_read<<<148 * 4, 32, 8 * 4096>>>(base, ddocs, n, sink);
          CK(cudaDeviceSynchronize());
          printf("launch %d: gran_limit %zu len %s align %d reader %s payload %.3f MB\n", launch++, g,
                 lenmode ? "U{1..63}x64" : "2048", aligns[ai], reader ? "bulk" : "ldg", payload / 1e6);
        }
      }
  }
  return 0;
}
