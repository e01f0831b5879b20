// Throwaway probe: producer-only throughput of the MaxSim gather (random docs
// of 1..63 rows x 64 B from an 18 GB table into a ring of 32 KB smem stages)
// with the per-stage doc plan already in registers (no metadata latency):
//   mode 0: 1-D cp.async.bulk per doc, L2 evict_first hint
//   mode 1: 1-D cp.async.bulk per doc, no hint
//   mode 2: 2-D tensor TMA, 8-row boxes (reads ceil8(t) rows), L2 promo 256B
//   mode 3: 2-D tensor TMA, boxes of 8/4/2/1 rows (exact rows)
//   mode 4: 1-D cp.async.bulk per doc + prefetch.global.L2 of the doc first
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra LAB_WAIT;}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_hint(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tile2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int col, int row) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"(map), "r"(col), "r"(row), "r"(su32(bar)) : "memory");
}

struct Maps { CUtensorMap m8, m4, m2, m1; };

// docs: (row0, t, slot-in-stage) per doc; stage_doc0[s] = first doc of stage s (global)
template <int MODE, int NS, int W>
__global__ void __launch_bounds__((W + 1) * 32, 1)
prod(const __grid_constant__ Maps maps, const uint8_t* __restrict__ rows, const uint4* __restrict__ docs,
     const uint32_t* __restrict__ stage_doc0, uint32_t stages_per_cta, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], MODE == 5 ? W * 32 : W); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t st0 = blockIdx.x * stages_per_cta;
  if (warp < W) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    // software-pipelined metadata: docs of stage st+1 loaded while st issues
    uint32_t d0 = stage_doc0[st0], d1 = stage_doc0[st0 + 1];
    const uint32_t me = warp * 32 + lane;
    uint4 cur = (d0 + me < d1) ? docs[d0 + me] : make_uint4(0, 0, 0, 0);
    uint4 cur2 = (W == 1 && d0 + me + 32 < d1) ? docs[d0 + me + 32] : make_uint4(0, 0, 0, 0);
    for (uint32_t st = 0; st < stages_per_cta; ++st) {
      const uint32_t n0 = stage_doc0[st0 + st + 1], n1 = stage_doc0[st0 + st + 2];
      const uint4 nxt = (n0 + me < n1) ? docs[n0 + me] : make_uint4(0, 0, 0, 0);
      const uint4 nxt2 = (W == 1 && n0 + me + 32 < n1) ? docs[n0 + me + 32] : make_uint4(0, 0, 0, 0);
      const uint32_t s = st % NS;
      // bytes this stage
      uint32_t bytes = 0;
      auto nb = [&](uint4 d) -> uint32_t {
        if (!d.y) return 0u;
        if (MODE == 2) return ((d.y + 7) / 8) * 512u;
        return d.y * 64u;
      };
      bytes = nb(cur) + nb(cur2);
      for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      if (MODE == 5) {
        const uint32_t sbase5 = su32(sm + s * 32768);
        // docs of this warp: lanes hold (row0, t, slot); copy each doc cooperatively
        for (int h2 = 0; h2 < 2; ++h2) {
          const uint4 dd = h2 ? cur2 : cur;
          const uint32_t act = __ballot_sync(0xffffffffu, dd.y != 0);
          for (uint32_t m = act; m; m &= m - 1) {
            const int src_l = __ffs(m) - 1;
            const uint32_t r0 = __shfl_sync(0xffffffffu, dd.x, src_l), t = __shfl_sync(0xffffffffu, dd.y, src_l),
                           sl = __shfl_sync(0xffffffffu, dd.z, src_l);
            const uint8_t* src = rows + (size_t)r0 * 64;
            const uint32_t dst = sbase5 + sl * 64;
            for (uint32_t c = lane; c < t * 4; c += 32)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 16), "l"(src + c * 16) : "memory");
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
        cur = nxt; cur2 = nxt2;
        continue;
      }
      if (lane == 0) mbar_arrive_tx(&full[s], bytes);
      __syncwarp();
      const uint32_t sbase = su32(sm + s * 32768);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 d = h ? cur2 : cur;
        if (!d.y) continue;
        const uint32_t dst = sbase + d.z * 64;
        if (MODE == 0) bulk_hint(dst, rows + (size_t)d.x * 64, d.y * 64, &full[s], pol);
        else if (MODE == 1) bulk(dst, rows + (size_t)d.x * 64, d.y * 64, &full[s]);
        else if (MODE == 4) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rows + (size_t)d.x * 64));
          bulk(dst, rows + (size_t)d.x * 64, d.y * 64, &full[s]);
        } else if (MODE == 2) {
          for (uint32_t g = 0; g < (d.y + 7) / 8; ++g) tile2d(dst + g * 512, &maps.m8, &full[s], 0, d.x + 8 * g);
        } else {
          uint32_t r = 0;
          for (; r + 8 <= d.y; r += 8) tile2d(dst + r * 64, &maps.m8, &full[s], 0, d.x + r);
          if (d.y - r >= 4) { tile2d(dst + r * 64, &maps.m4, &full[s], 0, d.x + r); r += 4; }
          if (d.y - r >= 2) { tile2d(dst + r * 64, &maps.m2, &full[s], 0, d.x + r); r += 2; }
          if (d.y - r >= 1) { tile2d(dst + r * 64, &maps.m1, &full[s], 0, d.x + r); r += 1; }
        }
      }
      cur = nxt; cur2 = nxt2;
    }
  } else if (warp == W && lane == 0) {
    uint32_t acc = 0;
    for (uint32_t st = 0; st < stages_per_cta; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&full[s], (st / NS) & 1);
      acc ^= *reinterpret_cast<uint32_t*>(sm + s * 32768 + (st & 1023) * 4);
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  const uint64_t N = 8800000;
  std::mt19937_64 rng(1);
  std::vector<uint64_t> rp(N + 1, 0);
  for (uint64_t i = 0; i < N; ++i) rp[i + 1] = rp[i] + 1 + rng() % 63;
  const uint64_t T = rp[N];
  uint8_t* d_rows;
  CK(cudaMalloc(&d_rows, T * 64));
  CK(cudaMemset(d_rows, 1, T * 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // plan: random docs packed into stages of 512 8-aligned slots
  std::vector<uint4> docs;
  std::vector<uint32_t> sd0;
  uint32_t slot = 0;
  double bytes = 0;
  sd0.push_back(0);
  const uint32_t n_stages = sms * 40;
  while (sd0.size() <= n_stages + 2) {
    uint64_t id = rng() % N;
    uint32_t t = (uint32_t)(rp[id + 1] - rp[id]);
    uint32_t pad = (t + 7) & ~7u;
    if (slot + pad > 512) { sd0.push_back((uint32_t)docs.size()); slot = 0; }
    docs.push_back(make_uint4((uint32_t)rp[id], t, slot, 0));
    slot += pad;
    if (sd0.size() <= n_stages) bytes += t * 64.0;
  }
  uint4* d_docs; uint32_t* d_sd0; uint32_t* sink;
  CK(cudaMalloc(&d_docs, docs.size() * 16)); CK(cudaMemcpy(d_docs, docs.data(), docs.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_sd0, sd0.size() * 4)); CK(cudaMemcpy(d_sd0, sd0.data(), sd0.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&sink, 4));
  Maps maps;
  CUtensorMap* mm[4] = {&maps.m8, &maps.m4, &maps.m2, &maps.m1};
  int br[4] = {8, 4, 2, 1};
  for (int i = 0; i < 4; ++i) {
    cuuint64_t gdim[2] = {32, T}, gstride[1] = {64};
    cuuint32_t box[2] = {32, (cuuint32_t)br[i]}, estr[2] = {1, 1};
    CUresult r = encode(mm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d_rows, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d failed %d\n", i, r); return 1; }
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int ns, int W) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768));
    const uint32_t spc = n_stages / sms;
    for (int w = 0; w < 2; ++w) kern<<<sms, 32 * (W + 1), ns * 32768>>>(maps, d_rows, d_docs, d_sd0, spc, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<sms, 32 * (W + 1), ns * 32768>>>(maps, d_rows, d_docs, d_sd0, spc, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-34s NS=%d W=%d %7.3f ms  useful %6.0f GB/s\n", name, ns, W, ms, bytes / ms / 1e6);
  };
  run("bulk1d evict_first", prod<0, 4, 2>, 4, 2);
  run("cp.async per doc", prod<5, 4, 1>, 4, 1);
  run("cp.async per doc", prod<5, 4, 2>, 4, 2);
  run("cp.async per doc", prod<5, 4, 4>, 4, 4);
  run("cp.async per doc", prod<5, 6, 4>, 6, 4);
  return 0;
}
