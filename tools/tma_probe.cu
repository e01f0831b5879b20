// Throwaway probe: TMA tile::gather4 (4 arbitrary table rows per instruction,
// SWIZZLE_64B) as the MaxSim B-operand producer.
// (1) correctness: gather 128 random rows into a SW64 K-major tile, run one
//     tcgen05.mma against a 128x32 A (interleaved layout), compare with CPU.
// (2) throughput: ring of NS x 32 KB stages filled by W issuing warps with
//     gather4 + mbarrier complete_tx, consumer warp releases.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_fp16.h>
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
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int col, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(dst), "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// ---------------- (1) correctness ----------------
__global__ void check_kernel(const __grid_constant__ CUtensorMap map, const int* rowsel, const __half* A /*128x32*/, float* out /*128x128*/) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm;            // 128 rows x 64 B, SW64 (1024-aligned)
  uint8_t* sA = sm + 8192;     // 128 rows x 32 K interleaved
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tm;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 4; i += blockDim.x) {
    int r = i / 4, c = i % 4;
    *reinterpret_cast<uint4*>(sA + (r / 8) * 512 + c * 128 + (r % 8) * 16) = *reinterpret_cast<const uint4*>(A + r * 32 + c * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (tid == 0) { mbar_init(&bar, 1); mbar_init(&mbar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    mbar_arrive_tx(&bar, 128 * 64);
    for (int g = 0; g < 32; ++g)
      gather4(su32(sB + g * 256), &map, &bar, 0, rowsel[4 * g], rowsel[4 * g + 1], rowsel[4 * g + 2], rowsel[4 * g + 3]);
  }
  mbar_wait(&bar, 0);
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int ks = 0; ks < 2; ++ks) {
      uint64_t ad = desc(su32(sA) + ks * 256, 128, 512, 0);
      uint64_t bd = desc(su32(sB) + ks * 32, 16, 512, 4);  // SWIZZLE_64B, K-major
      asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                   :: "r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
  }
  mbar_wait(&mbar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) out[(warp * 32 + tid % 32) * 128 + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tm));
}

// ---------------- (2) throughput ----------------
template <int W, int NS>
__global__ void __launch_bounds__((W + 1) * 32, 1)
pipe_tma(const __grid_constant__ CUtensorMap map, const uint2* __restrict__ grp, uint64_t n_groups_total, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], W); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint64_t per_cta = n_groups_total / gridDim.x;
  const uint64_t g_begin = blockIdx.x * per_cta;
  const uint32_t n_st = (uint32_t)(per_cta / 64);
  if (warp < W) {
    for (uint32_t st = 0; st < n_st; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      const uint32_t sbase = su32(sm + s * 32768);
      const uint2* g = grp + g_begin + (uint64_t)st * 64;
      // 128 gather4 ops per stage (512 slots); warp w takes ops w, w+W, ... one per lane
      constexpr int OPS = 128 / W;
      if (lane == 0) mbar_arrive_tx(&full[s], OPS * 256);
      __syncwarp();
      for (int o = lane; o < OPS; o += 32) {
        const int op = warp + o * W;  // 4 slots: op*4 .. +3 -> group op/2, half op%2
        const uint2 gr = g[op >> 1];
        const int b = (op & 1) * 4;
        const int r0 = min(gr.x + b, gr.y), r1 = min(gr.x + b + 1, gr.y), r2 = min(gr.x + b + 2, gr.y), r3 = min(gr.x + b + 3, gr.y);
        gather4(sbase + op * 256, &map, &full[s], 0, r0, r1, r2, r3);
      }
    }
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


// cp.async.bulk (1-D) per doc: docs listed as (row0, t); a stage takes docs
// until 512 rows; W warps, one op per lane.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
template <int W, int NS>
__global__ void __launch_bounds__((W + 1) * 32, 1)
pipe_bulk(const uint4* __restrict__ rows, const uint2* __restrict__ docs /*(r0, slot0) per doc*/, const uint32_t* __restrict__ stage_doc0,
          uint32_t n_stages_total, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], W); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t per_cta = n_stages_total / gridDim.x;
  const uint32_t st0 = blockIdx.x * per_cta;
  if (warp < W) {
    for (uint32_t st = 0; st < per_cta; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      const uint32_t sbase = su32(sm + s * 32768);
      const uint32_t d0 = stage_doc0[st0 + st], d1 = stage_doc0[st0 + st + 1];
      // bytes this warp will issue
      uint32_t my = 0;
      for (uint32_t d = d0 + warp * 32 + lane; d < d1; d += W * 32) {
        const uint2 a = docs[d], b = docs[d + 1];
        my += (b.y - a.y) * 64;
      }
      for (int o = 16; o; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
      if (lane == 0) mbar_arrive_tx(&full[s], my);
      __syncwarp();
      const uint32_t slot_base = docs[d0].y;
      for (uint32_t d = d0 + warp * 32 + lane; d < d1; d += W * 32) {
        const uint2 a = docs[d], b = docs[d + 1];
        bulk_g2s(sbase + (a.y - slot_base) * 64, rows + (size_t)a.x * 4, (b.y - a.y) * 64, &full[s]);
      }
    }
  } else if (lane == 0) {
    uint32_t acc = 0;
    for (uint32_t st = 0; st < per_cta; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&full[s], (st / NS) & 1);
      acc ^= *reinterpret_cast<uint32_t*>(sm + s * 32768 + (st & 1023) * 4);
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}


__device__ __forceinline__ void tile2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int col, int row) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"(map), "r"(col), "r"(row), "r"(su32(bar)) : "memory");
}
// tiled boxes of BR rows (BR multiple of 8): each op loads BR consecutive rows starting at a group's first row
template <int W, int NS, int BR>
__global__ void __launch_bounds__((W + 1) * 32, 1)
pipe_tile(const __grid_constant__ CUtensorMap map, const uint2* __restrict__ grp, uint64_t n_groups_total, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], W); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint64_t per_cta = n_groups_total / gridDim.x;
  const uint64_t g_begin = blockIdx.x * per_cta;
  const uint32_t n_st = (uint32_t)(per_cta / 64);
  constexpr int OPS = 512 / BR / W;
  if (warp < W) {
    for (uint32_t st = 0; st < n_st; ++st) {
      const uint32_t s = st % NS;
      mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
      const uint32_t sbase = su32(sm + s * 32768);
      const uint2* g = grp + g_begin + (uint64_t)st * 64;
      if (lane == 0) mbar_arrive_tx(&full[s], OPS * BR * 64);
      __syncwarp();
      for (int o = lane; o < OPS; o += 32) {
        const int op = warp + o * W;
        const uint2 gr = g[op * (BR / 8)];
        tile2d(sbase + op * BR * 64, &map, &full[s], 0, (int)gr.x);
      }
    }
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
  __half* d_rows;
  CK(cudaMalloc(&d_rows, T * 64));
  // fill: small random values via a host chunk copied repeatedly (checked region explicitly)
  {
    std::vector<__half> chunk(1 << 22);
    for (auto& h : chunk) h = __float2half((int)(rng() % 2001 - 1000) / 1000.f);
    for (uint64_t off = 0; off < T * 32; off += chunk.size())
      CK(cudaMemcpy(d_rows + off, chunk.data(), std::min<uint64_t>(chunk.size(), T * 32 - off) * 2, cudaMemcpyHostToDevice));
  }
  for (int box_rows : {1}) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {32, T}, gstride[1] = {64};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows}, estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d_rows, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box {32,%d}: %d\n", box_rows, (int)r);
    if (r != CUDA_SUCCESS) continue;
    // correctness
    std::vector<int> sel(128);
    for (auto& s : sel) s = (int)(rng() % T);
    sel[5] = sel[4];
    std::vector<__half> hA(128 * 32), hB(128 * 32);
    for (auto& h : hA) h = __float2half((int)(rng() % 2001 - 1000) / 1000.f);
    for (int i = 0; i < 128; ++i) CK(cudaMemcpy(hB.data() + i * 32, d_rows + (uint64_t)sel[i] * 32, 64, cudaMemcpyDeviceToHost));
    int* d_sel; __half* dA; float* dO;
    CK(cudaMalloc(&d_sel, 512)); CK(cudaMalloc(&dA, 8192)); CK(cudaMalloc(&dO, 128 * 128 * 4));
    CK(cudaMemcpy(d_sel, sel.data(), 512, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dA, hA.data(), 8192, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    check_kernel<<<1, 128, 16384>>>(map, d_sel, dA, dO);
    cudaError_t ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) { printf("check kernel failed: %s\n", cudaGetErrorString(ce)); return 1; }
    std::vector<float> o(128 * 128);
    CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int k = 0; k < 32; ++k) ref += (double)__half2float(hA[m * 32 + k]) * __half2float(hB[n * 32 + k]);
        maxerr = std::max(maxerr, std::fabs(ref - o[m * 128 + n]));
      }
    printf("  gather4+SW64 UMMA max abs err %g %s\n", maxerr, maxerr < 1e-3 ? "PASS" : "FAIL");
    // throughput
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
    double doc_bytes = bytes * (double)ng / grp.size();
    uint2* d_grp; uint32_t* sink;
    CK(cudaMalloc(&d_grp, ng * 8)); CK(cudaMemcpy(d_grp, grp.data(), ng * 8, cudaMemcpyHostToDevice)); CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, int threads, int ns) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768));
      for (int w = 0; w < 2; ++w) kern<<<sms, threads, ns * 32768>>>(map, d_grp, ng, sink);
      cudaError_t ce = cudaDeviceSynchronize();
      if (ce != cudaSuccess) { printf("%s failed: %s\n", name, cudaGetErrorString(ce)); exit(1); }
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) kern<<<sms, threads, ns * 32768>>>(map, d_grp, ng, sink);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      printf("  %-30s %7.3f ms  unique-row %6.0f GB/s\n", name, ms, doc_bytes / ms / 1e6);
    };
    run("gather4 W=1 NS=4", pipe_tma<1, 4>, 64, 4);
    run("gather4 W=2 NS=4", pipe_tma<2, 4>, 96, 4);
    run("gather4 W=4 NS=4", pipe_tma<4, 4>, 160, 4);
    run("gather4 W=4 NS=6", pipe_tma<4, 6>, 160, 6);
    run("gather4 W=8 NS=6", pipe_tma<8, 6>, 288, 6);
    run("gather4 W=16 NS=6", pipe_tma<16, 6>, 544, 6);
    run("gather4 W=32 NS=6", pipe_tma<32, 6>, 1056, 6);
    for (int br : {8, 32}) {
      CUtensorMap m2;
      cuuint64_t gdim[2] = {32, T}, gstride[1] = {64};
      cuuint32_t box[2] = {32, (cuuint32_t)br}, estr[2] = {1, 1};
      CUresult r2 = encode(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d_rows, gdim, gstride, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r2) { printf("encode br %d failed %d\n", br, (int)r2); continue; }
      auto runt = [&](const char* name, auto kern, int threads, int ns) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768));
        for (int w = 0; w < 2; ++w) kern<<<sms, threads, ns * 32768>>>(m2, d_grp, ng, sink);
        cudaError_t ce = cudaDeviceSynchronize();
        if (ce != cudaSuccess) { printf("%s failed: %s\n", name, cudaGetErrorString(ce)); exit(1); }
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) kern<<<sms, threads, ns * 32768>>>(m2, d_grp, ng, sink);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("  %-30s %7.3f ms  loaded %6.0f GB/s\n", name, ms, ng * 512.0 / ms / 1e6);
      };
      if (br == 8) { runt("tile8 W=2 NS=6", pipe_tile<2, 6, 8>, 96, 6); runt("tile8 W=4 NS=6", pipe_tile<4, 6, 8>, 160, 6); runt("tile8 W=8 NS=6", pipe_tile<8, 6, 8>, 288, 6); }
      else { runt("tile32 W=1 NS=6", pipe_tile<1, 6, 32>, 64, 6); runt("tile32 W=2 NS=6", pipe_tile<2, 6, 32>, 96, 6); runt("tile32 W=4 NS=6", pipe_tile<4, 6, 32>, 160, 6); }
    }
    {
      // bulk per doc: docs packed contiguously (no 8-alignment) into 512-row stages
      std::vector<uint2> docs; std::vector<uint32_t> sd0;
      uint32_t slot = 0, stage_start = 0; uint64_t b2 = 0;
      sd0.push_back(0);
      for (int i = 0; i < 512000; ++i) {
        uint64_t id = rng() % N;
        uint32_t r0 = (uint32_t)rp[id], t = (uint32_t)(rp[id + 1] - rp[id]);
        if (slot + t - stage_start > 512) { stage_start = slot; sd0.push_back((uint32_t)docs.size()); }
        docs.push_back(make_uint2(r0, slot)); slot += t; b2 += t * 64ull;
      }
      docs.push_back(make_uint2(0, slot));
      uint32_t nst = (uint32_t)((sd0.size() - 1) / sms * sms);
      double bb = 0; for (uint32_t d = 0; d < sd0[nst]; ++d) bb += (docs[d + 1].y - docs[d].y) * 64.0;
      uint2* d_docs; uint32_t* d_sd0;
      CK(cudaMalloc(&d_docs, docs.size() * 8)); CK(cudaMemcpy(d_docs, docs.data(), docs.size() * 8, cudaMemcpyHostToDevice));
      CK(cudaMalloc(&d_sd0, sd0.size() * 4)); CK(cudaMemcpy(d_sd0, sd0.data(), sd0.size() * 4, cudaMemcpyHostToDevice));
      auto runb = [&](const char* name, auto kern, int threads, int ns) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768));
        for (int w = 0; w < 2; ++w) kern<<<sms, threads, ns * 32768>>>((const uint4*)d_rows, d_docs, d_sd0, nst, sink);
        cudaError_t ce = cudaDeviceSynchronize();
        if (ce != cudaSuccess) { printf("%s failed: %s\n", name, cudaGetErrorString(ce)); exit(1); }
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) kern<<<sms, threads, ns * 32768>>>((const uint4*)d_rows, d_docs, d_sd0, nst, sink);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("  %-30s %7.3f ms  unique-row %6.0f GB/s\n", name, ms, bb / ms / 1e6);
      };
      runb("bulk/doc W=2 NS=6", pipe_bulk<2, 6>, 96, 6);
      cudaFree(d_docs); cudaFree(d_sd0);
    }
    cudaFree(d_grp); cudaFree(sink); cudaFree(d_sel); cudaFree(dA); cudaFree(dO);
  }
  return 0;
}
