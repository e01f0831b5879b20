// Throwaway probe: achievable HBM read bandwidth for the re-rank gather
// pattern (random docs of 1..63 rows x 64 B from an 18 GB table) vs a
// sequential read, with plain LDG.128 (many warps) and with cp.async into smem.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// warp per doc, 16B per lane, unroll U
template <int U>
__global__ void read_docs(const uint4* __restrict__ rows, const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ids,
                          int n, uint32_t* sink) {
  int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    uint32_t id = ids[i];
    uint64_t a = rp[id] * 4, b = rp[id + 1] * 4;  // uint4 units (64B rows)
    for (uint64_t v = a + lane; v < b; v += 32 * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = (v + 32 * u < b) ? __ldcs(rows + v + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void read_seq(const uint4* __restrict__ rows, uint64_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 x = __ldcs(rows + i);
    acc ^= x.x ^ x.y ^ x.z ^ x.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// cp.async gather into a smem ring, per CTA, like the MaxSim copy warps but
// without the MMA: stages of S KB, W warps, waits with cp.async.wait_group.
template <int STAGES>
__global__ void cpasync_docs(const uint4* __restrict__ rows, const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ids,
                             int n, uint32_t* sink) {
  extern __shared__ uint4 sm[];
  const int per_stage = 2048;  // 16B chunks per stage (32 KB)
  int t = threadIdx.x;
  int cnt = 0, stage = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    uint32_t id = ids[i];
    uint64_t a = rp[id] * 4, b = rp[id + 1] * 4;
    for (uint64_t v = a + t; v < b; v += blockDim.x) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + stage * per_stage + (cnt++ % per_stage));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(rows + v));
    }
    if ((i / gridDim.x) % 8 == 7) {
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1));
      stage = (stage + 1) % STAGES;
    }
  }
  asm volatile("cp.async.wait_all;");
  __syncthreads();
  if (sm[t].x == 0x12345678) sink[0] = 1;
}

int main() {
  const uint64_t N = 8800000;
  std::mt19937_64 rng(1);
  std::vector<uint64_t> rp(N + 1, 0);
  for (uint64_t i = 0; i < N; ++i) rp[i + 1] = rp[i] + 1 + rng() % 63;
  const uint64_t T = rp[N];
  printf("tokens %llu (%.1f GB)\n", (unsigned long long)T, T * 64 / 1e9);
  uint4* d_rows; uint64_t* d_rp; uint32_t* d_ids; uint32_t* sink;
  CK(cudaMalloc(&d_rows, T * 64)); CK(cudaMemset(d_rows, 1, T * 64));
  CK(cudaMalloc(&d_rp, (N + 1) * 8)); CK(cudaMemcpy(d_rp, rp.data(), (N + 1) * 8, cudaMemcpyHostToDevice));
  const int nq = 64 * 1000 * 8;  // 8 batches worth of random docs
  std::vector<uint32_t> ids(nq);
  for (auto& x : ids) x = rng() % N;
  uint64_t bytes = 0;
  for (auto x : ids) bytes += (rp[x + 1] - rp[x]) * 64;
  std::vector<uint32_t> sorted_ids = ids;
  std::sort(sorted_ids.begin(), sorted_ids.end());
  CK(cudaMalloc(&d_ids, nq * 4)); CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double b) {
    for (int w = 0; w < 2; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-44s %8.3f ms  %7.0f GB/s\n", name, ms, b / ms / 1e6);
  };
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaMemcpy(d_ids, ids.data(), nq * 4, cudaMemcpyHostToDevice));
  timeit("random docs LDG U=1 (8 warps/blk x 8 blk/SM)", [&] { read_docs<1><<<sms * 8, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("random docs LDG U=2", [&] { read_docs<2><<<sms * 8, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("random docs LDG U=4", [&] { read_docs<4><<<sms * 8, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("random docs LDG U=2 16 blk/SM", [&] { read_docs<2><<<sms * 16, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("random docs LDG U=2 2 blk/SM", [&] { read_docs<2><<<sms * 2, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  CK(cudaFuncSetAttribute(cpasync_docs<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
  CK(cudaFuncSetAttribute(cpasync_docs<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
  timeit("random docs cp.async 4x32KB, 128 thr, 1 CTA/SM", [&] { cpasync_docs<4><<<sms, 128, 4 * 32768>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("random docs cp.async 6x32KB, 256 thr, 1 CTA/SM", [&] { cpasync_docs<6><<<sms, 256, 6 * 32768>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  CK(cudaMemcpy(d_ids, sorted_ids.data(), nq * 4, cudaMemcpyHostToDevice));
  timeit("sorted docs LDG U=2", [&] { read_docs<2><<<sms * 8, 256>>>(d_rows, d_rp, d_ids, nq, sink); }, bytes);
  timeit("sequential read same bytes", [&] { read_seq<<<sms * 8, 256>>>(d_rows, bytes / 16, sink); }, bytes);
  timeit("sequential read 4 GB", [&] { read_seq<<<sms * 8, 256>>>(d_rows, 4ull << 30 >> 4, sink); }, 4.0 * (1ull << 30));
  return 0;
}
