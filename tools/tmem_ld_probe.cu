// Measurement probe (not product): TMEM read throughput of one SM on B200.
// The C2 MaxSim epilogue reads every accumulator column once: per 32 KB
// stage of rows, 128 lanes x 128 columns x 4 B = 64 KB of tcgen05.ld
// (2x the HBM bytes).  This probe times W warps (lane quarter = warp % 4)
// each issuing tcgen05.ld.32x32b.x{32} + wait::ld over a 512-column
// allocation, the same pattern as the epilogue (two loads in flight per
// warp, v[c & 1] ring), and reports bytes per SM clock.  One CTA per SM,
// all 148 SMs, so the figure also covers the whole chip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2312_05417_b200/csrc -o tools/tmem_ld_probe tools/tmem_ld_probe.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int W, int LW>
__global__ void __launch_bounds__(W * 32, 1) tmem_ld_probe(int iters, unsigned long long* cyc, float* sink) {
  using namespace espn_ptx;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = holder;
  const uint32_t q = (uint32_t)(warp & 3), colgrp = (uint32_t)(warp >> 2);  // lane quarter, column group
  const uint32_t ngrp = W / 4;
  float acc = 0.f;
  float v[2][LW];
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // each warp walks its share of the 512 columns, 2 chunks in flight
    const uint32_t cols = 512 / ngrp;
    const uint32_t c0 = colgrp * cols;
    const uint32_t addr = base + (q * 32u << 16) + c0;
    tmem_ld_32x32b<LW>(addr, v[0]);
#pragma unroll 1
    for (uint32_t c = 0; c < cols / LW; c += 2) {
      tmem_ld_wait();
      if (c + 1 < cols / LW) tmem_ld_32x32b<LW>(addr + LW * (c + 1), v[1]);
#pragma unroll
      for (int i = 0; i < LW; ++i) acc = fmaxf(acc, v[0][i]);
      tmem_ld_wait();
      if (c + 2 < cols / LW) tmem_ld_32x32b<LW>(addr + LW * (c + 2), v[0]);
#pragma unroll
      for (int i = 0; i < LW; ++i) acc = fmaxf(acc, v[1][i]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(base);
}

template <int W, int LW>
int run(int sms) {
  unsigned long long* cyc;
  float* sink;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&sink, 4096));
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(cyc, 0, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    // 160 KB of dynamic shared memory: one CTA per SM (each owns all 512 columns)
    CK(cudaFuncSetAttribute(tmem_ld_probe<W, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    tmem_ld_probe<W, LW><<<sms, W * 32, 160 * 1024>>>(iters, cyc, sink);
    CK(cudaGetLastError());
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double bytes_per_cta = (double)iters * 128 * 512 * 4;
    const double cyc_per_cta = (double)c / sms;
    if (rep == 1)
      printf("warps %2d x%d loads: %.1f B/clk/SM, %.2f TB/s chip (%.3f ms), 64 KB (one C2 stage) = %.0f clk\n", W, LW,
             bytes_per_cta / cyc_per_cta, bytes_per_cta * sms / (ms * 1e-3) / 1e12, ms, 65536.0 / (bytes_per_cta / cyc_per_cta));
  }
  cudaFree(cyc);
  cudaFree(sink);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 32>(sms);
  run<8, 32>(sms);
  run<8, 16>(sms);
  run<16, 32>(sms);
  return 0;
}
