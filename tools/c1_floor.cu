// Throwaway probe: the fixed cost floor of a synchronous batch-1 call
// (configs[0]) on this box, to size the single-launch small-batch path:
//   A  empty kernel + cudaStreamSynchronize
//   B  H2D 12 KB (pinned) + 1 empty kernel + D2H 128 B + sync, as a CUDA graph
//   C  same with 3 dependent empty kernels (plan -> MaxSim -> finalize shape)
//   D  H2D 12 KB + 1 kernel writing its outputs to mapped pinned memory, host
//      spins on a flag the kernel writes last (no D2H, no stream sync)
//   E  D with the kernel launch only (inputs already on the device)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <chrono>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_empty(const uint32_t* in, uint32_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && in) out[0] = in[0] + 1;
}
__global__ void k_flag(const uint32_t* in, uint32_t* out_h, volatile uint32_t* flag_h, uint32_t seq) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out_h[0] = in[0] + seq;
    __threadfence_system();
    *flag_h = seq;
  }
}

template <class F>
void timeit(const char* name, F f, int n = 3000) {
  for (int i = 0; i < 200; ++i) f(i);
  std::vector<double> v(n);
  for (int i = 0; i < n; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    f(i);
    auto t1 = std::chrono::steady_clock::now();
    v[i] = std::chrono::duration<double, std::micro>(t1 - t0).count();
  }
  std::sort(v.begin(), v.end());
  double m = 0;
  for (double x : v) m += x;
  printf("%-60s mean %6.1f us  p50 %6.1f  p99 %6.1f\n", name, m / n, v[n / 2], v[n * 99 / 100]);
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t inb = 12 * 1024, outb = 128;
  uint8_t *in_h, *out_h, *in_d, *out_d;
  CK(cudaHostAlloc(&in_h, inb, cudaHostAllocDefault));
  CK(cudaHostAlloc(&out_h, 4096, cudaHostAllocMapped));
  CK(cudaMalloc(&in_d, inb));
  CK(cudaMalloc(&out_d, 4096));
  uint32_t* flag_h;
  CK(cudaHostAlloc(&flag_h, 64, cudaHostAllocMapped));
  uint32_t *flag_d, *outm_d;
  CK(cudaHostGetDevicePointer((void**)&flag_d, flag_h, 0));
  CK(cudaHostGetDevicePointer((void**)&outm_d, out_h, 0));
  *flag_h = 0;
  std::vector<uint8_t> user(inb, 1), user_out(outb);

  timeit("A empty kernel + sync", [&](int) {
    k_empty<<<1, 32, 0, s>>>(nullptr, (uint32_t*)out_d);
    CK(cudaStreamSynchronize(s));
  });
  for (int nk : {1, 3}) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    CK(cudaMemcpyAsync(in_d, in_h, inb, cudaMemcpyHostToDevice, s));
    for (int i = 0; i < nk; ++i) k_empty<<<148, 128, 0, s>>>((const uint32_t*)in_d, (uint32_t*)out_d);
    CK(cudaMemcpyAsync(out_h, out_d, outb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    char name[128];
    snprintf(name, sizeof name, "%c graph: memcpy in, H2D 12KB, %d kernel(s), D2H 128B, sync, memcpy out", nk == 1 ? 'B' : 'C', nk);
    timeit(name, [&](int) {
      memcpy(in_h, user.data(), inb);
      CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      memcpy(user_out.data(), out_h, outb);
    });
    snprintf(name, sizeof name, "%c' same, eager (no graph)", nk == 1 ? 'B' : 'C');
    timeit(name, [&](int) {
      memcpy(in_h, user.data(), inb);
      CK(cudaMemcpyAsync(in_d, in_h, inb, cudaMemcpyHostToDevice, s));
      for (int i = 0; i < nk; ++i) k_empty<<<148, 128, 0, s>>>((const uint32_t*)in_d, (uint32_t*)out_d);
      CK(cudaMemcpyAsync(out_h, out_d, outb, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      memcpy(user_out.data(), out_h, outb);
    });
  }
  uint32_t seq = 0;
  timeit("D H2D 12KB + kernel -> mapped outputs, host spins on flag", [&](int) {
    ++seq;
    memcpy(in_h, user.data(), inb);
    CK(cudaMemcpyAsync(in_d, in_h, inb, cudaMemcpyHostToDevice, s));
    k_flag<<<148, 128, 0, s>>>((const uint32_t*)in_d, outm_d, flag_d, seq);
    while (*(volatile uint32_t*)flag_h != seq) {}
    memcpy(user_out.data(), out_h, outb);
  });
  timeit("E kernel -> mapped outputs, host spins on flag", [&](int) {
    ++seq;
    k_flag<<<148, 128, 0, s>>>((const uint32_t*)in_d, outm_d, flag_d, seq);
    while (*(volatile uint32_t*)flag_h != seq) {}
  });
  CK(cudaStreamSynchronize(s));
  return 0;
}
