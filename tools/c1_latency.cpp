// Batch-1 latency through the native C-ABI (configs[0]: 100k docs, t <= 32,
// d=32 fp16, 32 query tokens, top-1000 -> top-10), host buffers, synchronous
// espn_gpu_rerank calls -- what a C++ serving loop sees per query, without the
// Python layer the bench's e2e figure includes.
//   g++ -O2 -std=c++17 -I include tools/c1_latency.cpp -L paper_2312_05417_b200/lib -lespn_gpu \
//       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2312_05417_b200/lib -o /tmp/c1_latency
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "espn_gpu.h"

#define CK(x)                                                              \
  do {                                                                     \
    int rc_ = (x);                                                         \
    if (rc_) {                                                             \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, rc_, espn_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

// argv[1]: espn_kernel (0 auto, 1 tcgen05, 2 simt, 3 small)
int main(int argc, char** argv) {
  const uint32_t kern = argc > 1 ? (uint32_t)atoi(argv[1]) : ESPN_KERNEL_AUTO;
  const uint64_t N = 100000;
  const uint32_t d = 32, nq = 32, K = 1000, k = 10, reps = 3000;
  uint64_t* rp = nullptr;
  uint16_t* rows = nullptr;
  cudaMalloc(&rp, (N + 1) * sizeof(uint64_t));
  CK(espn_gpu_synth_table(N, d, ESPN_DTYPE_F16, 1, 32, 42, 1, 0, rp, nullptr, nullptr));
  uint64_t ntok = 0;
  cudaMemcpy(&ntok, rp + N, sizeof ntok, cudaMemcpyDeviceToHost);
  cudaMalloc(&rows, ntok * d * sizeof(uint16_t));
  CK(espn_gpu_synth_table(N, d, ESPN_DTYPE_F16, 1, 32, 42, 1, 0, rp, rows, nullptr));
  espn_table_desc td{};
  td.n_docs = N;
  td.d = d;
  td.dtype = ESPN_DTYPE_F16;
  td.d_cls = 128;
  td.value_width = 2;
  td.alignment = 4096;
  td.flags = ESPN_TABLE_DEVICE_BORROWED | ESPN_TABLE_ROWS_TILED;
  td.row_ptr = rp;
  td.rows = rows;
  espn_gpu_table* t = nullptr;
  CK(espn_gpu_table_open(&td, &t));
  espn_workspace_desc wd{};
  wd.max_queries = 1;
  wd.max_candidates = K;
  wd.max_query_tokens = nq;
  espn_gpu_workspace* w = nullptr;
  CK(espn_gpu_workspace_create(t, &wd, &w));

  std::mt19937_64 rng(7);
  std::normal_distribution<float> nd(0.f, 1.f);
  const int NB = 16;  // distinct queries rotate
  std::vector<std::vector<float>> q(NB, std::vector<float>(nq * d));
  std::vector<std::vector<uint32_t>> ids(NB, std::vector<uint32_t>(K));
  std::vector<std::vector<float>> cls(NB, std::vector<float>(K));
  for (int b = 0; b < NB; ++b) {
    for (auto& x : q[b]) x = nd(rng) * 0.17f;
    std::vector<uint32_t> all(N);
    for (uint32_t i = 0; i < N; ++i) all[i] = i;
    std::shuffle(all.begin(), all.end(), rng);
    for (uint32_t j = 0; j < K; ++j) {
      ids[b][j] = all[j];
      cls[b][j] = 1.0f - j * 1e-4f;  // sorted descending, distinct
    }
  }
  uint64_t off[2] = {0, K};
  uint32_t out_ids[k], out_n[1];
  float out_sc[k];
  std::vector<double> lat;
  for (uint32_t r = 0; r < reps + 50; ++r) {
    const int b = r % NB;
    espn_rerank_args a{};
    a.n_queries = 1;
    a.n_query_tokens = nq;
    a.query_tokens = q[b].data();
    a.cand_ids = ids[b].data();
    a.cand_cls = cls[b].data();
    a.cand_offsets = off;
    a.rerank_count = K;
    a.final_k = k;
    a.alpha = 1.0f;
    a.kernel = kern;
    espn_rerank_out o{};
    o.ids = out_ids;
    o.scores = out_sc;
    o.counts = out_n;
    const auto t0 = std::chrono::steady_clock::now();
    CK(espn_gpu_rerank(t, w, &a, &o, nullptr));
    const auto t1 = std::chrono::steady_clock::now();
    if (r >= 50) lat.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(lat.begin(), lat.end());
  double sum = 0;
  for (double x : lat) sum += x;
  std::printf("{\"config\": \"configs[0] batch 1, host buffers, synchronous C-ABI calls\", \"kernel\": %u, \"calls\": %zu, "
              "\"mean_us\": %.2f, \"p50_us\": %.2f, \"p99_us\": %.2f, \"queries_per_s\": %.0f}\n",
              kern, lat.size(), sum / lat.size(), lat[lat.size() / 2], lat[lat.size() * 99 / 100], lat.size() / (sum * 1e-6));
  espn_gpu_workspace_destroy(w);
  espn_gpu_table_close(t);
  cudaFree(rows);
  cudaFree(rp);
  return 0;
}
