// kernels_misc.cuh -- the non-tensor-core kernels of the re-rank path:
//   maxsim_simt_kernel  CUDA-core MaxSim (K2 variant for tiny/odd dims), bit-exact
//                       with the SPEC-order oracle (scoring.hpp:7-10, 20-21)
//   topk_kernel         K3/K4: aggregate (scoring.hpp:12-14) + top-k by
//                       (score desc, doc_id asc) (scoring.hpp:16-18) with the
//                       duplicate / non-finite rejections of rank()
//   gather_*            K1: StoreHandle::fetch_batch (store.hpp:91-94) as a
//                       coalesced 16-byte row copy into request-order CSR
//   synth_*             synthetic MS-MARCO-shaped table
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace espn_k {

// ============================================================================
// CUDA-core MaxSim.  One warp per (query, candidate) pair range; lane i owns
// query token i (kept in registers, already rounded to the table dtype), doc
// rows are read once with broadcast 16-byte loads.  Products and sums use
// __fmul_rn/__fadd_rn in ascending index order, so with identical decoded
// inputs the result equals the oracle bit for bit.
// ============================================================================
template <int D>
__global__ void __launch_bounds__(256)
maxsim_simt_kernel(const MaxSimParams p, uint32_t pairs_per_warp, uint64_t n_pairs_total) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint64_t pr = gw * pairs_per_warp;
  const uint64_t pr_end = min(pr + pairs_per_warp, n_pairs_total);
  if (pr >= pr_end) return;
  // pairs are enumerated over needed candidates only: query b contributes
  // min(R, n_b) pairs; unit_off carries the per-query pair prefix here.
  uint32_t lo = 0, hi = p.n_queries;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.unit_off[mid] <= pr) lo = mid; else hi = mid;
  }
  uint32_t b = lo;
  float q[D];
  int cur_b = -1;
  for (; pr < pr_end; ++pr) {
    while (pr >= p.unit_off[b + 1]) ++b;
    if ((int)b != cur_b) {
      cur_b = (int)b;
      const float* qs = p.q32 + ((size_t)b * p.nq + (lane < p.nq ? lane : 0)) * D;
      bool bad = false;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float x = espn_ptx::code_to_f32(espn_ptx::f32_to_code(__ldg(&qs[k]), p.bf16), p.bf16);
        bad |= !isfinite(x);
        q[k] = x;
      }
      if (bad && lane < p.nq) atomicOr(p.err, ERR_NONFINITE_QUERY);
    }
    const uint64_t c = p.cand_off[b] + (pr - p.unit_off[b]);
    const uint64_t loc = shard_local(__ldg(&p.cand_ids[c]), p.shard_count, p.shard_index, p.n_docs);
    if (loc == ~0ull) {
      if (lane == 0) atomicOr(p.err, ERR_UNKNOWN_DOC);
      continue;
    }
    const uint64_t r0 = __ldg(&p.row_ptr[loc]);
    const uint32_t t = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
    const uint8_t* doc = reinterpret_cast<const uint8_t*>(p.rows + r0 * D);
    float m = -INFINITY;
    for (uint32_t j = 0; j < t; ++j) {
      float acc = 0.0f;
#pragma unroll
      for (int k8 = 0; k8 < D / 8; ++k8) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(doc + RowLayout<D>::off(t, j, k8)));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float d0 = espn_ptx::code_to_f32((uint16_t)(w[h] & 0xFFFFu), p.bf16);
          const float d1 = espn_ptx::code_to_f32((uint16_t)(w[h] >> 16), p.bf16);
          acc = __fadd_rn(acc, __fmul_rn(q[k8 * 8 + 2 * h], d0));
          acc = __fadd_rn(acc, __fmul_rn(q[k8 * 8 + 2 * h + 1], d1));
        }
      }
      if (acc > m) m = acc;
    }
    float s = 0.0f;
    for (uint32_t i = 0; i < p.nq; ++i) s = __fadd_rn(s, __shfl_sync(0xffffffffu, m, i));
    if (lane == 0) p.bow_out[c] = s;
  }
}

// ============================================================================
// Top-k: one CTA per query.  Scores become 64-bit keys
//   key = orderable(score) << 32 | ~doc_id
// so "larger key first" is exactly (score desc, doc_id asc); a shared-memory
// bitonic sort over chunks keeps the running best k.
// ============================================================================
constexpr int kTopkThreads = 512;
constexpr int kTopkSort = 4096;      // keys per sort pass (32 KB)
constexpr int kTopkHash = 8192;      // duplicate-detection hash slots
constexpr int kMaxK = 1024;

__device__ __forceinline__ uint32_t float_order(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // canonical +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_float(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ uint64_t make_key(float s, uint32_t id) {
  return ((uint64_t)float_order(s) << 32) | (uint64_t)(~id);
}

// Descending bitonic sort of keys[0..n) (n power of two) by the whole block.
__device__ void bitonic_sort_desc(uint64_t* keys, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = keys[i], b = keys[ixj];
          const bool desc_block = (i & k) == 0;
          if (desc_block ? (a < b) : (a > b)) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// keys chunk producer: fills keys[0..cnt) for chunk [c0, c0+cnt) of query b.
template <typename KeyFn>
__device__ void topk_select(uint64_t* keys, uint64_t* best, int k, uint64_t n, KeyFn key_of,
                            int* best_n_out) {
  int best_n = 0;
  const int chunk = kTopkSort - k;
  for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
    const int cnt = (int)min((uint64_t)chunk, n - c0);
    int tot = cnt + best_n;
    int pw2 = 1;
    while (pw2 < tot) pw2 <<= 1;
    for (int i = threadIdx.x; i < pw2; i += blockDim.x) {
      uint64_t v;
      if (i < cnt) v = key_of(c0 + i);
      else if (i < tot) v = best[i - cnt];
      else v = 0;  // below every real key
      keys[i] = v;
    }
    __syncthreads();
    bitonic_sort_desc(keys, pw2);
    best_n = tot < k ? tot : k;
    for (int i = threadIdx.x; i < best_n; i += blockDim.x) best[i] = keys[i];
    __syncthreads();
  }
  *best_n_out = best_n;
}

__global__ void __launch_bounds__(kTopkThreads)
topk_kernel(const TopKParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint64_t* best = keys + kTopkSort;
  uint32_t* hash = reinterpret_cast<uint32_t*>(best + kMaxK);
  const uint32_t b = blockIdx.x;
  const uint64_t c0 = p.cand_off[b];
  const uint64_t n = p.cand_off[b + 1] - c0;
  const uint64_t n_needed = min((uint64_t)p.needed[b], n);
  const uint64_t n_scored = p.partial ? n : n_needed;
  const float alpha = p.alpha;
  // duplicate ids among scored candidates (rank() rejects them)
  if (n_scored <= kTopkHash / 2) {
    for (int i = threadIdx.x; i < kTopkHash; i += blockDim.x) hash[i] = 0xFFFFFFFFu;
    __syncthreads();
    for (uint64_t j = threadIdx.x; j < n_scored; j += blockDim.x) {
      const uint32_t id = p.cand_ids[c0 + j];
      uint32_t h = (id * 2654435761u) & (kTopkHash - 1);
      for (;;) {
        const uint32_t prev = atomicCAS(&hash[h], 0xFFFFFFFFu, id);
        if (prev == 0xFFFFFFFFu) break;
        if (prev == id) { atomicOr(p.err, ERR_DUPLICATE); break; }
        h = (h + 1) & (kTopkHash - 1);
      }
    }
    __syncthreads();
  }
  auto key_of = [&](uint64_t j) -> uint64_t {
    const uint32_t id = p.cand_ids[c0 + j];
    const float cls = p.cand_cls[c0 + j];
    const float bow = j < n_needed ? p.bow[c0 + j] : 0.0f;
    const float s = __fadd_rn(__fmul_rn(alpha, cls), bow);
    if (!isfinite(cls)) atomicOr(p.err, ERR_NONFINITE_CLS);
    else if (!isfinite(s)) atomicOr(p.err, ERR_NONFINITE_SCORE);
    return make_key(s, id);
  };
  int best_n = 0;
  topk_select(keys, best, (int)p.k, n_scored, key_of, &best_n);
  for (int i = threadIdx.x; i < (int)p.k; i += blockDim.x) {
    if (i < best_n) {
      const uint64_t key = best[i];
      p.out_ids[(size_t)b * p.k + i] = ~(uint32_t)(key & 0xFFFFFFFFu);
      p.out_scores[(size_t)b * p.k + i] = order_float((uint32_t)(key >> 32));
    }
  }
  if (threadIdx.x == 0) p.out_counts[b] = (uint32_t)best_n;
}

// K4: merge n_lists ranked lists per query ([list][query][k]) into one top-k.
__global__ void __launch_bounds__(kTopkThreads)
merge_topk_kernel(const uint32_t* ids, const float* scores, const uint32_t* counts,
                  uint32_t n_lists, uint64_t list_stride, uint32_t n_queries, uint32_t k,
                  uint32_t* out_ids, float* out_scores, uint32_t* out_counts) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint64_t* best = keys + kTopkSort;
  const uint32_t b = blockIdx.x;
  const uint64_t n = (uint64_t)n_lists * k;
  auto key_of = [&](uint64_t j) -> uint64_t {
    const uint32_t l = (uint32_t)(j / k), i = (uint32_t)(j % k);
    const size_t base = (size_t)l * list_stride;
    const size_t o = base + (size_t)b * k + i;
    if (i >= counts[base + b]) return 0;
    return make_key(scores[o], ids[o]);
  };
  int best_n = 0;
  topk_select(keys, best, (int)k, n, key_of, &best_n);
  // entries with key 0 are padding from short lists
  __shared__ int valid;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < (int)k; i += blockDim.x) {
    if (i < best_n && best[i] != 0) {
      out_ids[(size_t)b * k + i] = ~(uint32_t)(best[i] & 0xFFFFFFFFu);
      out_scores[(size_t)b * k + i] = order_float((uint32_t)(best[i] >> 32));
      atomicAdd(&valid, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out_counts[b] = (uint32_t)valid;
}

// ============================================================================
// K1 gather: request-order CSR of token rows.
// ============================================================================
__global__ void gather_count_kernel(const uint64_t* row_ptr, uint64_t n_docs, uint32_t shard_count,
                                    uint32_t shard_index, const uint32_t* ids, uint64_t n,
                                    uint64_t* out_row_ptr, uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t loc = shard_local(ids[i], shard_count, shard_index, n_docs);
    uint64_t t = 0;
    if (loc != ~0ull) t = row_ptr[loc + 1] - row_ptr[loc];
    else atomicOr(err, ERR_UNKNOWN_DOC);
    out_row_ptr[i + 1] = t;
  }
}

// Inclusive scan of a[1..n] in place (a[0] = 0), single block, chunked.
__global__ void __launch_bounds__(1024) scan_u64_kernel(uint64_t* a, uint64_t n) {
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t carry_sh;
  if (threadIdx.x == 0) { carry_sh = 0; a[0] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t base = 0; base < n; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    uint64_t v = i < n ? a[i + 1] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      uint64_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += u;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    const uint64_t off = carry_sh + (wid ? warp_sums[wid - 1] : 0);
    if (i < n) a[i + 1] = v + off;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_sh = off + v;
    __syncthreads();
  }
}

// Warp per doc, 16-byte vector copies, 4 in flight per lane.  Reads the HBM
// tile layout (RowLayout) and writes plain row-major rows in request order.
template <int D>
__global__ void __launch_bounds__(256)
gather_copy_kernel(const uint16_t* rows, const uint64_t* row_ptr, uint64_t n_docs, uint32_t shard_count,
                   uint32_t shard_index, const uint32_t* ids, uint64_t n, const uint64_t* out_row_ptr,
                   uint16_t* out_rows) {
  using RL = RowLayout<D>;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const uint64_t loc = shard_local(ids[i], shard_count, shard_index, n_docs);
    if (loc == ~0ull) continue;
    const uint64_t r0 = row_ptr[loc];
    const uint32_t t = (uint32_t)(row_ptr[loc + 1] - r0);
    const uint32_t nvec = t * RL::CH;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rows + r0 * D);
    uint4* dst = reinterpret_cast<uint4*>(out_rows + out_row_ptr[i] * D);
    auto at = [&](uint32_t v) {
      return __ldcs(reinterpret_cast<const uint4*>(src + RL::off(t, v / RL::CH, v % RL::CH)));
    };
    uint32_t v = lane;
    for (; v + 96 < nvec; v += 128) {
      const uint4 a0 = at(v), a1 = at(v + 32), a2 = at(v + 64), a3 = at(v + 96);
      __stcs(dst + v, a0);
      __stcs(dst + v + 32, a1);
      __stcs(dst + v + 64, a2);
      __stcs(dst + v + 96, a3);
    }
    for (; v < nvec; v += 32) __stcs(dst + v, at(v));
  }
}

// Plain row-major CSR rows -> HBM tile layout (table open).  Warp per doc.
template <int D>
__global__ void __launch_bounds__(256)
tile_rows_kernel(const uint16_t* plain, const uint64_t* row_ptr, uint64_t n_docs, uint16_t* tiled) {
  using RL = RowLayout<D>;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n_docs; i += nwarps) {
    const uint64_t r0 = row_ptr[i];
    const uint32_t t = (uint32_t)(row_ptr[i + 1] - r0);
    const uint4* src = reinterpret_cast<const uint4*>(plain + r0 * D);
    uint8_t* dst = reinterpret_cast<uint8_t*>(tiled + r0 * D);
    for (uint32_t v = lane; v < t * RL::CH; v += 32)
      *reinterpret_cast<uint4*>(dst + RL::off(t, v / RL::CH, v % RL::CH)) = __ldcs(src + v);
  }
}

// ============================================================================
// Synthetic table: counter-based RNG (splitmix64) so every doc / row can be
// regenerated independently.
// ============================================================================
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Length of global doc `gid`: t_min + h % (t_max - t_min + 1).
__global__ void synth_lengths_kernel(uint64_t n_docs, uint32_t t_min, uint32_t t_max, uint64_t seed,
                                     uint32_t shard_count, uint32_t shard_index, uint64_t* row_ptr) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_docs;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gid = i * shard_count + shard_index;
    const uint64_t h = splitmix64(seed ^ (gid * 0xD1B54A32D192ED03ull));
    row_ptr[i + 1] = t_min + (uint32_t)(h % (uint64_t)(t_max - t_min + 1));
  }
}

// Warp per doc, lane per token row: value k of token j of global doc gid is
// Box-Muller of h = splitmix64(base + (j << 16) + k), base = splitmix64(seed ^ gid*phi).
template <int D>
__global__ void synth_rows_kernel(uint64_t n_docs, const uint64_t* row_ptr, uint32_t shard_count,
                                  uint32_t shard_index, uint64_t seed, uint32_t bf16, uint16_t* rows) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n_docs; i += nwarps)
  for (uint64_t j = lane, r0 = row_ptr[i], t = row_ptr[i + 1] - r0; j < t; j += 32) {
    const uint64_t gid = i * shard_count + shard_index;
    const uint64_t base = splitmix64(seed ^ (gid * 0x9E3779B97F4A7C15ull));
    float v[D];
    float ss = 0.0f;
#pragma unroll
    for (int k = 0; k < D; k += 2) {
      const uint64_t h = splitmix64(base + (j << 16) + k);
      const float u1 = ((uint32_t)(h >> 40) + 1) * (1.0f / 16777217.0f);
      const float u2 = ((uint32_t)(h & 0xFFFFFFu)) * (1.0f / 16777216.0f);
      const float rad = sqrtf(-2.0f * logf(u1));
      float sn, cs;
      sincospif(2.0f * u2, &sn, &cs);
      v[k] = rad * cs;
      v[k + 1] = rad * sn;
      ss += v[k] * v[k] + v[k + 1] * v[k + 1];
    }
    const float inv = rsqrtf(fmaxf(ss, 1e-30f));
    uint32_t packed[D / 2];
#pragma unroll
    for (int k = 0; k < D; k += 2) {
      uint16_t c0 = espn_ptx::f32_to_code(v[k] * inv, bf16);
      uint16_t c1 = espn_ptx::f32_to_code(v[k + 1] * inv, bf16);
      // flush subnormals: the reference codec mis-decodes them
      if (!bf16) {
        if ((c0 & 0x7C00u) == 0) c0 &= 0x8000u;
        if ((c1 & 0x7C00u) == 0) c1 &= 0x8000u;
      } else {
        if ((c0 & 0x7F80u) == 0) c0 &= 0x8000u;
        if ((c1 & 0x7F80u) == 0) c1 &= 0x8000u;
      }
      packed[k / 2] = (uint32_t)c0 | ((uint32_t)c1 << 16);
    }
    // HBM tile layout (RowLayout): chunk k of row j of this doc
    uint8_t* dst = reinterpret_cast<uint8_t*>(rows + r0 * D);
#pragma unroll
    for (int k = 0; k < D / 8; ++k)
      *reinterpret_cast<uint4*>(dst + RowLayout<D>::off((uint32_t)t, (uint32_t)j, k)) =
          make_uint4(packed[4 * k], packed[4 * k + 1], packed[4 * k + 2], packed[4 * k + 3]);
  }
}

__global__ void minmax_len_kernel(const uint64_t* row_ptr, uint64_t n_docs, unsigned long long* out) {
  // out[0] = min t, out[1] = max t, out[2] = count of non-monotone / zero-length docs
  unsigned long long mn = ~0ull, mx = 0, bad = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_docs;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = row_ptr[i], c = row_ptr[i + 1];
    if (c <= a) { ++bad; continue; }
    const uint64_t t = c - a;
    mn = t < mn ? t : mn;
    mx = t > mx ? t : mx;
  }
  atomicMin(&out[0], mn);
  atomicMax(&out[1], mx);
  if (bad) atomicAdd(&out[2], bad);
}

}  // namespace espn_k
