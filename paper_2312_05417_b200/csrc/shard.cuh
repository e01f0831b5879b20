// shard.cuh -- multi-GPU re-rank kernels.
//
// Every rank receives the SAME global batch -- the candidate generator's
// top-K per query (ivf.hpp:45-50), global doc ids -- as run_batch would hand
// it over (pipeline.hpp:81-85).  Two placements:
//
//   SHARD   (table = doc-id shard g of G, owner(doc) = doc_id % G): rank g
//           keeps its own candidates, stably (so each sub-list stays sorted by
//           (cls desc, id asc)), with needed count = how many of them fall in
//           the query's global top-R prefix (SPEC.md:276 (3)); scores and
//           ranks them locally; the packed local top-k lists of all ranks are
//           all-gathered and merged (the global top-k is contained in the
//           union of the local ones).
//   REPLICA (every rank holds the whole table): rank g scores the queries
//           [g*B/G, (g+1)*B/G) and the all-gather reassembles the batch.
//
// The packed per-rank block (int32 words; the layout sharding.py restates):
//   [0..3]      error bits of the rank's local pass (word 0), 0, 0, 0
//   [4 ..)      ids    [BQ][k]   (BQ = B for SHARD, ceil(B/G) for REPLICA)
//               scores [BQ][k]   (fp32 bits)
//               counts [BQ]
#pragma once
#include "common.cuh"
#include "kernels_misc.cuh"

namespace espn_k {

constexpr int kPackHeaderWords = 4;
__host__ __device__ __forceinline__ uint64_t pack_words(uint64_t bq, uint32_t k) {
  return kPackHeaderWords + bq * (2ull * k + 1ull);
}

struct ShardSplitParams {
  const uint32_t* ids;       // global lists (CSR over queries)
  const float* cls;
  const uint64_t* off;       // B + 1
  const uint32_t* need_in;   // optional global needed counts (default min(R, n))
  uint32_t n_queries;
  uint32_t rerank_count;
  uint32_t shards, shard;    // G, g
  uint64_t max_candidates;   // bound check of the (device) offsets
  uint64_t* loc_off;         // out B + 1: [b + 1] = own count (scanned afterwards)
  uint32_t* loc_need;        // out B: own candidates inside the global needed prefix
  uint32_t* loc_ids;         // out (scatter pass)
  float* loc_cls;
  uint32_t* err;
};

constexpr int kShardThreads = 256;

// Pass 1 (CTA per query): own candidates and own needed count.
__global__ void __launch_bounds__(kShardThreads) shard_count_kernel(const ShardSplitParams p) {
  __shared__ uint32_t red[2][kShardThreads / 32];
  const uint32_t b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t a = p.off[b], e = p.off[b + 1];
  const bool bad = e < a || e > p.max_candidates;
  const uint64_t n = bad ? 0 : e - a;
  const uint64_t cap = p.need_in ? (uint64_t)p.need_in[b] : (uint64_t)p.rerank_count;
  const uint64_t need = n < cap ? n : cap;
  uint32_t own = 0, own_need = 0;
  for (uint64_t j = tid; j < n; j += kShardThreads) {
    const bool mine = (p.ids[a + j] % p.shards) == p.shard;
    own += mine;
    own_need += (mine && j < need) ? 1u : 0u;
  }
  own = __reduce_add_sync(0xffffffffu, own);
  own_need = __reduce_add_sync(0xffffffffu, own_need);
  if (lane == 0) { red[0][wid] = own; red[1][wid] = own_need; }
  __syncthreads();
  if (tid == 0) {
    uint32_t s0 = 0, s1 = 0;
    for (int i = 0; i < kShardThreads / 32; ++i) { s0 += red[0][i]; s1 += red[1][i]; }
    p.loc_off[b + 1] = s0;
    p.loc_need[b] = s1;
    if (bad) atomicOr(p.err, ERR_BAD_OFFSETS);
  }
}

// Pass 3 (CTA per query, after the scan of loc_off): stable compaction of the
// own candidates, 256 at a time (ballot prefix per warp, warp totals in smem).
__global__ void __launch_bounds__(kShardThreads) shard_scatter_kernel(const ShardSplitParams p) {
  __shared__ uint32_t wtot[kShardThreads / 32];
  const uint32_t b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t a = p.off[b], e = p.off[b + 1];
  if (e < a || e > p.max_candidates) return;
  const uint64_t n = e - a;
  uint64_t dst = p.loc_off[b];
  for (uint64_t j0 = 0; j0 < n; j0 += kShardThreads) {
    const uint64_t j = j0 + tid;
    uint32_t id = 0;
    float c = 0.f;
    bool mine = false;
    if (j < n) {
      id = p.ids[a + j];
      c = p.cls[a + j];
      mine = (id % p.shards) == p.shard;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) wtot[wid] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (int i = 0; i < kShardThreads / 32; ++i) {
      before += (i < (int)wid) ? wtot[i] : 0u;
      total += wtot[i];
    }
    if (mine) {
      const uint64_t o = dst + before + __popc(bal & ((1u << lane) - 1u));
      p.loc_ids[o] = id;
      p.loc_cls[o] = c;
    }
    dst += total;
    __syncthreads();
  }
}

// The rank's error word into its packed block (graph-capturable, no host hop).
__global__ void pack_err_kernel(const uint32_t* err, int32_t* packed) {
  if (threadIdx.x < kPackHeaderWords) packed[threadIdx.x] = threadIdx.x == 0 ? (int32_t)*err : 0;
}

// Merge (SHARD): per query the G ranked lists of the all-gathered blocks ->
// the global top-k by (score desc, doc_id asc) (scoring.hpp:16-18).  Block 0
// also ORs every rank's error bits into `err` so all ranks report the same
// verdict.
__global__ void __launch_bounds__(kTopkThreads)
merge_packed_kernel(const int32_t* recv, uint32_t G, uint64_t P, uint32_t B, uint32_t k, uint32_t* out_ids,
                    float* out_scores, uint32_t* out_counts, uint32_t* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint64_t* best = keys + kTopkSort;
  const uint32_t b = blockIdx.x;
  if (b == 0 && threadIdx.x < G) {
    const uint32_t e = (uint32_t)recv[(uint64_t)threadIdx.x * P];
    if (e) atomicOr(err, e);
  }
  const uint64_t o_sc = kPackHeaderWords + (uint64_t)B * k, o_cnt = kPackHeaderWords + 2ull * B * k;
  const uint64_t n = (uint64_t)G * k;
  auto key_of = [&](uint64_t j) -> uint64_t {
    const uint32_t l = (uint32_t)(j / k), i = (uint32_t)(j % k);
    const int32_t* blk = recv + (uint64_t)l * P;
    if (i >= (uint32_t)blk[o_cnt + b]) return 0;
    const uint64_t o = (uint64_t)b * k + i;
    return make_key(__int_as_float(blk[o_sc + o]), (uint32_t)blk[kPackHeaderWords + o]);
  };
  int best_n = 0;
  topk_select(keys, best, (int)k, n, key_of, &best_n);
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

// Unpack (REPLICA): query b was scored by rank r = the owner of its slice;
// copy its list out of r's block.  Grid: B blocks of 128 threads.
__global__ void unpack_replica_kernel(const int32_t* recv, uint32_t G, uint64_t P, uint32_t B, uint32_t BQ, uint32_t k,
                                      uint32_t* out_ids, float* out_scores, uint32_t* out_counts, uint32_t* err) {
  const uint32_t b = blockIdx.x;
  if (b == 0 && threadIdx.x < G) {
    const uint32_t e = (uint32_t)recv[(uint64_t)threadIdx.x * P];
    if (e) atomicOr(err, e);
  }
  const uint32_t r = b / BQ, i = b - r * BQ;
  const int32_t* blk = recv + (uint64_t)r * P;
  const uint64_t o_sc = kPackHeaderWords + (uint64_t)BQ * k, o_cnt = kPackHeaderWords + 2ull * BQ * k;
  const uint32_t cnt = (uint32_t)blk[o_cnt + i];
  for (uint32_t j = threadIdx.x; j < cnt && j < k; j += blockDim.x) {
    out_ids[(size_t)b * k + j] = (uint32_t)blk[kPackHeaderWords + (uint64_t)i * k + j];
    out_scores[(size_t)b * k + j] = __int_as_float(blk[o_sc + (uint64_t)i * k + j]);
  }
  if (threadIdx.x == 0) out_counts[b] = cnt;
}

}  // namespace espn_k
