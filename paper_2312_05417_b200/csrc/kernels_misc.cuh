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
// query token i (kept in registers as fp32), doc
// rows are read once with broadcast 16-byte loads.  Products and sums use
// __fmul_rn/__fadd_rn in ascending index order on the fp32 query, so the
// result equals the oracle (fed the same fp32 query) bit for bit.
// ============================================================================
template <int D>
__global__ void __launch_bounds__(256)
maxsim_simt_kernel(const MaxSimParams p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // pairs are enumerated over needed candidates only: query b contributes
  // needed[b] pairs; unit_off (plan_kernel, unit_docs = 1) is the pair prefix.
  const uint64_t n_pairs_total = p.unit_off[p.n_queries];
  const uint64_t per = (n_pairs_total + nw - 1) / nw;  // contiguous range per warp
  uint64_t pr = gw * per;
  const uint64_t pr_end = min(pr + per, n_pairs_total);
  if (pr >= pr_end) return;
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
        // the reference multiplies the fp32 query as given (types.hpp:33-44);
        // qround (ESPN_RERANK_QUERY_ROUNDED) first rounds it to the table dtype
        const float x0 = __ldg(&qs[k]);
        const float x = p.qround ? espn_ptx::code_to_f32(espn_ptx::f32_to_code(x0, p.bf16), p.bf16) : x0;
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
    const uint8_t* doc = p.cand_src ? reinterpret_cast<const uint8_t*>(p.cand_src[c])
                                    : reinterpret_cast<const uint8_t*>(p.rows + r0 * D);
    if (!doc) continue;  // not staged (staging overflow, reported by stage_kernel)
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
// Batch plan (device side).  CTA c owns queries [256c, 256c+256): it sums the
// work units of all earlier queries (block reduction over <= B offsets, cheap
// next to the batch), scans its own, and writes needed[], unit_off[] and the
// tcgen05 unit table.  Validates the offsets (start 0, non-decreasing, total
// within the workspace); on error the plan is empty (n_units = 0) so no kernel
// touches memory through a bad offset.
// ============================================================================
constexpr int kPlanThreads = 128;  // 128 x <=80 regs fits beside a resident MaxSim CTA (next batch plans early)
__device__ __forceinline__ uint64_t plan_units(const PlanParams& q, uint32_t b, uint32_t* need_out, bool* bad) {
  const uint64_t a = q.cand_off[b], e = q.cand_off[b + 1];
  if (e < a) { *bad = true; return 0; }
  const uint64_t n = e - a;
  const uint64_t cap = q.needed_in ? (uint64_t)q.needed_in[b] : (uint64_t)q.rerank_count;
  const uint64_t need = n < cap ? n : cap;
  *need_out = (uint32_t)need;
  if (!q.write_tab) return need;
  uint64_t u = (need + q.unit_docs - 1) / q.unit_docs;
  if (q.tail_units) u += (n - need + q.unit_docs - 1) / q.unit_docs;
  return u;
}
// Submission of the planned batch to a running persistent server (last plan
// CTA to finish, one thread): sequence number, wait for the slot's previous
// batch, descriptor copy, release-publish.
__device__ __noinline__ void server_submit(const ServerSubmit& sb) {
  ServerQueue* Q = sb.server;
  unsigned long long seq;
  for (;;) {  // take the next sequence number unless the server stopped
    const unsigned long long st = ld_acquire_u64(&Q->state);
    if (st & kServerStopped) {  // no server to take it: fail the batch, release the waiter
      atomicOr(sb.msp.err, ERR_SERVER);
      __threadfence();
      st_release_u32(sb.msp.done_flag, 1u);
      return;
    }
    if (atomicCAS(&Q->state, st, st + 1ull) == st) {
      seq = st;
      break;
    }
  }
  ServerSlot* sl = &Q->slot[seq % kServerSlots];
  const uint32_t want = seq >= (unsigned long long)kServerSlots ? (uint32_t)(seq - kServerSlots + 1) : 0u;
  while (ld_acquire_u32(&sl->done) != want) __nanosleep(128);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(&sb.msp);
  uint32_t* dst = reinterpret_cast<uint32_t*>(&sl->p);
  for (int i = 0; i < (int)(sizeof(MaxSimParams) / 4); ++i) __stcg(dst + i, src[i]);
  __threadfence();
  st_release_u32(&sl->ready, (uint32_t)seq + 1u);
}

// MINB = 16 caps the plan at 32 registers: a served batch's plan CTA must fit
// beside a persistent MaxSim CTA, whose 17 warps x 96 registers leave only
// 1024 registers free on the SM sub-partition holding 5 of them (each of the 4
// sub-partitions has 16K registers; a CTA's warps are spread over all four).
template <int MINB>
__global__ void __launch_bounds__(kPlanThreads, MINB) plan_kernel(const PlanParams q, const ServerSubmit sb) {
  ktl_begin(q.dbg, 0);
  // the MaxSim kernel is a programmatic dependent: its prologue (barriers,
  // TMEM, operand zeroing) overlaps this kernel; it waits before reading the plan
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ uint64_t wsum[kPlanThreads / 32];
  __shared__ uint64_t base_sh;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t q0 = blockIdx.x * kPlanThreads;
  bool bad = false;
  uint32_t dummy;
  // units of queries [0, q0)
  uint64_t pre = 0;
  for (uint32_t b = tid; b < q0; b += kPlanThreads) pre += plan_units(q, b, &dummy, &bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) wsum[wid] = pre;
  __syncthreads();
  if (tid == 0) {
    uint64_t t = 0;
    for (int i = 0; i < kPlanThreads / 32; ++i) t += wsum[i];
    base_sh = t;
  }
  __syncthreads();
  const uint64_t base = base_sh;
  // own query: exclusive block scan of its units
  const uint32_t b = q0 + tid;
  uint32_t need = 0;
  const uint64_t u = b < q.n_queries ? plan_units(q, b, &need, &bad) : 0;
  uint64_t incl = u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  __syncthreads();
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  uint64_t woff = 0;
  for (uint32_t i = 0; i < wid; ++i) woff += wsum[i];
  const uint64_t excl = base + woff + incl - u;
  if (tid == 0 && q.cand_off[0] != 0 && !q.base_ok) bad = true;  // base_ok: a slice of a larger CSR
  const bool last = b + 1 == q.n_queries;
  bool over = false;
  if (last && (q.cand_off[q.n_queries] > q.max_candidates || excl + u > q.max_units)) over = true;
  if (u > kUnitMaxPerQuery) over = true;
  // the last CTA has seen every query (prefix loop + its own): its verdict is global
  const bool any_bad = __syncthreads_or(bad);
  if (any_bad && tid == 0) atomicOr(q.err, ERR_BAD_OFFSETS);
  if (over) atomicOr(q.err, ERR_CAPACITY);
  if (b < q.n_queries) {
    q.needed[b] = need;
    q.unit_off[b] = (uint32_t)excl;
    if (q.write_tab && excl + u <= q.max_units) {
      // MaxSim units over [0, need), then (fused partial re-rank) alpha*cls
      // tail units over [need, n)
      const uint64_t c0 = q.cand_off[b], n = q.cand_off[b + 1] - c0;
      const uint64_t um = (need + q.unit_docs - 1) / q.unit_docs;
      for (uint64_t j = 0; j < u; ++j) {
        const bool tail = j >= um;
        const uint64_t first = tail ? need + (j - um) * q.unit_docs : j * q.unit_docs;
        const uint64_t end = tail ? n : (uint64_t)need;
        const uint64_t c = c0 + first;
        const uint32_t nd = (uint32_t)min((uint64_t)q.unit_docs, end - first);
        q.unit_tab[excl + j] = make_uint4(b, unit_y(nd, (uint32_t)u, tail), (uint32_t)c, (uint32_t)(c >> 32));
      }
    }
    if (q.out_counts && u == 0) q.out_counts[b] = 0;  // fused top-k: no unit will rank this query
  }
  if (last) {
    if (q.fused_state) {  // fused top-k: this batch's dedup parity and the rows it uses
      const uint32_t ep = q.fused_state[0] + 1u;
      q.fused_state[0] = ep;
      q.fused_state[1 + (ep & 1u)] = q.n_queries;
    }
    q.unit_off[q.n_queries] = (uint32_t)(excl + u);
    // read by the MaxSim kernel; an invalid batch gets an empty plan
    *q.n_units = (any_bad || over) ? 0u : (uint32_t)(excl + u);
  }
  if (sb.server) {  // persistent server: the last plan CTA to finish publishes the batch
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(sb.plan_done, 1u) == gridDim.x - 1) {
        *sb.plan_done = 0;
        __threadfence();
        server_submit(sb);
      }
    }
  }
  ktl_end(q.dbg, 0);
}

// The caller's stream waits for its batch (persistent server): one thread
// polls the workspace's done flag and consumes it.  A batch that does not
// complete within timeout_ns (server stopped or stalled) raises ERR_SERVER
// instead of hanging the stream.
__global__ void server_wait_kernel(uint32_t* flag, uint32_t* err, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = ktl_now();
  while (ld_acquire_u32(flag) == 0u) {
    __nanosleep(256);
    if (ktl_now() - t0 > timeout_ns) {
      atomicOr(err, ERR_SERVER);
      return;
    }
  }
  *flag = 0u;
  __threadfence();
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
  ktl_begin(p.dbg, 2);
  if (*p.err & (ERR_BAD_OFFSETS | ERR_CAPACITY)) return;  // plan rejected the batch
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

// K3 fast path (final_k <= KMAX <= 32): one 256-thread CTA per query, no
// sort.  (1) Duplicate detection (rank() rejects duplicate ids,
// scoring.hpp:16-18) over the scored ids in a shared-memory open-addressing
// table WITHOUT atomics: entries are (id << 32 | index); each round every
// pending id is written to its probe slot if the slot looks empty, then read
// back after a barrier -- own entry = placed, same id with another index =
// duplicate, other id = probe on.  This phase reads only candidate ids, so it
// runs before the programmatic-dependent-launch wait and overlaps the MaxSim
// kernel's tail.  (2) Each thread keeps its best KMAX keys in registers;
// k rounds of warp max-reduction produce per-warp lists, merged the same way
// by warp 0.  Keys are (orderable score << 32 | ~doc_id): larger key =
// (score desc, doc_id asc), exactly rank()'s comparator.
constexpr int kTopkCtaThreads = 256;
template <int KMAX>
__global__ void __launch_bounds__(kTopkCtaThreads)
topk_cta_kernel(const TopKParams p, uint32_t hash_slots) {
  extern __shared__ __align__(16) uint64_t tk_smem[];
  uint64_t* hash = tk_smem;                          // hash_slots entries
  uint64_t* wl = tk_smem + hash_slots;               // 8 warps x KMAX merged lists
  __shared__ int any_pending;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t b = blockIdx.x;
  ktl_begin(p.dbg, 2);
  if (*p.err & (ERR_BAD_OFFSETS | ERR_CAPACITY)) return;  // plan rejected the batch
  const uint64_t c0 = p.cand_off[b];
  const uint64_t n = p.cand_off[b + 1] - c0;
  const uint64_t n_needed = min((uint64_t)p.needed[b], n);
  const uint64_t n_scored = p.partial ? n : n_needed;
  constexpr uint64_t EMPTY = ~0ull;
  if (n_scored * 2 <= hash_slots && !(p.dbg & 128u)) {
    for (uint32_t i = tid; i < hash_slots; i += kTopkCtaThreads) hash[i] = EMPTY;
    uint32_t dup = 0;
    for (uint64_t j0 = 0; j0 < n_scored; j0 += kTopkCtaThreads * 4) {
      uint32_t idv[4], hpos[4], pend = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t j = j0 + u * kTopkCtaThreads + tid;
        idv[u] = j < n_scored ? __ldg(&p.cand_ids[c0 + j]) : 0u;
        if (j < n_scored) pend |= 1u << u;
        hpos[u] = ((idv[u] * 2654435761u) >> 7) & (hash_slots - 1);
      }
      if (j0 == 0) __syncthreads();  // table initialised
      // one shared 64-bit CAS per probe: {id, position} claims an empty slot;
      // a slot holding the same id is a duplicate
      while (pend) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (pend & (1u << u)) {
            const uint64_t mine = ((uint64_t)idv[u] << 32) | (uint32_t)(j0 + u * kTopkCtaThreads + tid);
            const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(&hash[hpos[u]]),
                                           (unsigned long long)EMPTY, (unsigned long long)mine);
            if (old == EMPTY) {
              pend &= ~(1u << u);
            } else if ((uint32_t)(old >> 32) == idv[u]) {
              dup = 1;
              pend &= ~(1u << u);
            } else {
              hpos[u] = (hpos[u] + 1) & (hash_slots - 1);
            }
          }
        }
      }
    }
    if (dup) atomicOr(p.err, ERR_DUPLICATE);
  }
  (void)any_pending;
  // bow scores come from the preceding MaxSim kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const float alpha = p.alpha;
  uint64_t best[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) best[i] = 0;
  uint32_t bad = 0;
  for (uint64_t j0 = 0; j0 < n_scored; j0 += kTopkCtaThreads * 4) {
    uint32_t idv[4];
    float clv[4], bwv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // batch the loads
      const uint64_t j = j0 + u * kTopkCtaThreads + tid;
      idv[u] = j < n_scored ? __ldg(&p.cand_ids[c0 + j]) : 0u;
      clv[u] = j < n_scored ? __ldg(&p.cand_cls[c0 + j]) : 0.0f;
      bwv[u] = j < n_needed ? p.bow[c0 + j] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u * kTopkCtaThreads + tid >= n_scored) continue;
      const float sc = __fadd_rn(__fmul_rn(alpha, clv[u]), bwv[u]);
      bad |= !isfinite(clv[u]) ? ERR_NONFINITE_CLS : (!isfinite(sc) ? ERR_NONFINITE_SCORE : 0u);
      const uint64_t key = make_key(sc, idv[u]);
      if (key > best[KMAX - 1]) {
        best[KMAX - 1] = key;
#pragma unroll
        for (int i = KMAX - 1; i > 0; --i) {
          const uint64_t a = best[i - 1], c = best[i];
          best[i - 1] = a > c ? a : c;
          best[i] = a > c ? c : a;
        }
      }
    }
  }
  if (bad) atomicOr(p.err, bad);
  const uint32_t k = p.k;
  // per-warp merge: k rounds of warp max over the lanes' list heads
  for (uint32_t r = 0; r < k; ++r) {
    uint64_t m = best[0];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t x = __shfl_xor_sync(0xffffffffu, m, o);
      m = x > m ? x : m;
    }
    if (best[0] == m && m != 0) {
#pragma unroll
      for (int i = 0; i < KMAX - 1; ++i) best[i] = best[i + 1];
      best[KMAX - 1] = 0;
    }
    if (lane == 0) wl[wid * KMAX + r] = m;
  }
  __syncthreads();
  // block merge by warp 0: lane l < 8 walks warp l's sorted list
  if (wid == 0) {
    uint32_t pos = 0;
    uint32_t r = 0;
    for (; r < k; ++r) {
      uint64_t h = (lane < kTopkCtaThreads / 32 && pos < k) ? wl[lane * KMAX + pos] : 0;
      uint64_t m = h;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, m, o);
        m = x > m ? x : m;
      }
      if (m == 0) break;  // fewer than k scored candidates
      if (h == m) ++pos;
      if (lane == 0) {
        p.out_ids[(size_t)b * k + r] = ~(uint32_t)(m & 0xFFFFFFFFu);
        p.out_scores[(size_t)b * k + r] = order_float((uint32_t)(m >> 32));
      }
    }
    if (lane == 0) p.out_counts[b] = r;
  }
  ktl_end(p.dbg, 2);
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

// Warp per group of 8 requested docs.  Lanes 0-7 resolve the group's metadata
// together (id -> row_ptr pair, output offset: one dependent round trip per 8
// docs instead of per doc), then the warp copies the docs two at a time with
// 16-byte vectors, 8 loads per lane in flight.  Reads the HBM tile layout
// (RowLayout) and writes plain row-major rows in request order.
#ifndef ESPN_GATHER_MINB
#define ESPN_GATHER_MINB 4  // 4 CTAs per SM (<= 64 registers): 4.26 -> 4.70 TB/s on C2
#endif
template <int D>
__global__ void __launch_bounds__(256, ESPN_GATHER_MINB)
gather_copy_kernel(const uint16_t* rows, const uint64_t* doc_loc, const uint64_t* row_ptr, uint64_t n_docs,
                   uint32_t shard_count, uint32_t shard_index, const uint32_t* ids, uint64_t n,
                   const uint64_t* out_row_ptr, uint16_t* out_rows) {
  using RL = RowLayout<D>;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ngroups = (n + 7) / 8;
  for (uint64_t g = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; g < ngroups; g += nwarps) {
    const uint64_t i = g * 8 + (lane & 7);
    uint64_t src = 0, dst = 0;
    uint32_t t = 0;
    if (lane < 8 && i < n) {
      const uint64_t loc = shard_local(__ldg(&ids[i]), shard_count, shard_index, n_docs);
      dst = reinterpret_cast<uint64_t>(out_rows + __ldg(&out_row_ptr[i]) * D);
      if (loc != ~0ull) {  // (unknown ids were rejected by the count pass)
        const uint64_t r0 = __ldg(&row_ptr[loc]);
        t = (uint32_t)(__ldg(&row_ptr[loc + 1]) - r0);
        src = reinterpret_cast<uint64_t>(doc_rows(rows, doc_loc, loc, r0, D));
      }
    }
#pragma unroll 1
    for (int p = 0; p < 8; p += 2) {
      const uint32_t ta = __shfl_sync(0xffffffffu, t, p), tb = __shfl_sync(0xffffffffu, t, p + 1);
      const uint8_t* sa = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, src, p));
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, src, p + 1));
      uint4* da = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, dst, p));
      uint4* db = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, dst, p + 1));
      const uint32_t na = ta * RL::CH, nb = tb * RL::CH, nm = na > nb ? na : nb;
      for (uint32_t v0 = 0; v0 < nm; v0 += 128) {
        uint4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t v = v0 + u * 32 + lane;
          if (v < na) a[u] = __ldcs(reinterpret_cast<const uint4*>(sa + RL::off(ta, v / RL::CH, v % RL::CH)));
          if (v < nb) b[u] = __ldcs(reinterpret_cast<const uint4*>(sb + RL::off(tb, v / RL::CH, v % RL::CH)));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t v = v0 + u * 32 + lane;
          if (v < na) __stcs(da + v, a[u]);
          if (v < nb) __stcs(db + v, b[u]);
        }
      }
    }
  }
}

// Tiered table open: copy each doc's (tiled) rows from the full device copy to
// its tier -- HBM compact buffer or mapped pinned-host memory.  Warp per doc.
__global__ void __launch_bounds__(256)
relocate_rows_kernel(const uint8_t* src_rows, const uint64_t* row_ptr, const uint64_t* doc_loc, uint64_t n_docs,
                     uint32_t row_bytes) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n_docs; i += nwarps) {
    const uint64_t r0 = row_ptr[i];
    const uint64_t n16 = (row_ptr[i + 1] - r0) * row_bytes / 16;
    const uint4* src = reinterpret_cast<const uint4*>(src_rows + r0 * row_bytes);
    uint4* dst = reinterpret_cast<uint4*>(doc_loc[i] & ~1ull);
    for (uint64_t v = lane; v < n16; v += 32) dst[v] = __ldcs(src + v);
  }
}

// CTA size of the staging kernels: one CTA per query, a warp per candidate --
// every warp walks its docs one PCIe/HBM round trip at a time, so more warps
// per query mean more transfers in flight.
#ifndef ESPN_STAGE_THREADS
#define ESPN_STAGE_THREADS 1024
#endif
constexpr int kStageThreads = ESPN_STAGE_THREADS;

// Per-batch staging of host-tier rows (tiered tables).  CTA per query, warp per
// needed candidate: resident docs resolve to their HBM address; host-tier docs
// are copied (16-byte loads from mapped pinned memory, i.e. PCIe reads) into
// the staging buffer.  Writes the per-candidate row address the MaxSim kernel
// reads, and the per-query fetch accounting.
__global__ void __launch_bounds__(kStageThreads) stage_kernel(const StageParams s) {
  const uint32_t b = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t c0 = s.cand_off[b], c1 = s.cand_off[b + 1];
  if (c1 < c0 || c1 > s.max_candidates) return;  // invalid batch: the plan kernel reports it
  const uint64_t n = c1 - c0;
  const uint64_t cap = s.needed_in ? (uint64_t)s.needed_in[b] : (uint64_t)s.rerank_count;
  const uint64_t need = n < cap ? n : cap;
  unsigned long long resident = 0, staged = 0, bytes_moved = 0, hits = 0;
  for (uint64_t j = wid; j < need; j += nw) {
    const uint64_t loc = shard_local(s.cand_ids[c0 + j], s.shard_count, s.shard_index, s.n_docs);
    if (loc == ~0ull) {  // reported as DATA_INTEGRITY by the MaxSim kernel
      if (lane == 0) { s.cand_src[c0 + j] = 0; if (s.cand_status) s.cand_status[c0 + j] = 3; }
      continue;
    }
    const uint64_t a = s.doc_loc[loc];
    if (!(a & 1ull)) {
      if (lane == 0) { s.cand_src[c0 + j] = a; if (s.cand_status) s.cand_status[c0 + j] = 0; }
      ++resident;
      continue;
    }
    if (s.hint_map) {  // staged ahead by espn_gpu_prefetch_hints?
      const uint64_t e = s.hint_map[loc];
      if ((uint32_t)(e >> 32) == s.hint_epoch && (uint32_t)e != 0xffffffffu) {
        if (lane == 0) {
          s.cand_src[c0 + j] = reinterpret_cast<uint64_t>(s.stage) + ((e & 0xffffffffull) << 4);
          if (s.cand_status) s.cand_status[c0 + j] = 1;
        }
        ++hits;
        continue;
      }
    }
    if (a & kLocDisk) {  // disk tier, not staged by espn_gpu_prefetch_rows: cannot be copied from memory
      if (lane == 0) {
        atomicOr(s.err, ERR_NOT_PREFETCHED);
        s.cand_src[c0 + j] = 0;
        if (s.cand_status) s.cand_status[c0 + j] = 3;
      }
      continue;
    }
    const uint64_t bytes = (s.row_ptr[loc + 1] - s.row_ptr[loc]) * s.row_bytes;
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(s.cursor, (unsigned long long)bytes);
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off + bytes > s.stage_cap) {
      if (lane == 0) {
        atomicOr(s.err, ERR_STAGING);
        s.cand_src[c0 + j] = 0;
        if (s.cand_status) s.cand_status[c0 + j] = 3;
      }
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(a & ~1ull);
    uint4* dst = reinterpret_cast<uint4*>(s.stage + off);
    const uint64_t n16 = bytes / 16;
    uint64_t v = lane;
    for (; v + 96 < n16; v += 128) {  // 4 PCIe reads in flight per lane
      const uint4 x0 = src[v], x1 = src[v + 32], x2 = src[v + 64], x3 = src[v + 96];
      dst[v] = x0; dst[v + 32] = x1; dst[v + 64] = x2; dst[v + 96] = x3;
    }
    for (; v < n16; v += 32) dst[v] = src[v];
    if (lane == 0) {
      s.cand_src[c0 + j] = reinterpret_cast<uint64_t>(s.stage + off);
      if (s.cand_status) s.cand_status[c0 + j] = s.prefetch ? 1 : 2;
    }
    ++staged;
    bytes_moved += bytes;
  }
  if (lane == 0 && s.qstats) {
    unsigned long long* q = s.qstats + (size_t)b * 6;
    if (wid == 0) atomicAdd(&q[0], (unsigned long long)need);
    atomicAdd(&q[1], resident);
    atomicAdd(&q[s.prefetch ? 2 : 3], staged);
    atomicAdd(&q[s.prefetch ? 4 : 5], bytes_moved);
    if (hits) atomicAdd(&q[2], hits);
  }
}

// Hint staging (espn_gpu_prefetch_hints): the host-tier rows of each query's
// hinted docs -> staging buffer, one copy per doc per epoch (the first warp to
// claim the doc's hint-map entry copies it; the others skip).  The consumer
// (stage_kernel with hint_map) runs after this kernel on another stream,
// ordered by an event, so plain stores publish the entries.
__global__ void __launch_bounds__(kStageThreads) hint_stage_kernel(const HintParams s) {
  const uint32_t b = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t h0 = s.hint_off[b], h1 = s.hint_off[b + 1];
  if (h1 < h0 || h1 > s.max_hints) {
    if (threadIdx.x == 0) atomicOr(s.err, ERR_BAD_OFFSETS);
    return;
  }
  unsigned long long bytes_moved = 0;
  for (uint64_t j = h0 + wid; j < h1; j += nw) {
    const uint64_t loc = shard_local(s.hint_ids[j], s.shard_count, s.shard_index, s.n_docs);
    if (loc == ~0ull) continue;  // another shard's doc, or unknown: hints are advisory
    const uint64_t a = s.doc_loc[loc];
    if (!(a & kLocHost)) continue;                  // HBM-resident
    if ((a & kLocDisk) && !s.ext_src) continue;     // disk tier: only espn_gpu_prefetch_rows stages it
    const uint64_t bytes = (s.row_ptr[loc + 1] - s.row_ptr[loc]) * s.row_bytes;
    unsigned long long off = ~0ull;
    if (lane == 0) {
      const uint64_t e = s.hint_map[loc];
      if ((uint32_t)(e >> 32) != s.epoch &&
          atomicCAS(reinterpret_cast<unsigned long long*>(&s.hint_map[loc]), (unsigned long long)e,
                    ((unsigned long long)s.epoch << 32) | 0xffffffffull) == (unsigned long long)e) {
        // bounded bump allocation: a failed add is undone, so while any failure
        // is pending every add fails and successful regions never overlap
        const unsigned long long cur = atomicAdd(s.cursor, (unsigned long long)bytes);
        if (cur + bytes <= s.stage_cap) {
          off = cur;
        } else {
          atomicAdd(s.cursor, (unsigned long long)(0ull - bytes));
          s.hint_map[loc] = 0;  // budget spent: the consumer copies it on the critical path
        }
      }
    }
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off == ~0ull) continue;
    const uint64_t n16 = bytes / 16;
    if (s.ext_src) {  // caller rows (plain) -> tile layout in the staging slot
      const uint4* src = reinterpret_cast<const uint4*>(s.ext_src + s.ext_off[j]);
      uint8_t* dst = s.stage + off;
      const uint32_t t = (uint32_t)(s.row_ptr[loc + 1] - s.row_ptr[loc]), ch = s.d / 8;
      for (uint64_t v = lane; v < n16; v += 32) {
        const uint32_t jr = (uint32_t)(v / ch), cc = (uint32_t)(v % ch);
        *reinterpret_cast<uint4*>(dst + tile_off_rt(s.d, t, jr, cc)) = src[v];
      }
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(a & ~kLocHost);
      uint4* dst = reinterpret_cast<uint4*>(s.stage + off);
      uint64_t v = lane;
      for (; v + 96 < n16; v += 128) {  // 4 PCIe reads in flight per lane
        const uint4 x0 = src[v], x1 = src[v + 32], x2 = src[v + 64], x3 = src[v + 96];
        dst[v] = x0; dst[v + 32] = x1; dst[v + 64] = x2; dst[v + 96] = x3;
      }
      for (; v < n16; v += 32) dst[v] = src[v];
    }
    if (lane == 0) s.hint_map[loc] = ((uint64_t)s.epoch << 32) | (off >> 4);
    bytes_moved += bytes;
  }
  if (lane == 0 && s.qstats && bytes_moved) atomicAdd(&s.qstats[(size_t)b * 6 + 4], bytes_moved);
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

namespace espn_k {
// ============================================================================
// Reference scoring primitives on the device (the unmodified-header API of
// csrc/host/espn_ref_api.cpp): fp32 inputs, the reference's fixed order.
// ============================================================================
// maxsim_score (scoring.hpp:7-10): block i = query token i; thread j-strided
// over doc tokens: dot over k ascending (__fmul_rn/__fadd_rn), max over j
// (exact); then one thread sums the per-token maxima in ascending i.
__global__ void __launch_bounds__(256) maxsim_f32_kernel(const float* q, const float* doc, uint32_t t, uint32_t d,
                                                        float* qmax) {
  __shared__ float red[256];
  const uint32_t i = blockIdx.x;
  float m = -INFINITY;
  for (uint32_t j = threadIdx.x; j < t; j += blockDim.x) {
    float acc = 0.0f;
    for (uint32_t k = 0; k < d; ++k) acc = __fadd_rn(acc, __fmul_rn(q[(size_t)i * d + k], doc[(size_t)j * d + k]));
    m = acc > m ? acc : m;
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) qmax[i] = red[0];
}
__global__ void sum_ordered_kernel(const float* x, uint32_t n, float* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float s = 0.0f;
  for (uint32_t i = 0; i < n; ++i) s = __fadd_rn(s, x[i]);
  *out = s;
}

// rank (scoring.hpp:16-18): keys orderable(score) << 32 | ~id (descending =
// (score desc, id asc)); non-finite scores flagged.
__global__ void rank_keys_kernel(const uint32_t* ids, const float* scores, uint64_t n, unsigned long long* keys,
                                 uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float s = scores[i];
    if (!isfinite(s)) atomicOr(err, ERR_NONFINITE_SCORE);
    keys[i] = make_key(s, ids[i]);
  }
}
__global__ void rank_unkey_kernel(const unsigned long long* keys, uint64_t n, uint32_t* ids, float* scores) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    ids[i] = ~(uint32_t)(keys[i] & 0xFFFFFFFFull);
    scores[i] = order_float((uint32_t)(keys[i] >> 32));
  }
}
// duplicates: ids sorted ascending, any equal neighbours
__global__ void adjacent_dup_kernel(const uint32_t* sorted_ids, uint64_t n, uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (sorted_ids[i] == sorted_ids[i + 1]) atomicOr(err, ERR_DUPLICATE);
}
}  // namespace espn_k

namespace espn_k {
// Streamed table fill (espn_gpu_table_load_rows): warp per doc, plain rows
// from a bounce chunk -> the doc's tile-layout destination in HBM.
struct TileJob {
  uint64_t src;  // byte offset of the doc's plain rows in the chunk
  uint64_t dst;  // destination address
  uint32_t t;    // tokens
  uint32_t pad;
};
template <int D>
__global__ void __launch_bounds__(256) tile_jobs_kernel(const uint8_t* chunk, const TileJob* jobs, uint32_t n) {
  using RL = RowLayout<D>;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const TileJob j = jobs[i];
    const uint4* src = reinterpret_cast<const uint4*>(chunk + j.src);
    uint8_t* dst = reinterpret_cast<uint8_t*>(j.dst);
    for (uint32_t v = lane; v < j.t * RL::CH; v += 32)
      *reinterpret_cast<uint4*>(dst + RL::off(j.t, v / RL::CH, v % RL::CH)) = src[v];
  }
}
}  // namespace espn_k
