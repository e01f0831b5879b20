// small.cuh -- K5: the whole re-rank of a small batch in ONE launch.
//
// configs[0] (batch 1 x 1000 candidates) is latency-bound: the three-kernel
// chain plan -> tcgen05 MaxSim -> finalize spends most of its ~15-20 us in
// per-kernel startup (TMEM allocation, barrier init, three dependent global
// round trips before the first copy) and in the launch gaps, not in the 1 MB
// of rows.  This kernel does stages 3-6 of run_query (pipeline.hpp:56-64) for
// a few queries in one grid:
//   * grid (P, B): CTA (p, b) scores chunk p of query b's scored list -- the
//     needed prefix min(R, n) (or needed_counts[b]); with partial re-rank the
//     tail [needed, n) as alpha*cls (SPEC.md:276 (5));
//   * candidate metadata (id -> row_ptr pair) one thread per candidate, so the
//     CTA pays two dependent round trips, not two per document; the same
//     threads insert the ids into the query's duplicate hash in L2 (rank()'s
//     duplicate rejection, scoring.hpp:16-18) and check the answers later;
//   * MaxSim on the CUDA cores, two warps per document (each half of its
//     rows), lane = query token, fp32 query, __fmul_rn/__fadd_rn in the
//     reference's order (scoring.hpp:7-10, 20-21); rows staged per warp in
//     shared memory with one coalesced round trip per piece.  Bit-exact with
//     the oracle: the max over rows is order-free (a +-0 tie cannot change
//     the sum, which starts at +0), the sum over query tokens is sequential;
//   * aggregate alpha*cls + bow without contraction (scoring.hpp:12-14) and
//     the CTA's best k by rank counting, written sorted to a per-CTA list;
//   * the query's last CTA to arrive (atomic counter) merges the P lists in
//     shared memory -- warps k-way merge 32 lists each, warp 0 merges their
//     results -- writes the ranked list and resets the query's hash/counter.
// Errors are the same bits as the three-kernel path (offsets, capacity,
// unknown id, non-finite query / cls / score, duplicates).
#pragma once
#include "common.cuh"
#include "ptx.cuh"
#include "maxsim_tc.cuh"  // fused_merge (long lists fallback)

namespace espn_k {

constexpr int kSmallThreads = 512;        // 16 warps: 8 documents in flight, two warps each
constexpr int kSmallDocsPerRound = kSmallThreads / 64;
// d >= 96 keeps the fp32 query row (d registers per lane) without spilling at
// 256 threads (4 documents per round)
template <int D>
constexpr int small_threads() { return D >= 96 ? 256 : kSmallThreads; }
constexpr int kSmallMaxB = 16;            // queries per small batch
constexpr int kSmallMaxChunk = 256;       // scored candidates per CTA
constexpr int kSmallMaxList = 2048;       // scored candidates per query
constexpr int kSmallHashSlots = 4096;     // per-query duplicate hash (2x the longest list)
constexpr int kSmallMaxCtas = 296;        // 2 per SM
constexpr int kSmallLevel1Keys = 16 * kFusedMaxK;  // <= 16 level-1 lists of k
#ifndef ESPN_SMALL_SELECT
#define ESPN_SMALL_SELECT 1  // last-CTA merge by threshold select (0: two-level k-way merge only)
#endif
// per-warp fp32 row staging: at least one quad of rows, within the 48 KB of
// static shared memory next to the query (32 x d fp32)
template <int D>
constexpr int small_wbuf() { return D <= 32 ? 2048 : (4 * 4 * D <= 1024 ? 1024 : 2048); }

struct SmallParams {
  MaxSimParams m;              // table, batch and outputs; m.unit_top = B x P x k per-CTA lists
  const uint32_t* needed_in;   // optional per-query needed override
  uint64_t max_candidates;     // workspace capacity (offset validation)
  uint32_t partial;            // tail beyond needed scored alpha*cls
  uint32_t P;                  // CTAs per query
  uint32_t base_ok;            // cand_off[0] may be nonzero (query slice of a larger CSR)
  uint32_t* arrive;            // B arrival counters, zero between batches
  uint32_t* hash;              // B x kSmallHashSlots ids, 0xFFFFFFFF = empty between batches
  uint32_t* ff_seen;           // B: id 0xFFFFFFFF (the empty code) seen, 0 between batches
};

// Host-side sizing (espn_gpu.cu): CTAs per query for the longest scored list.
inline uint32_t small_ctas_per_query(uint64_t max_scored, uint32_t B) {
  uint64_t P = (max_scored + kSmallDocsPerRound - 1) / kSmallDocsPerRound;  // one round of documents
  const uint64_t cap = B ? (uint64_t)kSmallMaxCtas / B : 1;
  if (P > cap) P = cap;
  return P < 1 ? 1u : (uint32_t)P;
}

// ESPN_RERANK_PROFILE: device-timed duration (first CTA start -> last CTA end),
// the same accumulator protocol as the MaxSim kernel (MaxSimParams::prof)
__device__ __forceinline__ void small_prof_end(const MaxSimParams& p) {
  if (p.prof && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.prof[3], 1ull) == (unsigned long long)gridDim.x * gridDim.y - 1) {  // last CTA out
      const unsigned long long t0 = atomicAdd(&p.prof[2], 0ull);
      atomicAdd(&p.prof[0], ktl_now() - t0);
      atomicAdd(&p.prof[1], 1ull);
      p.prof[2] = ~0ull;
      p.prof[3] = 0;
    }
  }
}

// One warp merges nl <= 32 descending lists of k keys (0 = empty) at
// lists[l * k], lane l owning list l: k rounds of warp max over the heads.
// Writes k keys (0-filled) to out; returns the number of non-empty keys.
__device__ __forceinline__ uint32_t small_kway(const uint64_t* lists, uint32_t nl, uint32_t k, uint64_t* out,
                                               uint32_t lane) {
  uint32_t cur = 0;
  uint64_t head = lane < nl ? lists[lane * k] : 0ull;
  uint32_t r = 0;
  for (; r < k; ++r) {
    const uint64_t m = warp_max_key(head);
    if (m == 0) break;
    const uint32_t win = __ffs(__ballot_sync(0xffffffffu, head == m)) - 1;
    if (lane == win) {
      ++cur;
      head = cur < k ? lists[lane * k + cur] : 0ull;
    }
    if (lane == 0) out[r] = m;
  }
  for (uint32_t i = r + lane; i < k; i += 32) out[i] = 0ull;
  return r;
}

template <int D>
__global__ void __launch_bounds__(small_threads<D>()) rerank_small_kernel(const SmallParams sp) {
  const MaxSimParams& p = sp.m;
  using RL = RowLayout<D>;
  constexpr uint32_t NT = small_threads<D>();
  constexpr uint32_t NW = NT / 32;
  constexpr uint32_t NDR = NT / 64;                          // documents per round
  constexpr uint32_t WBUF = small_wbuf<D>();                 // per-warp staging
  constexpr uint32_t WROWS = WBUF / (4 * D) / 4 * 4;         // fp32 rows per staged piece, whole quads
  constexpr int REGION = NW * WBUF;                          // row staging | last CTA: lists + level-1 merges
  constexpr int LIST_KEYS = REGION / 8 - kSmallLevel1Keys;   // P x k keys merged in shared memory
  constexpr uint32_t HM = kSmallHashSlots - 1;
  __shared__ __align__(16) float sq[32 * D];                 // query tokens (fp32, as given)
  __shared__ uint64_t keys[kSmallMaxChunk];                  // this CTA's candidate keys
  __shared__ uint64_t m_src[kSmallMaxChunk];                 // per candidate: row address (1: unknown id)
  __shared__ uint32_t m_t[kSmallMaxChunk], m_id[kSmallMaxChunk];
  __shared__ float m_cls[kSmallMaxChunk];
  __shared__ float halfmax[NDR][32];                         // second half's row maxima per document
  // compute phase: NW row-staging buffers; the last CTA's merge phase reuses
  // the space for the P lists and the level-1 merges
  __shared__ __align__(16) uint8_t region[REGION];
  __shared__ uint32_t s_last, s_ncand;
  __shared__ uint64_t s_thr;
  static_assert(WROWS >= 4 && LIST_KEYS >= 1024, "row staging / merge scratch");
  static_assert(NT >= kSmallMaxChunk, "one thread per candidate");
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t b = blockIdx.y, pc = blockIdx.x, P = sp.P;
  ktl_begin(p.dbg, 1);
  if (p.prof && tid == 0) atomicMin(&p.prof[2], ktl_now());
  // ESPN_DEBUG bit 8: per-CTA phase stamps (start, inputs ready, scored, done)
  const uint32_t cta = blockIdx.y * gridDim.x + blockIdx.x;
  const bool trace = (p.dbg & 8u) && tid == 0 && cta < 256;
  if (trace) g_cta_prof[4 * cta] = ktl_now();
  // ---- this query's list (validated before any dependent read) ----
  uint64_t off0 = p.cand_off[b], off1 = p.cand_off[b + 1];
  const bool bad_off = off1 < off0 || (b == 0 && off0 != 0 && !sp.base_ok);
  const bool over = !bad_off && off1 > sp.max_candidates;
  if ((bad_off || over) && pc == 0 && tid == 0) atomicOr(p.err, bad_off ? ERR_BAD_OFFSETS : ERR_CAPACITY);
  if (bad_off || over) off0 = off1 = 0;  // treated as empty; the call fails
  const uint64_t n = off1 - off0;
  const uint64_t cap = sp.needed_in ? (uint64_t)sp.needed_in[b] : (uint64_t)p.rerank_count;
  const uint64_t need = n < cap ? n : cap;
  const uint64_t ns = sp.partial ? n : need;  // scored candidates
  const uint64_t chunk = (ns + P - 1) / P;
  const uint64_t j0 = min(ns, (uint64_t)pc * chunk), j1 = min(ns, j0 + chunk);
  const uint32_t nc = (uint32_t)(j1 - j0);
  // host sizing guards both (device offsets: a list longer than the workspace's declared max_list)
  const bool too_long = ns > (uint64_t)kSmallMaxList;
  if ((nc > (uint32_t)kSmallMaxChunk || (pc == 0 && too_long)) && tid == 0) atomicOr(p.err, ERR_CAPACITY);
  const uint32_t ncs = min(nc, (uint32_t)kSmallMaxChunk);
  const uint32_t nq = p.nq;
  uint32_t ebits = 0;
  // ---- candidate metadata, one thread per candidate (two dependent round
  // trips for the whole CTA), and its duplicate-hash insert: the CAS answer
  // is only looked at after scoring, so its latency hides behind it ----
  uint32_t* qhash = sp.hash + (size_t)b * kSmallHashSlots;
  uint32_t my_id = 0, h = 0, cas_old = 0;
  bool pend = false;
  if (tid < ncs) {
    const uint64_t j = j0 + tid, c = off0 + j;
    my_id = __ldg(&p.cand_ids[c]);
    m_id[tid] = my_id;
    m_cls[tid] = __ldg(&p.cand_cls[c]);
    if (!too_long) {
      if (my_id == 0xFFFFFFFFu) {
        if (atomicExch(&sp.ff_seen[b], 1u)) ebits |= ERR_DUPLICATE;
      } else {
        h = ((my_id * 2654435761u) >> 7) & HM;
        cas_old = atomicCAS(&qhash[h], 0xFFFFFFFFu, my_id);
        pend = true;
      }
    }
    uint64_t src = 0;
    uint32_t t = 0;
    if (j < need) {
      const uint64_t loc = shard_local(my_id, p.shard_count, p.shard_index, p.n_docs);
      if (loc == ~0ull) {
        ebits |= ERR_UNKNOWN_DOC;
        src = 1;  // marker: no key
      } else {
        const uint64_t r0 = __ldg(&p.row_ptr[loc]);
        t = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
        src = reinterpret_cast<uint64_t>(p.rows + r0 * D);
      }
    }
    m_src[tid] = src;
    m_t[tid] = t;
  }
  if (j0 < need && ncs > 0) {
    const float* qs = p.q32 + (size_t)b * nq * D;
    bool badq = false;
    for (uint32_t i = tid; i < nq * D; i += NT) {
      const float x0 = __ldg(&qs[i]);
      const float x = p.qround ? espn_ptx::code_to_f32(espn_ptx::f32_to_code(x0, p.bf16), p.bf16) : x0;
      badq |= !isfinite(x);
      sq[i] = x;
    }
    if (badq) atomicOr(p.err, ERR_NONFINITE_QUERY);
  }
  __syncthreads();
  if (trace) g_cta_prof[4 * cta + 1] = ktl_now();
  float q[D];  // lane i: query token i (lanes >= nq mirror token 0; their maxima are not summed)
  {
    const float* qr = sq + (lane < nq ? lane : 0u) * D;
#pragma unroll
    for (int k4 = 0; k4 < D; k4 += 4) {
      const float4 v = *reinterpret_cast<const float4*>(qr + k4);
      q[k4] = v.x; q[k4 + 1] = v.y; q[k4 + 2] = v.z; q[k4 + 3] = v.w;
    }
  }
  const float alpha = p.alpha;
  uint8_t* wbuf = region + wid * WBUF;
  const uint32_t slot = wid >> 1, half = wid & 1;  // document slot of the round, row half
  // ---- rounds of NDR documents, two warps each: MaxSim (needed prefix) +
  // aggregate -> key ----
  for (uint32_t d0 = 0; d0 < ncs; d0 += NDR) {  // uniform across the CTA
    const uint32_t jj = d0 + slot;
    const uint64_t j = j0 + jj;
    const bool mine = jj < ncs;
    const uint64_t src = mine ? m_src[jj] : 0ull;
    const uint32_t t = mine ? m_t[jj] : 0u;
    const bool scored = mine && j < need && src != 1;
    float m = -INFINITY;
    if (scored) {
      const uint8_t* doc = reinterpret_cast<const uint8_t*>(src);
      const uint32_t th = (t + 1) / 2;
      const uint32_t ra = half ? th : 0u, rb = half ? t : th;  // this warp's rows [ra, rb)
      // rows in pieces of WROWS: one coalesced round trip per piece; each
      // lane converts its 16-byte chunks to fp32 once (not every lane per
      // element) into the warp's buffer laid out [row quad][k][4 rows], so
      // one broadcast 16-byte load feeds four rows' k-th products, computed
      // two at a time by the paired multiply (FMUL2, per component exactly
      // __fmul_rn) and summed per row with scalar __fadd_rn in ascending k
      // (the reference's order).  (A paired add after the paired multiply is
      // fused by ptxas into FFMA2 -- one rounding -- even with explicit .rn
      // and -fmad=false, so the sums stay scalar.)
      float* fbuf = reinterpret_cast<float*>(wbuf);
      for (uint32_t r0 = ra; r0 < rb; r0 += WROWS) {
        const uint32_t nr = min(WROWS, rb - r0);
        const uint32_t nv = nr * RL::CH;
        __syncwarp();  // the previous piece is consumed
        for (uint32_t v = lane; v < nv; v += 32) {
          const uint32_t jl = v / RL::CH, cc = v % RL::CH;
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(doc + RL::off(t, r0 + jl, cc)));
          const uint32_t w[4] = {x.x, x.y, x.z, x.w};
          float* dst = fbuf + ((jl >> 2) * D + cc * 8) * 4 + (jl & 3);
#pragma unroll
          for (int hh = 0; hh < 4; ++hh) {
            dst[(2 * hh) * 4] = espn_ptx::code_to_f32((uint16_t)(w[hh] & 0xFFFFu), p.bf16);
            dst[(2 * hh + 1) * 4] = espn_ptx::code_to_f32((uint16_t)(w[hh] >> 16), p.bf16);
          }
        }
        __syncwarp();
        uint32_t jr = 0;
        for (; jr + 4 <= nr; jr += 4) {  // a whole quad: two rows per paired op
          const float4* fq = reinterpret_cast<const float4*>(fbuf) + (jr >> 2) * D;
          float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
          for (int kk = 0; kk < D; ++kk) {
            const float4 x = fq[kk];
            const float2 qq = make_float2(q[kk], q[kk]);
            const float2 p01 = espn_ptx::mul2_rn(qq, make_float2(x.x, x.y));
            const float2 p23 = espn_ptx::mul2_rn(qq, make_float2(x.z, x.w));
            a0 = __fadd_rn(a0, p01.x);
            a1 = __fadd_rn(a1, p01.y);
            a2 = __fadd_rn(a2, p23.x);
            a3 = __fadd_rn(a3, p23.y);
          }
          if (a0 > m) m = a0;
          if (a1 > m) m = a1;
          if (a2 > m) m = a2;
          if (a3 > m) m = a3;
        }
        for (; jr < nr; ++jr) {  // the last < 4 rows, one at a time
          const float* fr = fbuf + (jr >> 2) * D * 4 + (jr & 3);
          float acc = 0.0f;
#pragma unroll
          for (int kk = 0; kk < D; ++kk) acc = __fadd_rn(acc, __fmul_rn(q[kk], fr[kk * 4]));
          if (acc > m) m = acc;
        }
      }
    }
    if (half) halfmax[slot][lane] = m;
    __syncthreads();
    if (!half && mine) {
      float bow = 0.0f;
      if (scored) {
        const float m2 = halfmax[slot][lane];
        if (m2 > m) m = m2;
        float s = 0.0f;
        for (uint32_t i = 0; i < nq; ++i) s = __fadd_rn(s, __shfl_sync(0xffffffffu, m, i));
        bow = s;
        if (p.bow_out && lane == 0) p.bow_out[off0 + j] = s;
      }
      if (lane == 0) {
        uint64_t key = 0;
        if (src != 1) {
          const float cl = m_cls[jj];
          const float sc = __fadd_rn(__fmul_rn(alpha, cl), bow);
          ebits |= !isfinite(cl) ? ERR_NONFINITE_CLS : (!isfinite(sc) ? ERR_NONFINITE_SCORE : 0u);
          key = make_key(sc, m_id[jj]);
        }
        keys[jj] = key;
      }
    }
    __syncthreads();  // halfmax / staging buffers reused by the next round
  }
  // ---- duplicate hash: the early CAS answers, further probes on collision ----
  while (pend) {
    if (cas_old == 0xFFFFFFFFu) break;
    if (cas_old == my_id) { ebits |= ERR_DUPLICATE; break; }
    h = (h + 1) & HM;
    cas_old = atomicCAS(&qhash[h], 0xFFFFFFFFu, my_id);
  }
  if (ebits) atomicOr(p.err, ebits);
  if (trace) g_cta_prof[4 * cta + 2] = ktl_now();
  // ---- the CTA's best k, sorted: key i goes to position rank(i) ----
  const uint32_t k = p.k;
  unsigned long long* mylist = p.unit_top + ((size_t)b * P + pc) * k;
  uint32_t nz = 0;
  {
    const uint64_t v = tid < ncs ? keys[tid] : 0ull;
    uint32_t rk = 0;
    if (v != 0)
      for (uint32_t i = 0; i < ncs; ++i) rk += keys[i] > v ? 1u : 0u;
    if (v != 0 && rk < k) __stcg(&mylist[rk], (unsigned long long)v);
    nz = (uint32_t)__syncthreads_count(v != 0);
  }
  for (uint32_t r = min(nz, k) + tid; r < k; r += NT) __stcg(&mylist[r], 0ull);
  // ---- arrival; the query's last CTA finishes it ----
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&sp.arrive[b], 1u) == P - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) {
    if (trace) g_cta_prof[4 * cta + 3] = ktl_now();
    ktl_end(p.dbg, 1);
    small_prof_end(p);
    return;
  }
  __threadfence();
  const unsigned long long* lists = p.unit_top + (size_t)b * P * k;
  const uint32_t nkeys = P * k;
  bool merged = false;
  if (nkeys <= (uint32_t)LIST_KEYS && P <= 32u * NW) {
    // the P lists -> shared memory in one round trip
    uint64_t* L0 = reinterpret_cast<uint64_t*>(region);
    uint64_t* L1 = L0 + LIST_KEYS;
    for (uint32_t i = tid; i < nkeys; i += NT) L0[i] = __ldcg(&lists[i]);
    if (tid == 0) {
      s_thr = 1ull;  // fewer than k non-empty lists: every non-empty key competes
      s_ncand = 0u;
    }
    __syncthreads();
#if ESPN_SMALL_SELECT
    // Threshold select (replaces two rounds of serial k-way merging, which
    // took ~7 us of the 17 us batch-1 kernel, small_timeline_r2.txt): the
    // lists are sorted and keys are unique, so with T = the k-th largest
    // list head there are k keys >= T and the query's top k are exactly the
    // k largest keys >= T.  Those come from the <= k lists whose head is
    // >= T, so there are at most k * k of them; each is placed by counting
    // the larger ones.  (Keys repeat only for duplicate ids, which fail the
    // call; more than kSmallLevel1Keys survivors falls back to the merge.)
    if (tid < P) {
      const uint64_t h = L0[tid * k];
      if (h != 0) {
        uint32_t above = 0;
        for (uint32_t m = 0; m < P; ++m) above += L0[m * k] > h ? 1u : 0u;
        if (above == k - 1) s_thr = h;
      }
    }
    __syncthreads();
    const uint64_t T = s_thr;
    for (uint32_t i = tid; i < nkeys; i += NT) {
      const uint64_t v = L0[i];
      if (v >= T) {
        const uint32_t at = atomicAdd(&s_ncand, 1u);
        if (at < (uint32_t)kSmallLevel1Keys) L1[at] = v;
      }
    }
    __syncthreads();
    const uint32_t M = s_ncand;
    if (M <= (uint32_t)kSmallLevel1Keys) {
      for (uint32_t i = tid; i < M; i += NT) {
        const uint64_t v = L1[i];
        uint32_t r = 0;
        for (uint32_t j = 0; j < M; ++j) r += L1[j] > v ? 1u : 0u;
        if (r < k) {
          p.out_ids[(size_t)b * k + r] = ~(uint32_t)(v & 0xFFFFFFFFu);
          p.out_scores[(size_t)b * k + r] = order_float((uint32_t)(v >> 32));
        }
      }
      if (tid == 0) p.out_counts[b] = min(M, k);
      merged = true;
    }
#endif
  }
  if (merged) {
    // (placed by the threshold select)
  } else if (nkeys <= (uint32_t)LIST_KEYS && P <= 32u * NW) {
    // warps k-way merge 32 lists each (level 1), warp 0 merges their results
    uint64_t* L0 = reinterpret_cast<uint64_t*>(region);
    uint64_t* L1 = L0 + LIST_KEYS;
    const uint32_t n1 = (P + 31) / 32;
    if (wid < n1) small_kway(L0 + (size_t)wid * 32 * k, min(32u, P - wid * 32), k, L1 + wid * k, lane);
    __syncthreads();
    if (wid == 0) {
      uint64_t* fin = L0;  // level 0 is consumed
      const uint32_t cnt = small_kway(L1, n1, k, fin, lane);
      __syncwarp();
      for (uint32_t r = lane; r < cnt; r += 32) {
        const uint64_t v = fin[r];
        p.out_ids[(size_t)b * k + r] = ~(uint32_t)(v & 0xFFFFFFFFu);
        p.out_scores[(size_t)b * k + r] = order_float((uint32_t)(v >> 32));
      }
      if (lane == 0) p.out_counts[b] = cnt;
    }
  } else if (wid == 0) {  // long: the chunked k-way merge straight from the lists
    fused_merge<LIST_KEYS>(p, b, b * P, P, reinterpret_cast<uint64_t*>(region), lane, /*kway=*/true);
  }
  // the batch is done for this query: reset its hash, empty-code flag and counter
  {
    uint4* h4 = reinterpret_cast<uint4*>(qhash);
    for (uint32_t i = tid; i < kSmallHashSlots / 4; i += NT)
      h4[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  }
  if (tid == 0) {
    sp.ff_seen[b] = 0u;
    sp.arrive[b] = 0u;  // every CTA of the query has arrived
  }
  ktl_end(p.dbg, 1);
  __syncthreads();  // (the profile's end stamp after the merge)
  if (trace) g_cta_prof[4 * cta + 3] = ktl_now() | (1ull << 63);  // the merging CTA
  small_prof_end(p);
}

template <int D>
cudaError_t launch_small(const SmallParams& sp, uint32_t B, cudaStream_t s) {
  rerank_small_kernel<D><<<dim3(sp.P, B), small_threads<D>(), 0, s>>>(sp);
  return cudaGetLastError();
}
inline cudaError_t launch_small_rt(uint32_t d, const SmallParams& sp, uint32_t B, cudaStream_t s) {
  switch (d) {
    case 8: return launch_small<8>(sp, B, s);
    case 16: return launch_small<16>(sp, B, s);
    case 32: return launch_small<32>(sp, B, s);
    case 48: return launch_small<48>(sp, B, s);
    case 64: return launch_small<64>(sp, B, s);
    case 96: return launch_small<96>(sp, B, s);
    case 128: return launch_small<128>(sp, B, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace espn_k
