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
//   * MaxSim on the CUDA cores, warp per document, lane = query token, fp32
//     query, __fmul_rn/__fadd_rn in the reference's order (scoring.hpp:7-10,
//     20-21): bit-exact with the oracle, like maxsim_simt_kernel; rows are read
//     from the tile layout (RowLayout::off) with broadcast 16-byte loads;
//   * aggregate alpha*cls + bow without contraction (scoring.hpp:12-14) and
//     the CTA's best k by rank counting, written sorted to a per-CTA list;
//   * the query's last CTA to arrive (atomic counter, reset by itself) merges
//     the P lists (fused_merge, the finalize merge) in warp 0 while warps 1-7
//     run rank()'s duplicate check (scoring.hpp:16-18) over the query's scored
//     ids in a shared-memory hash.
// Errors are the same bits as the three-kernel path (offsets, capacity,
// unknown id, non-finite query / cls / score, duplicates).
#pragma once
#include "common.cuh"
#include "ptx.cuh"
#include "maxsim_tc.cuh"  // fused_merge

namespace espn_k {

constexpr int kSmallThreads = 256;        // 8 warps
constexpr int kSmallMaxB = 16;            // queries per small batch
constexpr int kSmallMaxChunk = 256;       // scored candidates per CTA
constexpr int kSmallMaxList = 2048;       // scored candidates per query (dedup hash: 2x)
constexpr int kSmallMaxCtas = 296;        // 2 per SM
constexpr int kSmallMergeKeys = 1016;     // merge scratch (P x k keys; longer -> k-way merge)
constexpr int kSmallWarpRowBytes = 2048;  // per-warp row staging (one piece: 32 rows at d=32)
constexpr int kSmallRegionBytes = 24 * 1024;  // row staging | last CTA: merge keys + dedup hash

struct SmallParams {
  MaxSimParams m;              // table, batch and outputs; m.unit_top = B x P x k per-CTA lists
  const uint32_t* needed_in;   // optional per-query needed override
  uint64_t max_candidates;     // workspace capacity (offset validation)
  uint32_t partial;            // tail beyond needed scored alpha*cls
  uint32_t P;                  // CTAs per query
  uint32_t base_ok;            // cand_off[0] may be nonzero (query slice of a larger CSR)
  uint32_t* arrive;            // B arrival counters, zero between batches
};

// Host-side sizing (espn_gpu.cu): CTAs per query for the longest scored list.
inline uint32_t small_ctas_per_query(uint64_t max_scored, uint32_t B) {
  uint64_t P = (max_scored + 7) / 8;  // one document per warp
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

template <int D>
__global__ void __launch_bounds__(kSmallThreads) rerank_small_kernel(const SmallParams sp) {
  const MaxSimParams& p = sp.m;
  using RL = RowLayout<D>;
  constexpr uint32_t NW = kSmallThreads / 32;
  constexpr uint32_t WBUF = kSmallWarpRowBytes;              // per-warp row staging
  constexpr uint32_t WROWS = WBUF / (2 * D);                 // rows per staged piece
  __shared__ __align__(16) float sq[32 * D];                 // query tokens (fp32, as given)
  __shared__ uint64_t keys[kSmallMaxChunk];                  // this CTA's candidate keys
  __shared__ uint64_t m_src[kSmallMaxChunk];                 // per candidate: row address (0: none)
  __shared__ uint32_t m_t[kSmallMaxChunk], m_id[kSmallMaxChunk];
  __shared__ float m_cls[kSmallMaxChunk];
  // compute phase: NW row-staging buffers; the last CTA's merge phase reuses
  // the space for the merge keys (warp 0) and the duplicate hash (warps 1-7)
  __shared__ __align__(16) uint8_t region[kSmallRegionBytes];
  __shared__ uint32_t s_last, s_ff;
  static_assert(NW * WBUF <= kSmallRegionBytes && WROWS >= 1, "row staging");
  static_assert((kSmallMergeKeys + 8) * 8 + 2 * kSmallMaxList * 4 <= kSmallRegionBytes, "merge scratch");
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t b = blockIdx.y, pc = blockIdx.x, P = sp.P;
  ktl_begin(p.dbg, 1);
  if (p.prof && tid == 0) atomicMin(&p.prof[2], ktl_now());
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
  if ((nc > (uint32_t)kSmallMaxChunk || (pc == 0 && ns > (uint64_t)kSmallMaxList)) && tid == 0) atomicOr(p.err, ERR_CAPACITY);
  const uint32_t ncs = min(nc, (uint32_t)kSmallMaxChunk);
  const uint32_t nq = p.nq;
  uint32_t ebits = 0;
  // ---- candidate metadata (one thread per candidate: id -> row_ptr pair,
  // two dependent round trips for the whole CTA) and the query, together ----
  if (tid < ncs) {
    const uint64_t j = j0 + tid, c = off0 + j;
    const uint32_t id = __ldg(&p.cand_ids[c]);
    m_id[tid] = id;
    m_cls[tid] = __ldg(&p.cand_cls[c]);
    uint64_t src = 0;
    uint32_t t = 0;
    if (j < need) {
      const uint64_t loc = shard_local(id, p.shard_count, p.shard_index, p.n_docs);
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
    for (uint32_t i = tid; i < nq * D; i += kSmallThreads) {
      const float x0 = __ldg(&qs[i]);
      const float x = p.qround ? espn_ptx::code_to_f32(espn_ptx::f32_to_code(x0, p.bf16), p.bf16) : x0;
      badq |= !isfinite(x);
      sq[i] = x;
    }
    if (badq) atomicOr(p.err, ERR_NONFINITE_QUERY);
  }
  __syncthreads();
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
  // ---- warp per candidate: MaxSim (needed prefix) + aggregate -> key ----
  for (uint32_t jj = wid; jj < ncs; jj += NW) {
    const uint64_t j = j0 + jj;
    const uint64_t src = m_src[jj];
    const uint32_t t = m_t[jj];
    float bow = 0.0f;
    const bool ok = src != 1;
    if (j < need && ok) {
      const uint8_t* doc = reinterpret_cast<const uint8_t*>(src);
      float m = -INFINITY;
      // the doc's rows in pieces of WROWS: one coalesced round trip per piece
      // into the warp's buffer (kept in the tile layout), then every lane
      // reads each row with broadcast 16-byte shared loads
      for (uint32_t r0 = 0; r0 < t; r0 += WROWS) {
        const uint32_t nr = min(WROWS, t - r0);
        const uint32_t nv = nr * RL::CH;
        __syncwarp();  // the previous piece is consumed
        for (uint32_t v = lane; v < nv; v += 32) {
          const uint32_t jr = r0 + v / RL::CH, cc = v % RL::CH;
          const uint32_t o = RL::off(t, jr, cc);
          *reinterpret_cast<uint4*>(wbuf + (jr - r0) * (2 * D) + cc * 16) = __ldg(reinterpret_cast<const uint4*>(doc + o));
        }
        __syncwarp();
        // four rows at a time: independent accumulators, each summed in
        // ascending k (the reference's order); maxima applied in row order
        uint32_t jr = 0;
        for (; jr + 4 <= nr; jr += 4) {
          float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int k8 = 0; k8 < D / 8; ++k8) {
            uint4 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = *reinterpret_cast<const uint4*>(wbuf + (jr + r) * (2 * D) + k8 * 16);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float d0 = espn_ptx::code_to_f32((uint16_t)(w[h] & 0xFFFFu), p.bf16);
                const float d1 = espn_ptx::code_to_f32((uint16_t)(w[h] >> 16), p.bf16);
                acc[r] = __fadd_rn(acc[r], __fmul_rn(q[k8 * 8 + 2 * h], d0));
                acc[r] = __fadd_rn(acc[r], __fmul_rn(q[k8 * 8 + 2 * h + 1], d1));
              }
            }
          }
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (acc[r] > m) m = acc[r];
        }
        for (; jr < nr; ++jr) {
          float acc = 0.0f;
#pragma unroll
          for (int k8 = 0; k8 < D / 8; ++k8) {
            const uint4 v = *reinterpret_cast<const uint4*>(wbuf + jr * (2 * D) + k8 * 16);
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
      }
      float s = 0.0f;
      for (uint32_t i = 0; i < nq; ++i) s = __fadd_rn(s, __shfl_sync(0xffffffffu, m, i));
      bow = s;
      if (p.bow_out && lane == 0) p.bow_out[off0 + j] = s;
    }
    if (lane == 0) {
      uint64_t key = 0;
      if (ok) {
        const float cl = m_cls[jj];
        const float sc = __fadd_rn(__fmul_rn(alpha, cl), bow);
        ebits |= !isfinite(cl) ? ERR_NONFINITE_CLS : (!isfinite(sc) ? ERR_NONFINITE_SCORE : 0u);
        key = make_key(sc, m_id[jj]);
      }
      keys[jj] = key;
    }
  }
  if (ebits) atomicOr(p.err, ebits);
  __syncthreads();
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
  for (uint32_t r = min(nz, k) + tid; r < k; r += kSmallThreads) __stcg(&mylist[r], 0ull);
  // ---- arrival; the query's last CTA finishes it ----
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&sp.arrive[b], 1u) == P - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) {
    ktl_end(p.dbg, 1);
    small_prof_end(p);
    return;
  }
  __threadfence();
  if (wid == 0) {
    uint64_t* fmk = reinterpret_cast<uint64_t*>(region);
    fused_merge<kSmallMergeKeys>(p, b, b * P, P, fmk, lane, /*kway=*/chunk < k);
  } else {
    // duplicate check over the query's scored ids (warps 1-7)
    uint32_t* hash = reinterpret_cast<uint32_t*>(region + (kSmallMergeKeys + 8) * 8);
    constexpr uint32_t HS = 2 * kSmallMaxList, HM = HS - 1;
    const uint32_t t7 = tid - 32;
    constexpr uint32_t N7 = kSmallThreads - 32;
    for (uint32_t i = t7; i < HS; i += N7) hash[i] = 0xFFFFFFFFu;
    if (t7 == 0) s_ff = 0;
    asm volatile("bar.sync 1, %0;" ::"n"(N7) : "memory");
    uint32_t dup = 0;
    const uint64_t nd = min(ns, (uint64_t)kSmallMaxList);
    for (uint64_t j = t7; j < nd; j += N7) {
      const uint32_t id = __ldg(&p.cand_ids[off0 + j]);
      if (id == 0xFFFFFFFFu) {
        dup |= atomicExch(&s_ff, 1u);
        continue;
      }
      uint32_t h = ((id * 2654435761u) >> 7) & HM;
      for (;;) {
        const uint32_t old = atomicCAS(&hash[h], 0xFFFFFFFFu, id);
        if (old == 0xFFFFFFFFu) break;
        if (old == id) { dup = 1; break; }
        h = (h + 1) & HM;
      }
    }
    if (dup) atomicOr(p.err, ERR_DUPLICATE);
  }
  if (tid == 0) sp.arrive[b] = 0u;  // every CTA of the query has arrived
  ktl_end(p.dbg, 1);
  __syncthreads();  // (the profile's end stamp after the merge and the dedup)
  small_prof_end(p);
}

template <int D>
cudaError_t launch_small(const SmallParams& sp, uint32_t B, cudaStream_t s) {
  rerank_small_kernel<D><<<dim3(sp.P, B), kSmallThreads, 0, s>>>(sp);
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
