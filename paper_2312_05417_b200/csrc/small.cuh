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
constexpr int kSmallMergeKeys = 1536;     // merge scratch (P x k keys; longer -> chunked merge)

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
  __shared__ __align__(16) float sq[32 * D];                      // query tokens (fp32, as given)
  __shared__ uint64_t keys[kSmallMaxChunk];         // this CTA's candidate keys
  __shared__ __align__(16) uint64_t fmk[kSmallMergeKeys + 8];      // last CTA: merge keys (warp 0)
  __shared__ uint32_t hash[2 * kSmallMaxList];                      // last CTA: dedup hash (warps 1-7)
  __shared__ uint32_t s_last, s_ff;
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
  // ---- query -> shared memory (only if this CTA has MaxSim work) ----
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
  uint32_t ebits = 0;
  // ---- warp per candidate: MaxSim (needed prefix) + aggregate -> key ----
  for (uint32_t jj = wid; jj < ncs; jj += kSmallThreads / 32) {
    const uint64_t j = j0 + jj, c = off0 + j;
    const uint32_t id = __ldg(&p.cand_ids[c]);
    const float cl = __ldg(&p.cand_cls[c]);
    float bow = 0.0f;
    bool ok = true;
    if (j < need) {
      const uint64_t loc = shard_local(id, p.shard_count, p.shard_index, p.n_docs);
      if (loc == ~0ull) {
        ok = false;
        ebits |= ERR_UNKNOWN_DOC;
      } else {
        const uint64_t r0 = __ldg(&p.row_ptr[loc]);
        const uint32_t t = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
        const uint8_t* doc = reinterpret_cast<const uint8_t*>(p.rows + r0 * D);
        float m = -INFINITY;
        // four rows at a time: independent accumulators, each summed in
        // ascending k (the reference's order); maxima applied in row order
        uint32_t jr = 0;
        for (; jr + 4 <= t; jr += 4) {
          float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int k8 = 0; k8 < D / 8; ++k8) {
            uint4 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = __ldg(reinterpret_cast<const uint4*>(doc + RowLayout<D>::off(t, jr + r, k8)));
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
        for (; jr < t; ++jr) {
          float acc = 0.0f;
#pragma unroll
          for (int k8 = 0; k8 < D / 8; ++k8) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(doc + RowLayout<D>::off(t, jr, k8)));
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
        for (uint32_t i = 0; i < nq; ++i) s = __fadd_rn(s, __shfl_sync(0xffffffffu, m, i));
        bow = s;
        if (p.bow_out && lane == 0) p.bow_out[c] = s;
      }
    }
    if (lane == 0) {
      uint64_t key = 0;
      if (ok) {
        const float sc = __fadd_rn(__fmul_rn(alpha, cl), bow);
        ebits |= !isfinite(cl) ? ERR_NONFINITE_CLS : (!isfinite(sc) ? ERR_NONFINITE_SCORE : 0u);
        key = make_key(sc, id);
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
    fused_merge<kSmallMergeKeys>(p, b, b * P, P, fmk, lane);
  } else {
    // duplicate check over the query's scored ids (warps 1-7)
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
