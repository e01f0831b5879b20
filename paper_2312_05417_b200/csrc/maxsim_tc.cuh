// maxsim_tc.cuh -- K2: fused gather + MaxSim on the sm_100a tensor cores.
//
// Restates maxsim_score (proj/include/espn/scoring.hpp:7-10) for
// a whole batch of (query, candidate) pairs, fused with the candidate gather of
// StoreHandle::fetch_batch (store.hpp:91-94) and with no score matrix in HBM.
//
// Mapping:
//   * A work unit is (query b, up to `unit_docs` consecutive needed candidates).
//     Each doc's t token rows occupy ceil8(t) consecutive 8-aligned "slots";
//     a stage holds 4 quarters x NQC slots.
//   * The table is stored in the HBM tile layout (RowLayout, common.cuh), so a
//     document is one contiguous byte range per K-panel that ONE 1-D
//     cp.async.bulk (TMA engine, UBLKCP) lands directly in the UMMA K-major
//     SWIZZLE_{32,64,128}B operand layout -- no per-element address math, no
//     register hop.  The pad slots of a doc's last 8-slot group get copies of
//     its last row (pad-patch warp), so no column ever needs masking.
//   * Warp roles (TcLayout): 8 epilogue, MMA issuer, 2 bulk-copy producers
//     (loader-built op lists), unit loader (ids -> row_ptr issued before the
//     slot wait; slot plan, doc-start bitmap, copy ops, pad patches), combine
//     (ordered sums), dedup + rank (fused top-k), query tile, pad patch.
//   * tcgen05.mma (M=128, N<=NQC, K=16) per quarter and K-step.  A is a 128-row
//     window over [96 zero rows | Q (32 rows) | 96 zero rows ...] whose offset
//     puts the query tokens on TMEM lanes 32w..32w+31 for quarter w
//     ("block-diagonal" A), so all four lane quarters -- and all epilogue
//     warps -- get useful work from every MMA into one accumulator buffer.
//     d = 128 uses the replicated-A mode instead (TcCfg::REPA).
//   * Epilogue warp (w, h) reads its lanes with tcgen05.ld: thread i holds
//     query token i's dot products against a 64-slot range along columns, so
//     the max over doc tokens is a register max tree per 8-slot group and a
//     branch-free doc-boundary scan; per-doc partial maxima go to SMEM (shared
//     red.max) and the combine warp sums the q maxima per doc in ascending
//     query-token order (the oracle's summation order).
#pragma once
#ifndef ESPN_PLANES
#define ESPN_PLANES 4
#endif
// 1: every lane of the loader / query / combine / rank warps arrives on the
// unit and bow-ring barriers (each lane's arrive releases its own writes);
// 0: __syncwarp + one arriving lane (A/B measurement knob)
#ifndef ESPN_ARRIVE_ALL
#define ESPN_ARRIVE_ALL 1
#endif
#include "common.cuh"
#include "ptx.cuh"

namespace espn_k {

template <int D, bool SPLIT>
struct TcCfg;
// SPLIT: the fp32 query is carried as q = hi + lo, both in the table dtype
// (hi = round(q), lo = round(q - hi)), and every K-step issues two MMAs into
// the same accumulator.  The products then carry the query at 22 (f16) / 16
// (bf16) significant bits instead of 11 / 8 -- the reference multiplies the
// fp32 query (types.hpp:33-44, scoring.hpp:7-10), and a bf16-rounded query
// alone is off by up to ~3.5e-3 relative.  The A tile doubles (lo slots after
// the hi slots), so the larger dims run fewer unit slots.
// REPA: replicated-A mode -- A = the query tile four times (no zero rows) and
// ONE MMA per K-step covers the whole stage (N = 4 x NQC); lane quarter w of
// the accumulator holds every slot, epilogue warps of quarter w read columns
// [w NQC, (w+1) NQC).  Same MAC count as the block-diagonal mode, 4x fewer
// (wider) MMA instructions and a 3x smaller A tile; needs 4 x NQC TMEM
// columns per buffer, so it is used where NQC is small (d = 128).
template <bool S> struct TcCfg<16, S>  { static constexpr int NQC = 128, NS = 6, UNITMAX = 64, NU = 3; static constexpr bool REPA = false; };
#ifndef ESPN_D32_NQC
#define ESPN_D32_NQC 128
#endif
#ifndef ESPN_NO_PATCH
#define ESPN_NO_PATCH 1  // 1: no pad-patch warp, the epilogue masks pad columns (C2 35.7 vs 36.5 us); 0: the 17-warp patch design
#endif
#ifndef ESPN_MMA_DESC
#define ESPN_MMA_DESC 0  // A/B knob: 1 = descriptors stepped per quarter instead of rebuilt per MMA
#endif
#ifndef ESPN_D32_NS
#define ESPN_D32_NS 4
#endif
#ifndef ESPN_D32_NU
#define ESPN_D32_NU 3  // unit slots in flight
#endif
#ifndef ESPN_D32_UNITMAX
#define ESPN_D32_UNITMAX 96  // docs per work unit, d = 32 rounded query (served C2: 32.9 us; 64: 35.8; 128 with NU 2: 34.0)
#endif
template <bool S> struct TcCfg<32, S>  { static constexpr int NQC = S ? 128 : ESPN_D32_NQC, NS = S ? 4 : ESPN_D32_NS, UNITMAX = S ? 64 : ESPN_D32_UNITMAX, NU = S ? 3 : ESPN_D32_NU; static constexpr bool REPA = false; };
template <bool S> struct TcCfg<64, S>  { static constexpr int NQC = 64,  NS = 3, UNITMAX = 64, NU = S ? 2 : 3; static constexpr bool REPA = false; };
template <bool S> struct TcCfg<128, S> { static constexpr int NQC = 64,  NS = 2, UNITMAX = 32, NU = S ? 1 : 2; static constexpr bool REPA = true; };

template <int D, bool SPLIT_ = false>
struct TcLayout {
  using C = TcCfg<D, SPLIT_>;
  static constexpr bool SPLIT = SPLIT_;
  using RL = RowLayout<D>;
  static constexpr int NQC = C::NQC, NS = C::NS, UNITMAX = C::UNITMAX, NU = C::NU;
  static constexpr bool REPA = C::REPA;
  static constexpr int ROWB = RL::ROWB, PW = RL::PW, NP = RL::NP;
  static constexpr uint32_t SWZ = PW == 128 ? 2u : PW == 64 ? 4u : 6u;  // UMMA layout code
  static constexpr int KSTEPS = D / 16;
  static constexpr int STAGE_SLOTS = 4 * NQC;
  static constexpr int PANEL_BYTES = STAGE_SLOTS * PW;  // one K-panel of a stage
  static constexpr int STAGE_BYTES = NP * PANEL_BYTES;
  // A (query) operand: the same K-major swizzled panel layout as the rows
  // (RowLayout with t = A_ROWS), so the tensor core reads A conflict-free
  static constexpr int CH = D / 8;                 // 16-byte chunks per query row
  static constexpr int LO_ROWS = NU * 128;         // SPLIT: lo slots start LO_ROWS rows after the hi slots
  static constexpr int A_ROWS = (REPA ? 0 : 96) + (SPLIT ? 2 : 1) * NU * 128;  // zeros | Q0 | zeros | Q1 | ... (REPA: Q0 x4 | Q1 x4 ...)
  static constexpr int A_PANEL_BYTES = A_ROWS * PW;
  static constexpr int A_BYTES = NP * A_PANEL_BYTES;
  static constexpr int MAX_SLOTS = UNITMAX * 64;   // slot budget of one unit
  static constexpr int NG = MAX_SLOTS / 8;         // 8-slot groups
  static constexpr int MAXW = NG / 32;             // bitmap words (one bit per group)
  static constexpr int MAX_STAGES = MAX_SLOTS / STAGE_SLOTS;  // stages of a full unit
  static constexpr int MAX_OPS = (UNITMAX + MAX_STAGES) * NP;  // docs + stage straddles, per K-panel
  static constexpr int PM_STRIDE = UNITMAX + 1;    // padded: conflict-free emits and combine
  static constexpr int PM_FLOATS = NU * 32 * PM_STRIDE;  // per unit slot: [query token][doc] keys
  static constexpr int BUFC = REPA ? 4 * NQC : NQC;  // TMEM columns per accumulator buffer
  static constexpr int NBUF = (512 / BUFC) < 4 ? (512 / BUFC) : 4;
  static constexpr uint32_t TMEM_COLS = NBUF * BUFC <= 32 ? 32 : NBUF * BUFC <= 64 ? 64
                                      : NBUF * BUFC <= 128 ? 128 : NBUF * BUFC <= 256 ? 256 : 512;
  static constexpr int NPROD = 2;                  // bulk-copy producer warps
  static constexpr int PLANES = ESPN_PLANES;       // issuing lanes per producer warp
  static constexpr int NEPI = 8;                   // epilogue warps: 4 lane quarters x 2 column halves
#ifndef ESPN_MMA_WARP_LATE
  static constexpr int MMA_WARP = NEPI;
  static constexpr int PROD_WARP0 = NEPI + 1;
  static constexpr int LOADER_WARP = PROD_WARP0 + NPROD;
  static constexpr int COMBINE_WARP = LOADER_WARP + 1;
#else
  // A/B knob: the MMA warp on SM sub-partition 3 (warp % 4), beside the
  // lightest roles (query tile, epilogue quarter 3)
  static constexpr int PROD_WARP0 = NEPI;
  static constexpr int LOADER_WARP = PROD_WARP0 + NPROD;
  static constexpr int MMA_WARP = LOADER_WARP + 1;
  static constexpr int COMBINE_WARP = MMA_WARP + 1;
#endif
  static constexpr int DEDUP_WARP = COMBINE_WARP + 1;  // fused top-k: duplicate check
  static constexpr int RANK_WARP = DEDUP_WARP + 1;     // fused top-k: keys, unit top-k
  static constexpr int QUERY_WARP = RANK_WARP + 1;     // unit query tile -> A operand slot
  static constexpr int PATCH_WARP = QUERY_WARP + 1;    // pad slots <- copies of the doc's last row
  static constexpr int NWARPS = ESPN_NO_PATCH ? PATCH_WARP : PATCH_WARP + 1;  // (no pad-patch warp: 16)
  static constexpr int NB = 8;                     // bow ring (combine -> rank) depth, in units
  static constexpr int HALF = NQC / 2;             // columns per epilogue warp per stage
#ifndef ESPN_EPI_LW
#define ESPN_EPI_LW 32  // A/B knob: columns per tcgen05.ld of the epilogue (64 = one load per stage half)
#endif
  static constexpr int LW = HALF < ESPN_EPI_LW ? HALF : ESPN_EPI_LW; // tcgen05.ld width (columns)
  static constexpr int NLD = HALF / LW;            // loads per epilogue warp per stage
  static constexpr int NGH = HALF / 8;             // 8-slot groups per epilogue warp per stage
  static constexpr int NTHREADS = NWARPS * 32;
  static constexpr int MAXREG = NWARPS <= 16 ? 120 : 96;  // see maxsim_tc_kernel

  struct Unit {
    uint32_t b, nd, S, tail;   // tail: alpha*cls tail unit (no MaxSim)
    uint64_t cfirst;            // candidate index of the unit's first doc
    uint32_t bitmap[MAXW];      // bit g: a doc starts at group g
    uint32_t wprefix[MAXW];     // docs starting before word w
    // Pad patches (loader-built): for each doc whose last 8-slot group is
    // partial, {stage-relative slot of its last row | pad count << 16 |
    // stage << 20}, in stage order.
    uint32_t pt[UNITMAX];
    uint32_t n_pt;
#if ESPN_NO_PATCH
    uint8_t vc[NG];             // per 8-slot group: its valid (non-pad) slots
#endif
    // Bulk-copy plan (loader-built): one op per (doc, stage piece, K-panel)
    // {src lo, src hi, byte offset in the stage, bytes}, in stage order;
    // stage st issues ops [op_beg[st], op_beg[st+1]) (last stage: to n_ops),
    // producer pw the ops of parity pw, expecting stage_tx[st][pw] bytes.
    uint4 op[MAX_OPS];
    uint32_t op_beg[MAX_STAGES];
    uint32_t stage_tx[MAX_STAGES][2];
    uint32_t n_ops;
  };
  // Byte offsets inside dynamic shared memory (1024-aligned base).
  static constexpr int OFF_B = 0;
  static constexpr int OFF_A = OFF_B + NS * STAGE_BYTES;
  static constexpr int OFF_PM = OFF_A + A_BYTES;
  static constexpr int OFF_UNIT = OFF_PM + PM_FLOATS * 4;
  static constexpr int OFF_UK = (OFF_UNIT + NU * (int)sizeof(Unit) + 15) / 16 * 16;  // rank warp: unit keys
  static constexpr int OFF_RING = OFF_UK + UNITMAX * 8;
  static constexpr int OFF_BAR = OFF_RING + NB * UNITMAX * 4;
  static constexpr int N_BARS = 3 * NS + 2 * NBUF + 3 * NU + 2 * NB;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int MERGE_KEYS = 640;           // persistent server: the dedup warp's merge scratch
  static constexpr int OFF_FM = (OFF_TMEM + 16 + 15) / 16 * 16;
  // persistent server: the CTA's batch gate -- a 4-deep ring of batch
  // descriptors copied from the global queue by the loader warp, and
  // {published count, stop marker, per-ring-slot finished-warp counts}
  static constexpr int DESC_RING = 4;
  static constexpr int OFF_DESC = OFF_FM + MERGE_KEYS * 8;
  static constexpr int OFF_GATE = OFF_DESC + DESC_RING * (int)sizeof(MaxSimParams);
  static constexpr int SMEM_BYTES = OFF_GATE + 32 + 1024;  // + alignment slack
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(UNITMAX % 32 == 0, "the rank and combine warps hold UNITMAX / 32 docs per lane");
  static_assert(STAGE_BYTES % 1024 == 0 && A_BYTES % 16 == 0, "alignment");
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// ---- fused top-k helpers (combine warp) --------------------------------------
// Duplicate rejection of rank() (scoring.hpp:16-18) across all units of a
// query, by the dedicated dedup warp: the unit's ids go into the query's
// open-addressing hash in global memory (L2-resident, atomicCAS, 0xFFFFFFFF =
// empty; that id itself is tracked by ff_seen).  The table is sized 8x the
// list, so nearly every insert lands on its first probe; a lane's CAS are
// issued together.  The query's last arrival clears it (fused_merge).
template <int NK>
__device__ __forceinline__ void fused_dedup(const MaxSimParams& p, uint32_t par, uint32_t b, uint64_t cfirst,
                                            uint32_t nd, uint32_t lane) {
  uint32_t* tab = p.dedup + ((size_t)par * p.max_queries + b) * p.hash_slots;
  uint32_t* ff = p.ff_seen + (size_t)par * p.max_queries + b;
  const uint32_t mask = p.hash_slots - 1;
  uint32_t id[NK], h[NK], pend = 0, dup = 0, full = 0;
#pragma unroll
  for (int r = 0; r < NK; ++r) {
    const uint32_t k = r * 32 + lane;
    id[r] = k < nd ? __ldcg(&p.cand_ids[cfirst + k]) : 0u;
    h[r] = ((id[r] * 2654435761u) >> 7) & mask;
    if (k < nd) {
      if (id[r] == 0xFFFFFFFFu) dup |= atomicExch(ff, 1u);
      else pend |= 1u << r;
    }
  }
  for (uint32_t probe = 0; pend; ++probe) {
    uint32_t old[NK];
#pragma unroll
    for (int r = 0; r < NK; ++r) old[r] = (pend >> r) & 1u ? atomicCAS(&tab[h[r]], 0xFFFFFFFFu, id[r]) : 0u;
#pragma unroll
    for (int r = 0; r < NK; ++r) {
      if (!((pend >> r) & 1u)) continue;
      if (old[r] == 0xFFFFFFFFu || old[r] == id[r]) {
        dup |= old[r] == id[r];
        pend &= ~(1u << r);
      } else {
        h[r] = (h[r] + 1) & mask;
      }
    }
    if (probe >= mask) { full = 1; break; }  // table full: a longer list than the workspace's max_list
  }
  if (dup) atomicOr(p.err, ERR_DUPLICATE);
  if (full) atomicOr(p.err, ERR_CAPACITY);
}

// The query's last arrival: merge the units' best-k lists (unit_top, each
// sorted descending, 0 = empty) into the final ranked list, then reset the
// query's counters.  Keys are unique (duplicate ids are an
// error), so the final list is "every key whose rank (number of greater keys)
// is < k".  With all n = nu*k keys staged in shared memory:
//   * threshold T = max over lists of its k-th key: a key below T has at
//     least k greater keys, so only keys >= T are candidates (about 2k);
//   * candidates are compacted in place (ballot prefix), each lane counts
//     the candidates greater than its own, and writes it at its rank.
// Longer inputs (n > FMK) fall back to a chunked k-way merge (k rounds of
// warp max over list heads).
// `kway`: always the k-way merge -- for many SHORT lists (fewer than k
// entries each, e.g. the single-launch small-batch kernel's per-CTA lists)
// every list's k-th key is empty, the threshold is 0 and the counting rank
// would be quadratic in the number of keys.
template <int FMK>
__device__ __forceinline__ void fused_merge(const MaxSimParams& p, uint32_t b, uint32_t u0, uint32_t nu,
                                            uint64_t* fm, uint32_t lane, bool kway = false) {
  const uint32_t kk = p.k;
  const unsigned long long* src = p.unit_top + (size_t)u0 * kk;
  const uint32_t n = nu * kk;
  uint32_t cnt = 0;
  if (!kway && n + 8 <= (uint32_t)FMK) {
    const unsigned long long tf0 = ktl_now();
    uint64_t th = 0;
    for (uint32_t i0 = 0; i0 < n; i0 += 256) {  // 8 loads per lane in flight
      uint64_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        v[u] = i < n ? __ldcg(&src[i]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        if (i < n) {
          fm[i] = v[u];
          if (i % kk == kk - 1 && v[u] > th) th = v[u];
        }
      }
    }
    th = warp_max_key(th);
    __syncwarp();
    const unsigned long long tf1 = ktl_now();
    uint32_t nc = 0;
    {  // compact candidates (v >= th, v != 0) to fm[0, nc)
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint64_t v = i < n ? fm[i] : 0ull;
      const bool c = v != 0 && v >= th;
      const uint32_t bal = __ballot_sync(0xffffffffu, c);
      __syncwarp();
      if (c) fm[nc + __popc(bal & ((1u << lane) - 1u))] = v;
      nc += __popc(bal);
      __syncwarp();
    }
    for (uint32_t i0 = 0; i0 < nc; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint64_t v = i < nc ? fm[i] : ~0ull;
      uint32_t rk = 0;
      for (uint32_t j0 = 0; j0 < nc; j0 += 8) {  // 8 independent broadcast loads per step
        uint64_t x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = fm[j0 + u];  // fm has >= nc + 8 slots (FMK >= n + 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) rk += (j0 + u < nc && x[u] > v) ? 1u : 0u;
      }
      if (i < nc && rk < kk) {
        p.out_ids[(size_t)b * kk + rk] = ~(uint32_t)(v & 0xFFFFFFFFu);
        p.out_scores[(size_t)b * kk + rk] = order_float((uint32_t)(v >> 32));
      }
    }
    }
    cnt = min(nc, kk);
    if ((p.dbg & 256u) && lane == 0) {
      atomicAdd(&g_fin[0], tf1 - tf0);
      atomicAdd(&g_fin[1], ktl_now() - tf1);
      atomicAdd(&g_fin[2], 1ull);
      atomicAdd(&g_fin[3], nc);
    }
  } else {
    // chunks of up to 63 unit lists plus the running result (list 0); lane l
    // owns lists l and l+32 and keeps their heads in registers
    const uint32_t lpc = min(64u, (uint32_t)FMK / kk);
    uint64_t mine = 0;  // lane r < cnt: the r-th best so far
    for (uint32_t l0 = 0; l0 < nu; l0 += lpc - 1) {
      const uint32_t nl = min(lpc - 1, nu - l0) + 1;
      if (lane < kk) fm[lane] = mine;
      const uint32_t nk = (nl - 1) * kk;
      for (uint32_t i0 = 0; i0 < nk; i0 += 256) {  // 8 loads per lane in flight
        uint64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0 + u * 32 + lane;
          v[u] = i < nk ? __ldcg(&src[(size_t)l0 * kk + i]) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0 + u * 32 + lane;
          if (i < nk) fm[kk + i] = v[u];
        }
      }
      __syncwarp();
      uint32_t c0 = 0, c1 = 0;  // cursors of lists lane, lane + 32
      uint64_t h0 = lane < nl ? fm[lane * kk] : 0ull;
      uint64_t h1 = lane + 32 < nl ? fm[(lane + 32) * kk] : 0ull;
      uint32_t c = 0;
      for (; c < kk; ++c) {
        const uint64_t lb = h0 > h1 ? h0 : h1;
        const uint64_t m = warp_max_key(lb);
        if (m == 0) break;
        if (lane == c) mine = m;
        const uint32_t win = __ffs(__ballot_sync(0xffffffffu, lb == m)) - 1;
        if (lane == win) {
          if (h0 == m) {
            ++c0;
            h0 = c0 < kk ? fm[lane * kk + c0] : 0ull;
          } else {
            ++c1;
            h1 = c1 < kk ? fm[(lane + 32) * kk + c1] : 0ull;
          }
        }
      }
      if (lane >= c) mine = 0;
      cnt = c;
      __syncwarp();
    }
    if (lane < cnt) {
      p.out_ids[(size_t)b * kk + lane] = ~(uint32_t)(mine & 0xFFFFFFFFu);
      p.out_scores[(size_t)b * kk + lane] = order_float((uint32_t)(mine >> 32));
    }
  }
  if (lane == 0) p.out_counts[b] = cnt;
  __syncwarp();
}

// Fused top-k, last step: one warp per query merges its units' best-k lists
// (fused_merge) into the ranked output.
// Launched as a programmatic dependent of the MaxSim kernel: its CTAs are
// resident (waiting) as MaxSim CTAs retire, and the wait releases when the
// whole MaxSim grid -- every unit list and every dedup insert -- is done.
constexpr int kFinalizeWarps = 4;
constexpr int kFinalizeKeys = 640;  // per-warp merge scratch (keys)
__global__ void __launch_bounds__(kFinalizeWarps * 32) finalize_kernel(const MaxSimParams p) {
  __shared__ uint64_t fmk[kFinalizeWarps][kFinalizeKeys];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t b = blockIdx.x * kFinalizeWarps + w;
  ktl_begin(p.dbg, 2);
  // the plan completed before MaxSim released this grid: its outputs can be
  // read before the wait
  uint32_t u0 = 0, nu = 0;
  if (b < p.n_queries) {
    u0 = p.unit_off[b];
    nu = p.unit_off[b + 1] - u0;
  }
  const uint32_t rejected = *p.err & (ERR_BAD_OFFSETS | ERR_CAPACITY);
  const unsigned long long tw0 = ktl_now();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if ((p.dbg & 256u) && lane == 0) { atomicAdd(&g_fin[4], ktl_now() - tw0); atomicAdd(&g_fin[5], tw0); }
  if (rejected) return;  // plan rejected the batch
  if (b < p.n_queries && nu > 0) fused_merge<kFinalizeKeys>(p, b, u0, nu, fmk[w], lane);
  ktl_end(p.dbg, 2);
}

// Shared-memory views and barrier set of one MaxSim CTA.
template <int D, bool SPLIT>
struct TcSmem {
  uint8_t* sB;
  uint8_t* sA;
  float* pm;
  typename TcLayout<D, SPLIT>::Unit* units;
  uint8_t* smem;
  uint64_t* full_bar;     // [NS]  producer (expect_tx) -> MMA
  uint64_t* empty_bar;    // [NS]  MMA commit -> producer
  uint64_t* tfull_bar;    // [NBUF] MMA commit -> epilogue
  uint64_t* tempty_bar;   // [NBUF] epilogue -> MMA
  uint64_t* ufull_bar;    // [NU] loader + query warp -> producer, MMA, epilogue, patch
  uint64_t* uempty_bar;   // [NU] combine -> loader / query warp
  uint64_t* edone_bar;    // [NU] epilogue (all lanes) -> combine
  uint64_t* bdone_bar;    // [NB] combine -> rank (bow ring entry full)
  uint64_t* bfree_bar;    // [NB] rank -> combine (bow ring entry free)
  uint64_t* patched_bar;  // [NS] patch warp -> MMA (stage rows + pads ready)
  uint32_t tmem_base;
};

// Pipeline position of one warp role, carried across the batches of a
// persistent launch: gu = unit iterations done (unit slot us = gu % NU and the
// slot barriers' phase), gs = stages done (stage / TMEM buffer and phases),
// rot = the round-robin origin (the next batch's unit 0 goes to CTA rot,
// so units spread over the CTAs across batches, not only within one).
struct TcRoleState {
  uint32_t gu = 0, gs = 0, rot = 0;
};

// One batch through every warp role of the CTA (the body of the MaxSim
// kernel; a persistent launch runs it once per queued batch).  `slot` != NULL:
// persistent mode -- the rank and dedup warps report the batch done and the
// dedup warps merge the queries' unit lists (instead of finalize_kernel).
template <int D, bool SPLIT>
__device__ __forceinline__ void tc_batch(const MaxSimParams& p, const TcSmem<D, SPLIT>& S, TcRoleState& rs,
                                         ServerSlot* slot, uint32_t seq) {
  using L = TcLayout<D, SPLIT>;
  using namespace espn_ptx;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t G = gridDim.x;
  const uint32_t n_units = slot ? __ldcg(p.n_units) : *p.n_units;  // planned on the device (plan_kernel)
  const uint32_t first = (blockIdx.x + G - rs.rot) % G;
  const uint32_t cnt = n_units > first ? (n_units - first + G - 1) / G : 0u;  // this CTA's units
  const uint32_t gu0 = rs.gu;
  rs.gu += cnt;
  rs.rot = (uint32_t)(((uint64_t)rs.rot + n_units) % G);
  typename L::Unit* units = S.units;
  uint8_t* smem = S.smem;
  // ESPN_DEBUG bit 8: per warp, cycles of this batch and cycles spent waiting
  // on mbarriers, summed over all CTAs into g_cta_prof[2 * warp + {0, 1}]
  // (tools/role_profile.py) -- which role is the bottleneck
#ifdef ESPN_ROLE_PROFILE  // opt-in build (tools/role_profile.py): even unexecuted, it costs ~15% on C2
  const bool tr = (p.dbg & 8u) != 0;
#else
  constexpr bool tr = false;
#endif
  unsigned long long wacc = 0;
  const long long tb0 = tr ? clock64() : 0;
  // (and per barrier kind: g_cta_prof[64 + 12 * warp + kind], kind = the
  // barrier array: full, empty, tfull, tempty, ufull, uempty, edone, bdone,
  // bfree, patched)
  auto bar_kind = [&](const uint64_t* bar) -> int {
    const int i = (int)(bar - S.full_bar);
    constexpr int e0 = L::NS, e1 = e0 + L::NS, e2 = e1 + L::NBUF, e3 = e2 + L::NBUF, e4 = e3 + L::NU,
                  e5 = e4 + L::NU, e6 = e5 + L::NU, e7 = e6 + L::NB, e8 = e7 + L::NB;
    return i < e0 ? 0 : i < e1 ? 1 : i < e2 ? 2 : i < e3 ? 3 : i < e4 ? 4 : i < e5 ? 5 : i < e6 ? 6 : i < e7 ? 7
         : i < e8 ? 8 : 9;
  };
#define ESPN_WAIT(bar, par)                                                        \
  do {                                                                             \
    if (tr) {                                                                      \
      const long long t0_ = clock64();                                             \
      espn_ptx::mbar_wait(bar, par);                                               \
      const unsigned long long dt_ = (unsigned long long)(clock64() - t0_);        \
      wacc += dt_;                                                                 \
      if (lane == 0) atomicAdd(&g_cta_prof[64 + 12 * warp + bar_kind(bar)], dt_); \
    } else {                                                                       \
      espn_ptx::mbar_wait(bar, par);                                               \
    }                                                                              \
  } while (0)

  if (warp == L::LOADER_WARP) {
    // ============================ UNIT LOADER ===================================
    // (Software-pipelining the three dependent metadata round trips across
    // units -- unit table of it+2, ids of it+1, row_ptr of it in one go -- was
    // measured: the loader's busy share fell from 91 to 84 % but the step did
    // not get faster, 37.5 vs 37.1 us; tools/role_profile.py.)
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t ug = first + it * G, gi = gu0 + it;
      const uint32_t us = gi % L::NU;
      typename L::Unit& U = units[us];
      // Unit table entry (device-planned): query b, doc count, first candidate.
      const uint4 ue = __ldcg(&p.unit_tab[ug]);
      const uint32_t b = ue.x, nd = ue.y & 0xFFu, tail = ue.y >> 31;
      const uint64_t cfirst = (uint64_t)ue.z | ((uint64_t)ue.w << 32);
      // Every global load of the unit is issued before waiting for its slot:
      // candidate ids (<= 2 per lane), then the dependent row_ptr / staged
      // addresses, so the slot wait overlaps their latency.  Per-batch inputs
      // use L2-coherent loads: a persistent CTA outlives the batch's buffers.
      constexpr int NK = L::UNITMAX / 32;
      uint32_t tk[NK];
      uint64_t srck[NK];
#pragma unroll
      for (int r = 0; r < NK; ++r) {
        const uint32_t k = r * 32 + lane;
        tk[r] = 0;
        srck[r] = 0;
        if (k < nd && !tail) {
          const uint64_t loc = shard_local(__ldcg(&p.cand_ids[cfirst + k]), p.shard_count, p.shard_index, p.n_docs);
          if (loc != ~0ull) {
            const uint64_t r0 = __ldg(&p.row_ptr[loc]);
            tk[r] = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
            srck[r] = p.cand_src ? __ldcg(&p.cand_src[cfirst + k])  // tiered: staged / resident address
                                 : (uint64_t)(p.rows + r0 * D);
            if (srck[r] == 0) tk[r] = 0;  // not staged (staging overflow, reported by stage_kernel)
          } else {
            atomicOr(p.err, ERR_UNKNOWN_DOC);
          }
        }
      }
      ESPN_WAIT(&S.uempty_bar[us], ((gi / L::NU) & 1) ^ 1);
      for (int i = lane; i < L::MAXW; i += 32) U.bitmap[i] = 0;
      for (int i = lane; i < L::MAX_STAGES; i += 32) {
        U.op_beg[i] = 0xFFFFFFFFu;
        U.stage_tx[i][0] = 0;
        U.stage_tx[i][1] = 0;
      }
      __syncwarp();
      // doc info + slot prefix sum (warp scan) + group plan + copy ops
      uint32_t carry = 0, ocarry = 0, pcarry = 0;
#pragma unroll
      for (int r = 0; r < NK; ++r) {
        const uint32_t k = r * 32 + lane;
        const uint32_t t = tk[r];
        const uint64_t srcaddr = srck[r];
        const uint32_t pad = (t + 7u) & ~7u;
        uint32_t incl = pad;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const uint32_t start = carry + incl - pad;
        const bool fits = k < nd && t > 0 && start + pad <= (uint32_t)L::MAX_SLOTS;
        const uint32_t st0 = start / L::STAGE_SLOTS, st1 = fits ? (start + t - 1) / L::STAGE_SLOTS : st0;
        const uint32_t npc = fits ? (st1 - st0 + 1) * L::NP : 0u;  // copy ops of this doc
        uint32_t oincl = npc;
        const uint32_t npt = (fits && pad != t) ? 1u : 0u;  // pad patch of this doc
        uint32_t pincl = npt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, oincl, o);
          const uint32_t vp = __shfl_up_sync(0xffffffffu, pincl, o);
          if (lane >= o) { oincl += v; pincl += vp; }
        }
        if (fits) {
          atomicOr(&U.bitmap[start >> 8], 1u << ((start >> 3) & 31));
          if (npt) {  // the doc's last row and its pads share one 8-slot group, one stage
            const uint32_t last = start + t - 1, stl = last / L::STAGE_SLOTS;
            const uint32_t pi = pcarry + pincl - 1;
            U.pt[pi] = (last - stl * L::STAGE_SLOTS) | ((pad - t) << 16) | (stl << 20);
          }
#if ESPN_NO_PATCH
          {
            const uint32_t g0 = start >> 3, ngr = pad >> 3;
            for (uint32_t gg = 0; gg + 1 < ngr; ++gg) U.vc[g0 + gg] = 8;
            U.vc[g0 + ngr - 1] = (uint8_t)(t - 8 * (ngr - 1));
          }
#endif
          // one op per stage piece and K-panel: the piece [a, e) of the doc's
          // slots inside stage st lands at (a - x0) * PW of panel pn
          uint32_t o = ocarry + oincl - npc;
          for (uint32_t st = st0; st <= st1; ++st) {
            const uint32_t x0 = st * L::STAGE_SLOTS;
            const uint32_t a = max(start, x0), e = min(start + t, x0 + L::STAGE_SLOTS);
            const uint32_t ja = a - start, nb = (e - a) * (uint32_t)L::PW;
            atomicMin(&U.op_beg[st], o);
#pragma unroll
            for (int pn = 0; pn < L::NP; ++pn, ++o) {
              const uint64_t src = srcaddr + ((uint64_t)pn * t + ja) * L::PW;
              U.op[o] = make_uint4((uint32_t)src, (uint32_t)(src >> 32), pn * L::PANEL_BYTES + (a - x0) * L::PW, nb);
              atomicAdd(&U.stage_tx[st][o & 1u], nb);
            }
          }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
        ocarry += __shfl_sync(0xffffffffu, oincl, 31);
        pcarry += __shfl_sync(0xffffffffu, pincl, 31);
      }
      if (carry > (uint32_t)L::MAX_SLOTS) {
        if (lane == 0) atomicOr(p.err, ERR_UNIT_TOO_LARGE);
        carry = 0;  // skip the unit's MMA work; the call fails on the host
      }
      __syncwarp();
      if (lane == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < L::MAXW; ++i) {
          U.wprefix[i] = acc;
          acc += __popc(U.bitmap[i]);
        }
        U.b = b;
        U.cfirst = cfirst;
        U.nd = nd;
        U.S = carry;
        U.tail = tail;
        U.n_ops = ocarry;
        U.n_pt = pcarry;
      }
      __syncwarp();
      if (ESPN_ARRIVE_ALL || lane == 0) mbar_arrive(&S.ufull_bar[us]);  // every lane releases its own writes
    }
  } else if (warp == L::PATCH_WARP && !ESPN_NO_PATCH) {
    // ============================ PAD PATCH =====================================
    // Once a stage's rows have landed, every doc whose last 8-slot group is
    // partial gets copies of its last row in its pad slots (re-swizzled for
    // the slot), so each MMA column of a group is a real row of its doc and
    // the epilogue's group maxima need no masking.  One lane per doc.
    uint32_t& gs = rs.gs;
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t gi = gu0 + it, us = gi % L::NU;
      const typename L::Unit& U = units[us];
      ESPN_WAIT(&S.ufull_bar[us], (gi / L::NU) & 1);
      const uint32_t Sl = U.S, npt = U.n_pt;
      const uint32_t n_st = (Sl + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      uint32_t pc = 0;  // next patch of the unit (patches are in stage order)
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t s = gs % L::NS;
        ESPN_WAIT(&S.full_bar[s], (gs / L::NS) & 1);
        uint8_t* stage = S.sB + s * L::STAGE_BYTES;
        for (;;) {
          const uint32_t i = pc + lane;
          const uint32_t e = i < npt ? U.pt[i] : 0xFFFFFFFFu;
          const bool mine = i < npt && (e >> 20) == st;
          const uint32_t nmine = __popc(__ballot_sync(0xffffffffu, mine));  // a prefix of the lanes
          if (mine) {
            const uint32_t sl = e & 0xFFFFu, npad = (e >> 16) & 0xFu;
            const uint32_t sws = ((sl * (uint32_t)L::PW) >> 7) & (uint32_t)(L::RL::CPP - 1);
#pragma unroll
            for (int pn = 0; pn < L::NP; ++pn) {
              uint8_t* panel = stage + pn * L::PANEL_BYTES;
              uint4 c[L::RL::CPP];
#pragma unroll
              for (int cc = 0; cc < L::RL::CPP; ++cc)
                c[cc] = *reinterpret_cast<const uint4*>(panel + sl * L::PW + ((cc ^ sws) << 4));
              for (uint32_t r = 1; r <= npad; ++r) {
                const uint32_t ds = sl + r;
                const uint32_t swd = ((ds * (uint32_t)L::PW) >> 7) & (uint32_t)(L::RL::CPP - 1);
#pragma unroll
                for (int cc = 0; cc < L::RL::CPP; ++cc)
                  *reinterpret_cast<uint4*>(panel + ds * L::PW + ((cc ^ swd) << 4)) = c[cc];
              }
            }
          }
          pc += nmine;
          if (nmine < 32) break;
        }
        fence_proxy_async_smem();  // patched rows are read by the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.patched_bar[s]);
      }
    }
  } else if (warp == L::QUERY_WARP) {
    // ============================ QUERY TILE ====================================
    // The unit's query tokens -> A slot `us` (hi, and lo when SPLIT), in the
    // table dtype, in parallel with the loader's slot plan (ufull counts both).
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t ug = first + it * G, gi = gu0 + it, us = gi % L::NU;
      const uint4 ue = __ldcg(&p.unit_tab[ug]);
      const uint32_t b = ue.x, tail = ue.y >> 31;
      ESPN_WAIT(&S.uempty_bar[us], ((gi / L::NU) & 1) ^ 1);
      // Query tokens -> A slot `us` (rows 96+128*us .. +32), converted to the
      // table dtype; rows >= nq stay zero.  Item e = (row i, 8-value chunk c);
      // batches of 4 items per lane keep all their loads in flight together.
      if (!tail) {
        const float* q = p.q32 + (size_t)b * p.nq * D;
        const int abase = (L::REPA ? 0 : 96) + 128 * (int)us;
        constexpr int ITEMS = 32 * L::CH / 32;  // per lane
        constexpr int BATCH = ITEMS < 4 ? ITEMS : 4;
#pragma unroll
        for (int i0 = 0; i0 < ITEMS; i0 += BATCH) {
          float4 x[BATCH][2];
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            const int e = (i0 + u) * 32 + lane;
            const int i = e / L::CH, c = e % L::CH;
            if ((uint32_t)i < p.nq) {
              const float4* src = reinterpret_cast<const float4*>(q + i * D + c * 8);
              x[u][0] = __ldcg(src);
              x[u][1] = __ldcg(src + 1);
            } else {
              x[u][0] = x[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          bool bad = false;
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            const int e = (i0 + u) * 32 + lane;
            const int i = e / L::CH, c = e % L::CH;
            const float f[8] = {x[u][0].x, x[u][0].y, x[u][0].z, x[u][0].w,
                                x[u][1].x, x[u][1].y, x[u][1].z, x[u][1].w};
            uint32_t w4[4], l4[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint16_t h0 = f32_to_code(f[2 * h], p.bf16), h1 = f32_to_code(f[2 * h + 1], p.bf16);
              const float r0 = code_to_f32(h0, p.bf16), r1 = code_to_f32(h1, p.bf16);
              bad |= !isfinite(r0) || !isfinite(r1);
              w4[h] = (uint32_t)h0 | ((uint32_t)h1 << 16);
              if constexpr (L::SPLIT) {  // residuals (exact in fp32), rounded to the dtype
                const uint16_t l0 = f32_to_code(__fsub_rn(f[2 * h], r0), p.bf16);
                const uint16_t l1 = f32_to_code(__fsub_rn(f[2 * h + 1], r1), p.bf16);
                l4[h] = (uint32_t)l0 | ((uint32_t)l1 << 16);
              }
            }
            const int r = abase + i;
#pragma unroll
            for (int part = 0; part < (L::SPLIT ? 2 : 1); ++part) {
              const uint4 val = part ? make_uint4(l4[0], l4[1], l4[2], l4[3]) : make_uint4(w4[0], w4[1], w4[2], w4[3]);
              const int rr = r + part * L::LO_ROWS;
              *reinterpret_cast<uint4*>(S.sA + L::RL::off(L::A_ROWS, rr, c)) = val;
              if constexpr (L::REPA) {  // replicas for lane quarters 1..3
#pragma unroll
                for (int rq = 1; rq < 4; ++rq)
                  *reinterpret_cast<uint4*>(S.sA + L::RL::off(L::A_ROWS, rr + 32 * rq, c)) = val;
              }
            }
          }
          if (bad) atomicOr(p.err, ERR_NONFINITE_QUERY);
        }
      }
      fence_proxy_async_smem();  // A tile is read by the tensor core (async proxy)
      __syncwarp();
      if (ESPN_ARRIVE_ALL || lane == 0) mbar_arrive(&S.ufull_bar[us]);
    }
  } else if (warp >= L::PROD_WARP0 && warp < L::PROD_WARP0 + L::NPROD) {
    // ====================== BULK-COPY PRODUCERS (NPROD warps) ======================
    // PLANES lanes of producer pw issue the stage's copy ops of parity pw (one
    // cp.async.bulk each, planned by the loader); lane 0 arms the stage's full
    // barrier with their byte count.
    const uint32_t pw = warp - L::PROD_WARP0;
    const uint64_t policy = l2_policy_evict_first();
    uint32_t& gs = rs.gs;
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t gi = gu0 + it, us = gi % L::NU;
      const typename L::Unit& U = units[us];
      ESPN_WAIT(&S.ufull_bar[us], (gi / L::NU) & 1);
      const uint32_t Sl = U.S;
      const uint32_t n_st = (Sl + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t s = gs % L::NS;
        // ops [o0, o1) of this stage (loader-planned); this warp issues parity pw
        const uint32_t o0 = U.op_beg[st], o1 = st + 1 < n_st ? U.op_beg[st + 1] : U.n_ops;
        uint32_t bytes = U.stage_tx[st][pw];
        ESPN_WAIT(&S.empty_bar[s], ((gs / L::NS) & 1) ^ 1);
        if (p.dbg & 4u) bytes = 0;
        if (lane == 0) mbar_arrive_expect_tx(&S.full_bar[s], bytes);
        __syncwarp();
        if (!(p.dbg & 4u) && lane < L::PLANES) {
          const uint32_t sbase = smem_u32(S.sB + s * L::STAGE_BYTES);
          for (uint32_t o = o0 + ((o0 & 1u) ^ pw) + 2 * lane; o < o1; o += 2 * L::PLANES) {
            const uint4 op = U.op[o];
            bulk_g2s(sbase + op.z, reinterpret_cast<const void*>((uint64_t)op.x | ((uint64_t)op.y << 32)), op.w,
                     &S.full_bar[s], policy);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == L::MMA_WARP) {
    // ============================ MMA ISSUER ==================================
    // The whole warp walks the schedule (operands warp-uniform, in uniform
    // registers); one elected lane issues each tcgen05.mma / commit.
    uint32_t& gs = rs.gs;
    const uint32_t a_base = smem_u32(S.sA), b_base = smem_u32(S.sB);
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t gi = gu0 + it, us = gi % L::NU;
      ESPN_WAIT(&S.ufull_bar[us], (gi / L::NU) & 1);
      const uint32_t Sl = units[us].S;
      const uint32_t n_st = (Sl + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t s = gs % L::NS, buf = gs % L::NBUF;
#if ESPN_NO_PATCH
        ESPN_WAIT(&S.full_bar[s], (gs / L::NS) & 1);  // rows landed (pads masked by the epilogue)
#else
        ESPN_WAIT(&S.patched_bar[s], (gs / L::NS) & 1);  // rows landed and pads patched
#endif
        ESPN_WAIT(&S.tempty_bar[buf], ((gs / L::NBUF) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = S.tmem_base + buf * L::BUFC;
        const uint32_t x0 = st * L::STAGE_SLOTS;
        uint32_t acc = 0;
        if constexpr (L::REPA) {
          // one MMA per K-step over the whole stage: N = its slots (<= 4 NQC)
          const int rem = (int)Sl - (int)x0;
          const uint32_t nv = rem < L::STAGE_SLOTS ? (uint32_t)rem : (uint32_t)L::STAGE_SLOTS;
          const uint32_t idesc = umma_idesc_f16(128, (nv + 15u) & ~15u, p.bf16);
          const uint32_t a_addr = a_base + 128 * us * L::PW;
          const uint32_t b_addr = b_base + s * L::STAGE_BYTES;
          if (!(p.dbg & 2u))
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              const uint32_t kb = ks * 32;
              const uint64_t bd = umma_desc_sw(b_addr + (kb / L::PW) * L::PANEL_BYTES + (kb % L::PW), 8 * L::PW, L::SWZ);
#pragma unroll
              for (int part = 0; part < (L::SPLIT ? 2 : 1); ++part) {
                const uint64_t ad = umma_desc_sw(a_addr + part * L::LO_ROWS * L::PW + (kb / L::PW) * L::A_PANEL_BYTES +
                                                     (kb % L::PW), 8 * L::PW, L::SWZ);
                umma_f16_elect(d_tmem, ad, bd, idesc, acc);
                acc = 1;
              }
            }
        } else {
#if ESPN_MMA_DESC == 1
          // descriptors stepped per quarter (A 32 rows up the block-diagonal
          // window, B one quarter along the stage) instead of rebuilt per MMA
          uint64_t a_desc = umma_desc_sw(a_base + (96 + 128 * us) * L::PW, 8 * L::PW, L::SWZ);
          uint64_t b_desc = umma_desc_sw(b_base + s * L::STAGE_BYTES, 8 * L::PW, L::SWZ);
#pragma unroll 1
          for (int w = 0; w < 4; ++w) {
            const int rem = (int)Sl - (int)(x0 + w * L::NQC);
            if (rem <= 0) break;
            const uint32_t nv = rem < L::NQC ? (uint32_t)rem : (uint32_t)L::NQC;
            const uint32_t n_mma = (nv + 15u) & ~15u;
            if ((p.dbg & 2u) || ((p.dbg & 64u) && w > 0)) break;
            const uint32_t idesc = umma_idesc_f16(128, n_mma, p.bf16);
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              const uint32_t kb = ks * 32;
              const uint64_t bd = b_desc + (((kb / L::PW) * L::PANEL_BYTES + (kb % L::PW)) >> 4);
#pragma unroll
              for (int part = 0; part < (L::SPLIT ? 2 : 1); ++part) {
                const uint64_t ad = a_desc + ((part * L::LO_ROWS * L::PW + (kb / L::PW) * L::A_PANEL_BYTES +
                                               (kb % L::PW)) >> 4);
                umma_f16_elect(d_tmem, ad, bd, idesc, acc);
                acc = 1;
              }
            }
            a_desc -= (32 * L::PW) >> 4;
            b_desc += (L::NQC * L::PW) >> 4;
          }
#else
#pragma unroll 1
          for (int w = 0; w < 4; ++w) {
            const int rem = (int)Sl - (int)(x0 + w * L::NQC);
            if (rem <= 0) break;
            const uint32_t nv = rem < L::NQC ? (uint32_t)rem : (uint32_t)L::NQC;
            const uint32_t n_mma = (nv + 15u) & ~15u;
            if ((p.dbg & 2u) || ((p.dbg & 64u) && w > 0)) break;
            const uint32_t idesc = umma_idesc_f16(128, n_mma, p.bf16);
            const uint32_t a_row0 = 96 + 128 * us - 32 * w;
            const uint32_t a_addr = a_base + a_row0 * L::PW;
            const uint32_t b_addr = b_base + s * L::STAGE_BYTES + w * L::NQC * L::PW;
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              const uint32_t kb = ks * 32;  // K offset in bytes
              const uint64_t bd = umma_desc_sw(b_addr + (kb / L::PW) * L::PANEL_BYTES + (kb % L::PW),
                                               8 * L::PW, L::SWZ);
#pragma unroll
              for (int part = 0; part < (L::SPLIT ? 2 : 1); ++part) {  // hi, then lo (SPLIT)
                const uint64_t ad = umma_desc_sw(a_addr + part * L::LO_ROWS * L::PW + (kb / L::PW) * L::A_PANEL_BYTES +
                                                     (kb % L::PW), 8 * L::PW, L::SWZ);
                umma_f16_elect(d_tmem, ad, bd, idesc, acc);
                acc = 1;
              }
            }
          }
#endif
        }
        umma_commit_elect(&S.empty_bar[s]);
        umma_commit_elect(&S.tfull_bar[buf]);
      }
    }
    __syncwarp();
  } else if (warp < L::NEPI) {
    // ==================== EPILOGUE (warps 0..NEPI-1) ===========================
    // warp = h*4 + w: TMEM lane quarter w (== query-token quarter), column half h.
    // pm holds order-preserving int keys of the per-doc partial maxima; the two
    // halves of a quarter may both flush a doc straddling the split, so
    // flushes are shared-memory atomicMax (a few per stage).
    const int w = warp & 3, h = warp >> 2;
    uint32_t& gs = rs.gs;
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t gi = gu0 + it, us = gi % L::NU;
      const typename L::Unit& U = units[us];
      ESPN_WAIT(&S.ufull_bar[us], (gi / L::NU) & 1);
      const uint32_t Sl = U.S;
      int* my_pm = reinterpret_cast<int*>(S.pm) + (us * 32 + lane) * L::PM_STRIDE;
      const uint32_t n_st = (Sl + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t buf = gs % L::NBUF;
        ESPN_WAIT(&S.tfull_bar[buf], (gs / L::NBUF) & 1);
        tc_fence_after();
        const uint32_t xw = st * L::STAGE_SLOTS + w * L::NQC + h * L::HALF;
        const int remv = (p.dbg & 1u) ? 0 : (int)Sl - (int)xw;
        if (remv > 0) {
          // TMEM -> registers in NLD chunks of LW columns: chunk c+1 is read
          // (the SM's TMEM read port is the epilogue's floor) while chunk c's
          // group maxima are computed; the buffer is released after the last
          // chunk landed.  Only the short doc-boundary scan over NGH groups is
          // sequential.
          const uint32_t nv = remv < L::HALF ? (uint32_t)remv : (uint32_t)L::HALF;
          const uint32_t taddr0 = S.tmem_base + ((uint32_t)(w * 32) << 16) + buf * L::BUFC +
                                  (L::REPA ? w * L::NQC : 0) + h * L::HALF;
          float v[L::NLD < 2 ? L::NLD : 2][L::LW];  // two-chunk ring: chunk c in v[c & 1]
          tmem_ld_32x32b<L::LW>(taddr0, v[0]);
          const uint32_t G0 = xw >> 3;  // multiple of NGH
          const uint32_t bw = U.bitmap[G0 >> 5];
          const uint32_t sbits = (bw >> (G0 & 31)) & ((1u << L::NGH) - 1u);
          int doc = (int)(U.wprefix[G0 >> 5] + __popc(bw & ((2u << (G0 & 31)) - 1u))) - 1;
          constexpr int GPC = L::LW / 8;  // groups per chunk
          float gm[L::NGH];
#pragma unroll
          for (int c = 0; c < L::NLD; ++c) {
            tmem_ld_wait();
            if (c + 1 < L::NLD) {
              if ((uint32_t)(L::LW * (c + 1)) < nv) tmem_ld_32x32b<L::LW>(taddr0 + L::LW * (c + 1), v[(c + 1) & 1]);
            } else {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&S.tempty_bar[buf]);
            }
            // group maxima over the valid (non-pad) columns of chunk c
#pragma unroll
            for (int qq = 0; qq < GPC; ++qq) {
              const int q = c * GPC + qq;
              const float* x = &v[c & 1][8 * qq];
#if ESPN_NO_PATCH
              const uint32_t nvq = U.vc[G0 + q];  // warp-uniform
              if (nvq < 8) {
                float y[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) y[i] = (i == 0 || (uint32_t)i < nvq) ? x[i] : -INFINITY;
                gm[q] = fmaxf(fmax3(y[0], y[1], y[2]), fmax3(fmax3(y[3], y[4], y[5]), y[6], y[7]));
              } else {
                gm[q] = fmaxf(fmax3(x[0], x[1], x[2]), fmax3(fmax3(x[3], x[4], x[5]), x[6], x[7]));
              }
#else
              // pad columns hold copies of the doc's last row (patch warp): no masking
              gm[q] = fmaxf(fmax3(x[0], x[1], x[2]), fmax3(fmax3(x[3], x[4], x[5]), x[6], x[7]));
#endif
            }
          }
          if (p.dbg & 32u) continue;  // profiling knob: no scan / flush
          // doc-boundary scan, branch-free: after every group the running max
          // of the current doc goes to pm with a shared red.max (unconditional
          // -- a doc's last write carries its maximum; predicated flushes
          // compile into divergent branch blocks)
          float m = -INFINITY;
#pragma unroll
          for (int q = 0; q < L::NGH; ++q) {
            const bool valid = (uint32_t)(8 * q) < nv;
            const bool start = q > 0 && valid && ((sbits >> q) & 1u);
            doc += start ? 1 : 0;
            const float g = valid ? gm[q] : -INFINITY;
            m = start ? g : fmaxf(m, g);
            red_max_shared(&my_pm[doc], ord_key(m));
          }
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.tempty_bar[buf]);
        }
      }
      // all lanes' flushes of this unit are done: hand the slot to the combiner
      mbar_arrive(&S.edone_bar[us]);
    }
  } else if (warp == L::COMBINE_WARP) {
    // ============================ COMBINE ========================================
    // bow(doc) = sum_i pm[us][i][doc] (max over the doc's tokens, reduced by the
    // epilogue's atomicMax), i ascending (the oracle's summation order); then
    // the slot's keys are reset and the unit slot is released to the loader.
    // Runs concurrently with the epilogue of the next units.  Fused top-k: the
    // sums also go to the rank warp through the shared-memory bow ring.
    const bool fused = p.out_ids != nullptr;
    float* ring = reinterpret_cast<float*>(smem + L::OFF_RING);
    constexpr int NK = L::UNITMAX / 32;  // docs per lane
    for (uint32_t it = 0; it < cnt; ++it) {
      const uint32_t gi = gu0 + it, us = gi % L::NU;
      const typename L::Unit& U = units[us];
      ESPN_WAIT(&S.edone_bar[us], (gi / L::NU) & 1);
      const uint32_t nd = U.nd, tail = U.tail;
      const uint64_t j0 = U.cfirst;
      int* pmu = reinterpret_cast<int*>(S.pm) + us * 32 * L::PM_STRIDE;
      float bow[NK];
#pragma unroll
      for (int r = 0; r < NK; ++r) {
        const uint32_t k = r * 32 + lane;
        bow[r] = 0.0f;
        if (k < nd && !tail) {
          float sacc = 0.0f;
          for (uint32_t i = 0; i < p.nq; ++i) sacc = __fadd_rn(sacc, key_ord(pmu[i * L::PM_STRIDE + k]));
          bow[r] = sacc;
#pragma unroll 8
          for (uint32_t i = 0; i < 32; ++i) pmu[i * L::PM_STRIDE + k] = ord_key(-INFINITY);
        }
      }
      __syncwarp();
      if (ESPN_ARRIVE_ALL || lane == 0) mbar_arrive(&S.uempty_bar[us]);  // slot free
      if (fused) {
        const uint32_t j = gi % L::NB;
        ESPN_WAIT(&S.bfree_bar[j], ((gi / L::NB) & 1) ^ 1);
#pragma unroll
        for (int r = 0; r < NK; ++r) ring[j * L::UNITMAX + r * 32 + lane] = bow[r];
        __syncwarp();
        if (ESPN_ARRIVE_ALL || lane == 0) mbar_arrive(&S.bdone_bar[j]);  // every lane releases its own ring writes
      }
#pragma unroll
      for (int r = 0; r < NK; ++r)
        if (r * 32 + lane < nd && !tail) p.bow_out[j0 + r * 32 + lane] = bow[r];
    }
  } else if (warp == L::DEDUP_WARP || warp == L::RANK_WARP) {
    // ===================== DEDUP / RANK (fused top-k) ===========================
    // Both read their units straight from the unit table (the plan is
    // complete), so they never hold a unit slot: their latency (L2 atomics)
    // does not stall the copy pipeline.  DEDUP inserts the unit's ids into the
    // query's duplicate hash while the unit is scored.  RANK forms the keys
    // alpha*cls + bow (aggregate_score, scoring.hpp:12-14, no FMA contraction;
    // tail units alpha*cls) from the bow ring and writes the unit's best k,
    // sorted, to unit_top.  finalize_kernel (or, persistent, the dedup warps)
    // merges each query's unit lists.
    const bool fused = p.out_ids != nullptr;
    const bool is_rank = warp == L::RANK_WARP;
    uint64_t* fm = reinterpret_cast<uint64_t*>(smem + L::OFF_UK);  // rank warp: unit keys
    const float* ring = reinterpret_cast<const float*>(smem + L::OFF_RING);
    constexpr int NK = L::UNITMAX / 32;
    uint32_t par = 0;  // this batch's dedup table (plan_kernel advanced the epoch)
    if (fused) {
      par = __ldcg(&p.fused_state[0]) & 1u;
      if (!is_rank) {
        // clear this CTA's slice of the rows the previous fused batch used in
        // the other table (and its ff_seen flags), off the critical path
        const uint32_t prev_b = __ldcg(&p.fused_state[1 + (par ^ 1u)]);
        const size_t n4 = (size_t)prev_b * p.hash_slots / 4;
        uint4* t4 = reinterpret_cast<uint4*>(p.dedup + (size_t)(par ^ 1u) * p.max_queries * p.hash_slots);
        for (size_t i = (size_t)blockIdx.x * 32 + lane; i < n4; i += (size_t)G * 32)
          t4[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        uint32_t* ff = p.ff_seen + (size_t)(par ^ 1u) * p.max_queries;
        for (uint32_t i = blockIdx.x * 32 + lane; i < prev_b; i += G * 32) ff[i] = 0;
      }
    }
    for (uint32_t it = 0; it < cnt && fused; ++it) {
      const uint32_t ug = first + it * G, gi = gu0 + it;
      const uint4 ue = __ldcg(&p.unit_tab[ug]);
      const uint32_t b = ue.x, nd = ue.y & 0xFFu;
      const uint64_t j0 = (uint64_t)ue.z | ((uint64_t)ue.w << 32);
      if (!is_rank) {
        fused_dedup<NK>(p, par, b, j0, nd, lane);
        continue;
      }
      uint32_t idv[NK];
      float clv[NK];
#pragma unroll
      for (int r = 0; r < NK; ++r) {  // independent of the scoring: load before waiting
        const uint32_t k = r * 32 + lane;
        idv[r] = k < nd ? __ldcg(&p.cand_ids[j0 + k]) : 0u;
        clv[r] = k < nd ? __ldcg(&p.cand_cls[j0 + k]) : 0.0f;
      }
      const uint32_t j = gi % L::NB;
      ESPN_WAIT(&S.bdone_bar[j], (gi / L::NB) & 1);
      float bow[NK];
#pragma unroll
      for (int r = 0; r < NK; ++r) bow[r] = ring[j * L::UNITMAX + r * 32 + lane];
      __syncwarp();
      if (ESPN_ARRIVE_ALL || lane == 0) mbar_arrive(&S.bfree_bar[j]);
      uint64_t key[NK];
      uint32_t bad = 0;
#pragma unroll
      for (int r = 0; r < NK; ++r) {
        key[r] = 0;
        if (r * 32 + lane < nd) {
          const float sc = __fadd_rn(__fmul_rn(p.alpha, clv[r]), bow[r]);
          bad |= !isfinite(clv[r]) ? ERR_NONFINITE_CLS : (!isfinite(sc) ? ERR_NONFINITE_SCORE : 0u);
          key[r] = make_key(sc, idv[r]);
        }
      }
      if (bad) atomicOr(p.err, bad);
      // unit-local top-k by rank counting: rank(key) = #keys of the unit
      // greater than it (ids are unique, so ranks are distinct); the keys of
      // rank < k land sorted in unit_top, empty ranks are 0
      const uint32_t kk = p.k;
      unsigned long long* ut = p.unit_top + (size_t)ug * kk;
#pragma unroll
      for (int r = 0; r < NK; ++r) fm[r * 32 + lane] = key[r];
      __syncwarp();
      uint32_t rk[NK];
#pragma unroll
      for (int r = 0; r < NK; ++r) rk[r] = 0;
      for (uint32_t jj = 0; jj < nd; ++jj) {
        const uint64_t x = fm[jj];
#pragma unroll
        for (int r = 0; r < NK; ++r) rk[r] += x > key[r] ? 1u : 0u;
      }
#pragma unroll
      for (int r = 0; r < NK; ++r)
        if (r * 32 + lane < nd && rk[r] < kk) ut[rk[r]] = key[r];
      for (uint32_t i = nd + lane; i < kk; i += 32) ut[i] = 0ull;
      __syncwarp();
    }
    if (slot) {
      // ---- persistent server: batch completion + the merge of finalize_kernel ----
      __threadfence();  // this warp's unit_top / hash / error writes
      __syncwarp();
      if (lane == 0) atomicAdd(&slot->done_count, 1u);
      if (!is_rank) {
        const bool merges = fused && blockIdx.x < p.n_queries;  // this CTA merges queries blockIdx.x + i*G
        if (merges && lane == 0)
          while (ld_acquire_u32(&slot->done_count) < 2u * G) __nanosleep(256);
        __syncwarp();
        __threadfence();
        const uint32_t rejected = merges ? __ldcg(p.err) & (ERR_BAD_OFFSETS | ERR_CAPACITY) : 1u;
        if (merges && !rejected) {
          uint64_t* mfm = reinterpret_cast<uint64_t*>(smem + L::OFF_FM);
          for (uint32_t b = blockIdx.x; b < p.n_queries; b += G) {
            const uint32_t u0 = __ldcg(&p.unit_off[b]), nu = __ldcg(&p.unit_off[b + 1]) - u0;
            if (nu > 0) fused_merge<L::MERGE_KEYS>(p, b, u0, nu, mfm, lane);
          }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0 && atomicAdd(&slot->merge_count, 1u) == G - 1) {
          slot->done_count = 0;
          slot->merge_count = 0;
          __threadfence();
          st_release_u32(p.done_flag, 1u);
          st_release_u32(&slot->done, seq + 1u);
        }
      }
    }
  }
  if (tr && lane == 0) {
    atomicAdd(&g_cta_prof[2 * warp], (unsigned long long)(clock64() - tb0));
    atomicAdd(&g_cta_prof[2 * warp + 1], wacc);
  }
#undef ESPN_WAIT
}

template <int D, bool SPLIT>
// Register cap: the next batch's plan CTA (32 registers per thread) must fit
// beside a persistent server CTA on the busiest SM sub-partition (16 K
// registers): 4 warps x 120 with 16 warps, 5 warps x 96 with 17
__global__ void __maxnreg__((TcLayout<D, SPLIT>::MAXREG))
maxsim_tc_kernel(const MaxSimParams p) {
  using L = TcLayout<D, SPLIT>;
  using namespace espn_ptx;
  // swizzled operand atoms need 1024-byte aligned stage bases: align manually
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
  TcSmem<D, SPLIT> S;
  S.smem = smem;
  S.sB = smem + L::OFF_B;
  S.sA = smem + L::OFF_A;
  S.pm = reinterpret_cast<float*>(smem + L::OFF_PM);
  S.units = reinterpret_cast<typename L::Unit*>(smem + L::OFF_UNIT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  S.full_bar = bars;
  S.empty_bar = bars + L::NS;
  S.tfull_bar = bars + 2 * L::NS;
  S.tempty_bar = S.tfull_bar + L::NBUF;
  S.ufull_bar = S.tempty_bar + L::NBUF;
  S.uempty_bar = S.ufull_bar + L::NU;
  S.edone_bar = S.uempty_bar + L::NU;
  S.bdone_bar = S.edone_bar + L::NU;
  S.bfree_bar = S.bdone_bar + L::NB;
  S.patched_bar = S.bfree_bar + L::NB;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  if (p.prof && tid == 0) atomicMin(&p.prof[2], (unsigned long long)gtimer());
  ktl_begin(p.dbg, 1);

  // ---- one-time setup: zero operand tiles (stale NaN bit patterns would leak
  // into other quarters through the zero rows of A), barriers, TMEM ----------
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (L::OFF_PM) / 16;
    for (int i = tid; i < n16; i += L::NTHREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  {
    int* pmk = reinterpret_cast<int*>(smem + L::OFF_PM);
    for (int i = tid; i < L::PM_FLOATS; i += L::NTHREADS) pmk[i] = ord_key(-INFINITY);
    if (tid < 8) reinterpret_cast<uint32_t*>(smem + L::OFF_GATE)[tid] = 0u;
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&S.full_bar[i], L::NPROD);
      mbar_init(&S.empty_bar[i], 1);
    }
    for (int i = 0; i < L::NBUF; ++i) {
      mbar_init(&S.tfull_bar[i], 1);
      mbar_init(&S.tempty_bar[i], L::NEPI);
    }
    for (int i = 0; i < L::NU; ++i) {
      // unit loader + query-tile warp, every lane: a lane's own arrive
      // releases its shared-memory writes (compute-sanitizer racecheck does
      // not carry a __syncwarp + one-lane arrive across warps,
      // tools/racecheck_probe.cu)
      mbar_init(&S.ufull_bar[i], ESPN_ARRIVE_ALL ? 64 : 2);
      mbar_init(&S.uempty_bar[i], ESPN_ARRIVE_ALL ? 32 : 1);  // combine warp
      mbar_init(&S.edone_bar[i], 32 * L::NEPI);
    }
    for (int i = 0; i < L::NB; ++i) {
      mbar_init(&S.bdone_bar[i], ESPN_ARRIVE_ALL ? 32 : 1);  // combine warp, every lane
      mbar_init(&S.bfree_bar[i], ESPN_ARRIVE_ALL ? 32 : 1);  // rank warp, every lane
    }
    for (int i = 0; i < L::NS; ++i) mbar_init(&S.patched_bar[i], 1);
    mbar_fence_init();
  }
  if (warp == L::MMA_WARP) tmem_alloc<L::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  S.tmem_base = *tmem_holder;
  TcRoleState rs;

  if (!p.server) {
    // programmatic dependent of plan_kernel: everything above overlapped it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // let the dependent grid launch now (the plan is complete): the finalize
    // merge or the top-k kernel's id-only dedup prologue runs on the SMs'
    // spare resources concurrently with this kernel
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tc_batch<D, SPLIT>(p, S, rs, nullptr, 0u);
  } else {
    // ---- persistent re-rank server: every warp walks the queue in order ----
    // Only the loader warp's lane 0 polls the global queue (one poller per
    // CTA keeps the queue's cache line cool); it copies each batch descriptor
    // into the CTA's shared ring and opens the gate; the other warps wait on
    // the gate in shared memory and read the descriptor from the ring.
    ServerQueue* Q = p.server;
    const unsigned long long idle_ns = Q->idle_ns;
    MaxSimParams* ring = reinterpret_cast<MaxSimParams*>(smem + L::OFF_DESC);
    volatile uint32_t* gate = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_GATE);
    constexpr int NW = (int)(sizeof(MaxSimParams) / 4);
    for (uint32_t seq = 0;; ++seq) {
      ServerSlot* sl = &Q->slot[seq % kServerSlots];
      const uint32_t rslot = seq % L::DESC_RING;
      uint32_t stop = 0;
      if (warp == L::LOADER_WARP) {
        if (lane == 0) {
          const unsigned long long t_wait = gtimer();
          for (;;) {
            if (ld_acquire_u32(&sl->ready) == seq + 1u) break;
            const unsigned long long st = ld_acquire_u64(&Q->state);
            if (st == (kServerStopped | seq)) { stop = 1; break; }  // stopped here by another CTA
            if ((st & ~kServerStopped) == seq &&                    // nothing taken beyond what we wait for
                (ld_acquire_u32(&Q->stop_req) || gtimer() - t_wait > idle_ns) &&
                atomicCAS(&Q->state, (unsigned long long)seq, kServerStopped | seq) == seq) {
              stop = 1;
              break;
            }
            __nanosleep(400);
          }
          // the ring slot is free once every warp finished the batch RING before
          if (!stop && seq >= (uint32_t)L::DESC_RING)
            while (gate[2 + rslot] < (uint32_t)L::NWARPS * (seq / L::DESC_RING)) __nanosleep(32);
        }
        stop = __shfl_sync(0xffffffffu, stop, 0);
        if (!stop) {
          const uint32_t* src = reinterpret_cast<const uint32_t*>(&sl->p);
          uint32_t* dst = reinterpret_cast<uint32_t*>(&ring[rslot]);
          for (int i = lane; i < NW; i += 32) dst[i] = __ldcg(src + i);
          __threadfence_block();
        }
        __syncwarp();
        if (lane == 0) {
          if (stop) gate[1] = seq + 1u;
          else gate[0] = seq + 1u;
        }
      } else if (lane == 0) {
        for (;;) {
          if (gate[0] > seq) break;
          if (gate[1] == seq + 1u) { stop = 1; break; }
          __nanosleep(32);
        }
      }
      if (__shfl_sync(0xffffffffu, stop, 0)) break;
      __threadfence_block();
      tc_batch<D, SPLIT>(ring[rslot], S, rs, sl, seq);
      __syncwarp();
      if (lane == 0) atomicAdd(const_cast<uint32_t*>(&gate[2 + rslot]), 1u);  // done with the ring slot
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == L::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<L::TMEM_COLS>(S.tmem_base);
  }
  if (p.server && tid == 0 && atomicAdd(&p.server->exited, 1u) == gridDim.x - 1) {
    __threadfence_system();
    *reinterpret_cast<volatile uint32_t*>(p.server->alive_host) = 0u;  // the host may relaunch
  }
  ktl_end(p.dbg, 1);
  if ((p.dbg & 256u) && threadIdx.x == 0 && blockIdx.x < 256) g_cta_prof[4 * blockIdx.x] = ktl_now();
  if (p.prof && tid == 0) {
    __threadfence();
    if (atomicAdd(&p.prof[3], 1ull) == gridDim.x - 1) {  // last CTA out
      const unsigned long long t0 = atomicAdd(&p.prof[2], 0ull);
      atomicAdd(&p.prof[0], (unsigned long long)gtimer() - t0);
      atomicAdd(&p.prof[1], 1ull);
      p.prof[2] = ~0ull;
      p.prof[3] = 0;
    }
  }
}

}  // namespace espn_k
