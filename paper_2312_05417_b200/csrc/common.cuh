// common.cuh -- parameter blocks shared by the re-rank kernels.
#pragma once
#include <cstdint>

namespace espn_k {

// ESPN_DEBUG (env, read once by the library; 0 in production) -- profiling
// knobs, each removes or instruments one piece so its cost can be measured
// (scratch/timeline.py); results are NOT valid with bits 1-128 set:
//   1 no epilogue work   2 no MMAs   4 no row copies   8 CTA-0 role trace
//   32 no doc-boundary scan   64 quarter-0 MMAs only   128 top-k: no dedup
//   256 device timeline (below)   512 separate top-k kernel
//   0x10000 finalize as a programmatic dependent of MaxSim   0x40000 no graph for synchronous host calls
// ESPN_DEBUG bit 256: per-kernel device timeline of the re-rank step (first
// CTA start, last CTA end, globaltimer ns) -- slot 0 plan, 1 MaxSim, 2 top-k.
// Read/reset through espn_gpu_debug_timeline (profiling only).
__device__ unsigned long long g_ktl[8];
__device__ unsigned long long g_fin[8];  // profiling: summed finalize phase times
__device__ unsigned long long g_cta_prof[4 * 256];  // per CTA: end, rank-warp end, merges, dedup-warp end
__device__ __forceinline__ unsigned long long ktl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktl_begin(uint32_t dbg, int k) {
  if ((dbg & 256u) && threadIdx.x == 0) atomicMin(&g_ktl[2 * k], ktl_now());
}
__device__ __forceinline__ void ktl_end(uint32_t dbg, int k) {
  if ((dbg & 256u) && threadIdx.x == 0) atomicMax(&g_ktl[2 * k + 1], ktl_now());
}

// Global doc id -> local row index of this shard, or UINT64_MAX if the id is
// not stored here (unknown id / wrong shard -> DataIntegrityError).
__device__ __forceinline__ uint64_t shard_local(uint32_t id, uint32_t count, uint32_t index,
                                                uint64_t n_docs) {
  uint64_t local = id;
  if (count > 1) {
    if (id % count != index) return ~0ull;
    local = id / count;
  }
  return local < n_docs ? local : ~0ull;
}

// HBM tile layout of the table rows.  For the tensor-core dims
// (d in {16, 32, 64, 128}) each document's t token rows are stored as
// NP = max(1, 2d/128) K-panels of t rows x PW bytes (PW = min(2d, 128)), and
// inside a panel the 16-byte chunks of row j are XOR-permuted by
// sw(j) = ((j * PW) >> 7) & (PW/16 - 1) -- exactly the UMMA K-major
// SWIZZLE_{32,64,128}B pattern of a row sitting at an 8-row-aligned shared
// memory slot.  A document (or a panel of it) is therefore ONE contiguous
// byte range that a single cp.async.bulk drops into the MMA operand layout.
// Other dims keep plain row-major rows.  Doc boundaries come from row_ptr, so
// the layout is doc-relative: row j of a doc is its j-th token.
template <int D>
struct RowLayout {
  static constexpr bool TILED = (D == 16 || D == 32 || D == 64 || D == 128);
  static constexpr int ROWB = 2 * D;
  static constexpr int PW = TILED ? (ROWB < 128 ? ROWB : 128) : ROWB;
  static constexpr int NP = ROWB / PW;
  static constexpr int CPP = PW / 16;  // 16-byte chunks per panel row
  static constexpr int CH = ROWB / 16; // 16-byte chunks per row
  // byte offset (inside a doc of t rows) of 16-byte chunk c of row j
  __host__ __device__ static __forceinline__ uint32_t off(uint32_t t, uint32_t j, uint32_t c) {
    if (!TILED) return j * (uint32_t)ROWB + c * 16u;
    const uint32_t p = c / CPP, cc = c % CPP;
    const uint32_t sw = ((j * (uint32_t)PW) >> 7) & (uint32_t)(CPP - 1);
    return (p * t + j) * (uint32_t)PW + ((cc ^ sw) << 4);
  }
};

// Device-side error bits (mapped to espn_status by the host after sync).
enum : uint32_t {
  ERR_UNKNOWN_DOC = 1u << 0,     // candidate id >= n_docs  -> DATA_INTEGRITY
  ERR_NONFINITE_QUERY = 1u << 1, // query token not finite / not representable -> INVALID_INPUT
  ERR_NONFINITE_CLS = 1u << 2,   // cls score not finite -> INVALID_INPUT
  ERR_DUPLICATE = 1u << 3,       // duplicate candidate id -> INVALID_INPUT (scoring.hpp:16-18)
  ERR_NONFINITE_SCORE = 1u << 4, // aggregate score not finite -> INVALID_INPUT
  ERR_UNIT_TOO_LARGE = 1u << 5,  // internal: slot budget of a work unit exceeded
  ERR_BAD_OFFSETS = 1u << 6,     // cand_offsets not starting at 0 / decreasing -> INVALID_INPUT
  ERR_CAPACITY = 1u << 7,        // batch exceeds workspace capacity -> INVALID_INPUT
  ERR_STAGING = 1u << 8,         // host-tier rows of a batch exceed the staging buffer -> INVALID_CONFIG
  ERR_SERVER = 1u << 9,          // persistent server: the batch did not complete in time -> INVALID_STATE
  ERR_NOT_PREFETCHED = 1u << 10  // disk tier: a needed doc was not staged by espn_gpu_prefetch_rows -> INVALID_STATE
};

// doc_loc tier bits (tiered tables): bit 0 = not in HBM; bit 1 = on the disk
// tier (ESPN_TABLE_DISK_TIER: no in-memory copy, the word holds no address)
constexpr uint64_t kLocHost = 1ull, kLocDisk = 2ull;

// Staging of host-tier rows for one batch (stage_kernel): one CTA per query,
// one warp per needed candidate.
struct StageParams {
  const uint64_t* row_ptr;
  const uint64_t* doc_loc;     // per doc: address | tier bit
  uint64_t n_docs;
  uint32_t shard_count, shard_index;
  const uint32_t* cand_ids;
  const uint64_t* cand_off;    // B + 1
  const uint32_t* needed_in;   // optional per-query needed override
  uint32_t rerank_count;
  uint32_t n_queries;
  uint64_t max_candidates;     // bound check on (not yet validated) offsets
  uint32_t row_bytes;          // 2 * d
  uint32_t prefetch;           // 1: staged ahead (side stream), 0: critical path
  uint64_t* cand_src;          // out: per candidate, HBM address of its rows
  uint8_t* stage;              // HBM staging buffer
  uint64_t stage_cap;
  unsigned long long* cursor;  // bytes used in stage (zeroed before the launch)
  unsigned long long* qstats;  // B x 6 (espn_fetch_stats layout)
  uint32_t* err;
  const uint64_t* hint_map;    // optional (consumer of espn_gpu_prefetch_hints): per local doc,
                               // epoch << 32 | staged offset / 16
  uint32_t hint_epoch;
  uint8_t* cand_status;        // out, per needed candidate: 0 HBM-resident, 1 staged by the prefetcher,
                               // 2 staged on the critical path, 3 not staged (overflow / unknown id)
};

// Hint staging (espn_gpu_prefetch_hints): CTA per query, warp per hinted doc.
struct HintParams {
  const uint64_t* row_ptr;
  const uint64_t* doc_loc;
  uint64_t n_docs;
  uint32_t shard_count, shard_index;
  const uint32_t* hint_ids;
  const uint64_t* hint_off;    // n_queries + 1
  uint64_t max_hints;          // bound check on the (possibly device) offsets
  uint32_t row_bytes;
  uint64_t* hint_map;          // per local doc: epoch << 32 | staged offset / 16 (0xffffffff = claimed)
  uint32_t epoch;
  uint8_t* stage;
  uint64_t stage_cap;          // bytes the hints may use
  unsigned long long* cursor;
  unsigned long long* qstats;  // B x 6: [4] += bytes this query's warps staged
  uint32_t* err;
  // espn_gpu_prefetch_rows: the rows come from the caller (plain row-major
  // codes in device memory, hint j's doc at ext_src + ext_off[j]) and are
  // tiled into the staging slot; NULL: copy the doc's host-tier rows
  const uint8_t* ext_src;
  const uint64_t* ext_off;
  uint32_t d;
};

// Byte offset of 16-byte chunk c of row j inside a doc of t rows in the HBM
// tile layout -- RowLayout<D>::off for a run-time d.
__device__ __forceinline__ uint32_t tile_off_rt(uint32_t d, uint32_t t, uint32_t j, uint32_t c) {
  if (d != 16 && d != 32 && d != 64 && d != 128) return j * 2 * d + c * 16;
  const uint32_t pw = 2 * d < 128 ? 2 * d : 128, cpp = pw / 16;
  const uint32_t p = c / cpp, cc = c % cpp;
  const uint32_t sw = ((j * pw) >> 7) & (cpp - 1);
  return (p * t + j) * pw + ((cc ^ sw) << 4);
}

// Device-side batch planning (plan_kernel): per-query needed counts, work
// units of the MaxSim kernel, all from device-resident candidate offsets, so
// a whole re-rank batch is a fixed launch sequence (CUDA-graph capturable).
struct PlanParams {
  const uint64_t* cand_off;    // B + 1
  const uint32_t* needed_in;   // optional B: per-query needed override (sharding)
  uint32_t* needed;            // out B
  uint32_t* unit_off;          // out B + 1: prefix of work units (SIMT: of pairs)
  uint4* unit_tab;             // out: tcgen05 work units {b, n_docs, first candidate lo, hi}
  uint32_t* n_units;           // out: total work units
  uint32_t* err;
  uint64_t max_candidates;
  uint64_t max_units;
  uint32_t n_queries;
  uint32_t rerank_count;
  uint32_t unit_docs;          // docs per unit (tcgen05); 1 for SIMT (units = pairs)
  uint32_t write_tab;          // 1: tcgen05 (fill unit_tab)
  uint32_t tail_units;         // 1: fused top-k with partial re-rank -- also plan the
                               //    alpha*cls tail [needed, n) as MMA-free units
  uint32_t* out_counts;        // fused top-k: queries with no unit get count 0 here (else NULL)
  uint32_t* fused_state;       // fused top-k: advance {epoch, rows per parity} (else NULL)
  uint32_t base_ok;            // cand_off[0] may be nonzero (a query slice of a larger batch, REPLICA placement)
  uint32_t dbg;                // profiling knobs (ESPN_DEBUG env; 0 in production)
};

// Unit-table entry .y: bits 0-7 doc count, bits 8-30 units of the unit's query,
// bit 31 = alpha*cls tail unit (no MaxSim).
constexpr uint32_t kUnitTail = 1u << 31;
constexpr uint32_t kUnitMaxPerQuery = (1u << 23) - 1;
__host__ __device__ __forceinline__ uint32_t unit_y(uint32_t nd, uint32_t nu, bool tail) {
  return nd | (nu << 8) | (tail ? kUnitTail : 0u);
}

// Ranking keys: key = orderable(score) << 32 | ~doc_id, so "larger key first"
// is exactly rank()'s (score desc, doc_id asc) (scoring.hpp:16-18); key 0 is
// never produced by a finite score and marks an empty entry.
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
// Warp-wide max of a 64-bit key: two 32-bit redux.sync steps (high word, then
// low word among the lanes holding the high maximum).
__device__ __forceinline__ uint64_t warp_max_key(uint64_t v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? (uint32_t)v : 0u);
  return ((uint64_t)mh << 32) | ml;
}
constexpr int kFusedMaxK = 32;

// Absolute address of doc `loc`'s rows: untiered tables keep every row in one
// HBM buffer; tiered tables carry a per-doc address with the
// tier in bit 0 (0 = HBM, 1 = pinned host, mapped).
__device__ __forceinline__ const uint8_t* doc_rows(const uint16_t* rows, const uint64_t* doc_loc, uint64_t loc,
                                                   uint64_t r0, uint32_t d) {
  if (doc_loc) return reinterpret_cast<const uint8_t*>(doc_loc[loc] & ~1ull);
  return reinterpret_cast<const uint8_t*>(rows + r0 * d);
}

struct ServerQueue;
// One batch of (query, candidate list) pairs, resident on the device.
struct MaxSimParams {
  const uint16_t* rows;        // table token rows, d codes each
  const uint64_t* doc_loc;     // tiered tables: per-doc row address | tier bit (else NULL)
  const uint64_t* cand_src;    // tiered tables: per-candidate row address in HBM after staging
  const uint64_t* row_ptr;     // n_docs + 1
  uint64_t n_docs;             // local docs of this shard
  uint32_t shard_count;        // doc-id sharding: id % shard_count == shard_index
  uint32_t shard_index;        //   lives at local index id / shard_count
  const float* q32;            // B * nq * d fp32 query tokens
  const uint32_t* cand_ids;    // CSR over queries
  const uint64_t* cand_off;    // B + 1
  const uint32_t* unit_off;    // B + 1: SIMT path: per-query pair prefix
  const uint4* unit_tab;       // tcgen05 path: per work unit {b, n_docs, first candidate (u64 lo, hi)}
  const uint32_t* needed;      // B: needed (scored with MaxSim) candidates per query
  float* bow_out;              // per candidate MaxSim score (first min(R, n_b) of each query)
  uint32_t* err;               // error bits
  uint32_t n_queries;
  uint32_t nq;                 // query tokens, 1..32
  uint32_t rerank_count;       // R
  uint32_t unit_docs;          // docs per work unit (<= kUnitMax)
  const uint32_t* n_units;     // device: total work units (written by plan_kernel)
  uint32_t bf16;               // table dtype
  uint32_t qround;             // SIMT: round the query to the table dtype first (ESPN_RERANK_QUERY_ROUNDED)
  uint32_t dbg;                // profiling knobs (ESPN_DEBUG env; 0 in production)
  // ESPN_RERANK_PROFILE: device-timed kernel duration (globaltimer, min start
  // over CTAs -> end of the last CTA), accumulated as {sum_ns, launches,
  // start scratch, CTA-done counter}; graph-replay safe.  NULL = off.
  unsigned long long* prof;
  // Fused aggregate + top-k (combine warp); out_ids == NULL: off,
  // the separate top-k kernel runs instead.
  const float* cand_cls;
  float alpha;
  uint32_t k;                  // final_k (<= kFusedMaxK)
  uint32_t* out_ids;           // B * k
  float* out_scores;           // B * k
  uint32_t* out_counts;        // B
  unsigned long long* unit_top;  // per work unit: its best k keys, descending
  // Duplicate hash, double-buffered by batch parity: a fused batch inserts
  // into table[parity] and clears the rows table[parity ^ 1] held for the
  // previous fused batch (the state word pair {epoch, rows used per parity}
  // is advanced by plan_kernel), so no kernel pays a clear on its critical path.
  uint32_t* dedup;             // 2 x max_queries x hash_slots ids, 0xFFFFFFFF = empty
  uint32_t* ff_seen;           // 2 x max_queries: id 0xFFFFFFFF (the empty code) seen
  const uint32_t* fused_state; // {epoch, queries used by parity 0, by parity 1}
  uint32_t hash_slots;         // power of two >= 2 x longest scored list (8x: one-probe inserts)
  uint32_t max_queries;        // parity stride of dedup / ff_seen
  // Persistent re-rank server: the kernel launch carries only
  // `server`; each batch's parameters arrive through the server's queue.
  // done_flag: the workspace's completion flag (set by the server once the
  // batch's ranked lists are written, consumed by server_wait_kernel).
  struct ServerQueue* server;
  uint32_t* done_flag;
};

// ---- persistent re-rank server: the batch queue in device memory ----------------
// plan_kernel (the submitter, on the caller's stream) takes seq = tail++,
// waits for the slot of seq - kServerSlots to be done, writes the batch's
// MaxSimParams into slot seq % kServerSlots and publishes ready = seq + 1.
// Every warp of the persistent MaxSim kernel walks seq 0, 1, 2, ...; the
// rank + dedup warps of all CTAs count the batch done (done_count), the dedup
// warps merge the queries' unit lists (merge_count), the last one sets the
// workspace's done_flag and the slot's done = seq + 1.
constexpr int kServerSlots = 8;
struct ServerSlot {
  MaxSimParams p;
  uint32_t ready;        // seq + 1: published
  uint32_t done;         // seq + 1: ranked lists written, slot reusable
  uint32_t done_count;   // rank + dedup warps finished (target 2 x grid)
  uint32_t merge_count;  // dedup warps finished merging (target grid)
};
// state = kServerStopped | next sequence number.  A submitter takes seq =
// state++ only while not stopped (CAS); a server warp waiting at seq T for a
// batch that is not there stops the server -- on a host request or after
// idle_ns without work -- with CAS(state: T -> T | stopped).  Every warp of
// every CTA then sees "stopped at T" and exits at the same point, and no
// batch can be taken after it.  An idle server exits by itself so a device-
// wide synchronisation (cudaFree, cudaDeviceSynchronize) in the process is
// delayed by at most idle_ns instead of deadlocking; the library relaunches
// it on the next served batch.
constexpr unsigned long long kServerStopped = 1ull << 63;
struct ServerQueue {
  unsigned long long state;  // kServerStopped | next sequence number
  uint32_t stop_req;         // host: stop once the queue is drained
  uint32_t exited;           // CTAs that left the persistent loop
  unsigned long long idle_ns;
  uint32_t* alive_host;      // mapped pinned word: 1 while the kernel runs (last CTA out clears it)
  uint32_t pad[2];
  ServerSlot slot[kServerSlots];
};
// plan_kernel's submission to a running server (server == NULL: none)
struct ServerSubmit {
  ServerQueue* server;
  uint32_t* plan_done;      // per workspace: plan CTAs finished (reset by the submitter)
  MaxSimParams msp;         // the batch's parameters
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


struct TopKParams {
  const float* bow;            // per candidate MaxSim (valid for the first R of each query)
  const uint32_t* cand_ids;
  const float* cand_cls;
  const uint64_t* cand_off;    // B + 1
  const uint32_t* needed;      // B: first needed[b] candidates carry a MaxSim score
  uint32_t* out_ids;           // B * k
  float* out_scores;           // B * k
  uint32_t* out_counts;        // B
  uint32_t* err;
  uint32_t n_queries;
  uint32_t rerank_count;
  uint32_t k;
  uint32_t partial;            // tail beyond R scored alpha * cls
  float alpha;
  uint32_t dbg;                // profiling knobs (ESPN_DEBUG env; 0 in production)
};

}  // namespace espn_k
