/*
 * espn_gpu.h -- C-ABI of the B200-native ESPN re-ranking hot path
 * (gather candidate token rows -> MaxSim -> aggregate -> top-k).
 *
 * This is the drop-in boundary: the reference keeps re-ranking inside
 * `espn::run_query` (proj/include/espn/pipeline.hpp:56-64) over
 * `StoreHandle::fetch_batch` (store.hpp:91-94) + `maxsim_score` /
 * `aggregate_score` / `rank` (scoring.hpp:7-21).  These entry points replace
 * exactly that path; the C++ wrapper in include/espn_b200.hpp re-exposes them
 * with the reference's types and exceptions.  Conventions:
 *   - extern "C", POD structs, no exceptions, no STL, no torch types;
 *   - every call returns an espn_status (one code per error class of
 *     error.hpp:8-42) and leaves a thread-local message in espn_last_error();
 *   - tables are opaque, read-only after open and shareable across threads;
 *     a workspace holds per-stream scratch and must not be used by two
 *     threads at once (one in-flight batch per workspace);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 * There is no CPU fallback: without a usable sm_100 device every call that
 * touches the device returns ESPN_E_CUDA.
 */
#ifndef ESPN_GPU_H
#define ESPN_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESPN_GPU_ABI_VERSION 1

#if defined(__GNUC__)
#define ESPN_API __attribute__((visibility("default")))
#else
#define ESPN_API
#endif

/* error.hpp:14-42, plus a device/runtime failure class. */
typedef enum {
  ESPN_OK = 0,
  ESPN_E_INVALID_INPUT = 1,   /* InvalidInputError */
  ESPN_E_INVALID_STATE = 2,   /* InvalidStateError */
  ESPN_E_INVALID_CONFIG = 3,  /* InvalidConfigError */
  ESPN_E_FORMAT = 4,          /* FormatError */
  ESPN_E_IO = 5,              /* IoError */
  ESPN_E_DATA_INTEGRITY = 6,  /* DataIntegrityError */
  ESPN_E_CUDA = 7             /* device / runtime failure (espn::Error) */
} espn_status;

typedef enum { ESPN_DTYPE_F16 = 0, ESPN_DTYPE_BF16 = 1 } espn_dtype;

/* MaxSim implementation selector (north_star: tcgen05 path plus a CUDA-core
 * path for tiny dims, chosen by measurement).  SMALL: the whole re-rank of a
 * small batch (<= 16 queries, scored lists <= 2048, final_k <= 32, table in
 * HBM) in ONE launch on the CUDA cores -- bit-exact with the fp32-query
 * reference; for latency-bound callers (configs[0]: batch 1).  Opt-in: AUTO
 * keeps one arithmetic (tcgen05) for every batch size. */
typedef enum {
  ESPN_KERNEL_AUTO = 0,
  ESPN_KERNEL_TCGEN05 = 1,
  ESPN_KERNEL_SIMT = 2,
  ESPN_KERNEL_SMALL = 3
} espn_kernel;

typedef struct espn_gpu_table espn_gpu_table;
typedef struct espn_gpu_workspace espn_gpu_workspace;

/* Table flags. */
#define ESPN_TABLE_DEVICE_BORROWED 0x1u /* row_ptr/rows are device pointers owned by the caller */
#define ESPN_TABLE_ROWS_TILED 0x2u      /* rows are already in the HBM tile layout,
                                           e.g. written by espn_gpu_synth_table; otherwise rows are
                                           plain row-major and the library tiles them at open (a
                                           borrowed plain table gets a library-owned tiled copy) */

#define ESPN_TABLE_STREAMED 0x4u       /* rows == NULL: the table is allocated from row_ptr (and the resident
                                           mask) -- the HBM tier holds only the resident docs, the pinned-host
                                           tier the rest -- and filled by espn_gpu_table_load_rows in doc order,
                                           so neither the whole table nor its HBM-sized staging ever exists on
                                           the host or the device (a table larger than free HBM opens); calls
                                           that read rows fail with INVALID_STATE until every doc is loaded */

#define ESPN_TABLE_DISK_TIER 0x8u      /* with STREAMED + resident: the non-resident docs stay in the store
                                           file (the NVMe tier, PAPER.md's premise) -- no pinned or HBM copy is
                                           made; a batch that needs them must be staged by espn_gpu_prefetch_rows
                                           (rows the caller read from the file, espn_store_fetch) and re-ranked
                                           with ESPN_RERANK_PREFETCHED, else INVALID_STATE; gathers fail */

/* The embedding table (store.hpp:13-35).  The HBM tier holds BOW rows only as
 * CSR: doc i's t_i token rows live at rows[row_ptr[i]*d .. row_ptr[i+1]*d),
 * 2-byte codes of `dtype`.  Callers pass plain row-major rows; in HBM the
 * library keeps each document in the "tile layout" (d in {16,32,64,128}: K-panels
 * of <=128-byte rows with the UMMA swizzle applied per document)
 * so one bulk copy per document feeds the tensor cores.  Every read-back path
 * (espn_gpu_gather) returns plain rows.  d_cls / value_width / alignment describe the
 * reference's on-disk record (record_bytes = (d_cls + t*d)*value_width) and are
 * used only for QueryStats byte accounting.  Replaces open_store()
 * (store.hpp:109-112) + the manifest (store.hpp:20-35). */
typedef struct {
  uint64_t n_docs;
  uint32_t d;            /* token dim: multiple of 16, 16..256 */
  uint32_t dtype;        /* espn_dtype */
  uint32_t d_cls;
  uint32_t value_width;  /* 2 or 4 */
  uint32_t alignment;    /* 1, 512 or 4096 */
  uint32_t flags;        /* ESPN_TABLE_* */
  const uint64_t* row_ptr; /* n_docs + 1 token offsets, row_ptr[0] == 0 */
  const uint16_t* rows;    /* row_ptr[n_docs] * d codes */
  int32_t device;          /* CUDA device ordinal */
  /* Doc-id sharding (multi-GPU): this table holds the docs with
   * id % shard_count == shard_index, global id g at local index g / shard_count.
   * All ids crossing the ABI stay global.  0 or 1 = unsharded. */
  uint32_t shard_count;
  uint32_t shard_index;
  /* Tiered store (SURVEY.md §8 a9, configs[3]): optional HOST array of n_docs
   * flags; docs with resident[i] != 0 live in HBM, the others in a pinned-host
   * tier (the overflow tier) and are staged into HBM per batch -- ahead of time
   * by espn_gpu_prefetch on a side stream, or on the critical path.  NULL =
   * every doc HBM-resident. */
  const uint8_t* resident;
  uint32_t reserved[4];
} espn_table_desc;

typedef struct {
  uint64_t n_docs;
  uint64_t n_tokens;
  uint32_t d;
  uint32_t dtype;
  uint32_t max_tokens;     /* longest doc */
  uint32_t min_tokens;
  uint64_t hbm_bytes;      /* device bytes held by the table */
  uint64_t host_bytes;     /* pinned-host tier bytes (tiered tables) */
  uint64_t resident_docs;  /* docs in HBM (n_docs unless tiered) */
} espn_table_info;

/* Validates (t >= 1 per doc, row_ptr monotone; types.hpp:64-68) and uploads
 * the table to HBM (or adopts device pointers when DEVICE_BORROWED). */
ESPN_API int espn_gpu_table_open(const espn_table_desc* desc, espn_gpu_table** out);
ESPN_API int espn_gpu_table_close(espn_gpu_table* table);
/* ESPN_TABLE_STREAMED tables: loads docs [doc_begin, doc_begin + n) (the
 * next docs in order) from plain row-major HOST codes (the docs' rows back
 * to back, row_ptr order) into their tiers, tiled on the way (HBM docs through
 * a bounded pinned/device bounce, host-tier docs tiled directly into the
 * pinned tier).  Synchronous. */
ESPN_API int espn_gpu_table_load_rows(espn_gpu_table* table, uint64_t doc_begin, uint64_t n, const uint16_t* rows);
ESPN_API int espn_gpu_table_info(const espn_gpu_table* table, espn_table_info* out);

/* Per-stream scratch sized for at most max_queries queries and
 * max_candidates candidates per batch (sum over the batch). */
typedef struct {
  uint32_t max_queries;
  uint32_t max_candidates;
  uint32_t max_query_tokens; /* <= 32 */
  uint32_t max_list;         /* longest candidate list of a query (sizes the top-k duplicate
                                check when offsets are device-resident); 0 = min(max_candidates, 4096) */
  uint64_t staging_bytes;    /* tiered tables: HBM staging per batch for host-tier rows
                                (two buffers: one scoring, one prefetching); 0 = 64 MB */
  uint32_t reserved[2];
} espn_workspace_desc;

ESPN_API int espn_gpu_workspace_create(espn_gpu_table* table, const espn_workspace_desc* desc,
                              espn_gpu_workspace** out);
ESPN_API int espn_gpu_workspace_destroy(espn_gpu_workspace* ws);

/* Re-rank flags (PipelineConfig, pipeline.hpp:11-29, plus I/O placement). */
#define ESPN_RERANK_PARTIAL 0x1u      /* partial_rerank_enabled: tail beyond R scored alpha*cls */
#define ESPN_RERANK_DEVICE_IO 0x2u    /* all array pointers in args/out are device pointers */
#define ESPN_RERANK_ASYNC 0x4u        /* do not synchronize; errors surface in espn_gpu_workspace_sync */
#define ESPN_RERANK_WRITE_BOW 0x8u    /* also return per-candidate MaxSim (bow) scores */
#define ESPN_RERANK_PROFILE 0x10u     /* time the MaxSim and top-k kernels with CUDA events on
                                         `stream` (accumulated into espn_counters) */
#define ESPN_RERANK_PREFETCHED 0x40u  /* tiered table: this batch was staged by the last
                                         espn_gpu_prefetch of this workspace (same ids/offsets);
                                         otherwise host-tier rows are staged on the critical path */
#define ESPN_RERANK_SEPARATE_TOPK 0x80u /* rank in a separate top-k kernel instead of inside the
                                         tcgen05 MaxSim kernel (the fused path is the default when
                                         final_k <= 32; results are identical) */
#define ESPN_RERANK_QUERY_ROUNDED 0x100u /* round the fp32 query to the table dtype before MaxSim (one MMA
                                         per K-step; CUDA-core path too).  Default: the CUDA-core path
                                         multiplies the fp32 query exactly (types.hpp:33-44); the tcgen05
                                         path carries it as q = hi + lo in the table dtype (two MMAs per
                                         K-step, 16 significant bits) for bf16 tables and rounds it to f16
                                         (11 bits, <= ~5e-4 relative) for f16 tables */
#define ESPN_RERANK_QUERY_SPLIT 0x200u  /* tcgen05: hi + lo query for f16 tables too (22 significant bits;
                                         ~17% slower MaxSim at d = 32) */
#define ESPN_RERANK_DEVICE_OFFSETS 0x20u /* cand_offsets / needed_counts are DEVICE pointers (needs
                                         DEVICE_IO): the batch is planned on the device, the call has
                                         no host-side loop, no host sync with ASYNC, and is CUDA-graph
                                         capturable; validation errors surface at sync */

/* One batch of queries with their final candidate lists (ivf.hpp:45-50:
 * sorted (cls_score desc, doc_id asc), deduplicated), CSR over queries.
 * This is the "candidates in -> ranked out" seam of run_query stages 3-6
 * (SPEC.md:276): needed = first min(R, n_b) candidates of query b, each scored
 * alpha*cls + MaxSim(query, doc); tail beyond R scored alpha*cls when PARTIAL;
 * rank by (score desc, doc_id asc); truncate to final_k. */
typedef struct {
  uint32_t n_queries;            /* B */
  uint32_t n_query_tokens;       /* q (rows of QueryEmbedding, types.hpp:34-43), 1..32 */
  const float* query_tokens;     /* B * q * d fp32, row-major */
  const uint32_t* cand_ids;      /* cand_offsets[B] entries */
  const float* cand_cls;         /* cls_score per candidate */
  const uint64_t* cand_offsets;  /* B + 1; HOST pointer unless ESPN_RERANK_DEVICE_OFFSETS */
  uint32_t rerank_count;         /* R */
  uint32_t final_k;              /* k (>= 1) */
  float alpha;                   /* CLS scaling (aggregate_score) */
  uint32_t flags;                /* ESPN_RERANK_* */
  uint32_t kernel;               /* espn_kernel */
  /* Optional HOST array of B per-query needed counts overriding min(R, n_b):
   * with doc-id sharding a shard's needed set is its share of the global
   * top-R prefix, which differs per query. NULL = min(R, n_b). */
  const uint32_t* needed_counts;
  uint32_t reserved[3];
} espn_rerank_args;

/* Per-query fetch accounting of a batch (QueryStats, pipeline.hpp:45-53), for
 * tiered tables: needed = first min(R, n) candidates; resident = needed rows
 * already in HBM; prefetched = needed host-tier rows staged by espn_gpu_prefetch
 * before scoring; missed = needed host-tier rows staged on the critical path;
 * bytes are table-row bytes moved over PCIe. */
typedef struct {
  uint64_t needed;
  uint64_t resident;
  uint64_t prefetched;
  uint64_t missed;
  uint64_t prefetch_bytes;
  uint64_t critical_bytes;
} espn_fetch_stats;

typedef struct {
  uint32_t* ids;        /* B * final_k */
  float* scores;        /* B * final_k */
  uint32_t* counts;     /* B: entries written for each query */
  float* bow_scores;    /* optional (WRITE_BOW): cand_offsets[B] MaxSim scores; entries of
                           candidates beyond the needed prefix (R) are 0 */
  espn_fetch_stats* fetch_stats; /* optional HOST array of B (synchronous calls) */
} espn_rerank_out;

/* Synchronous calls with pageable host buffers move their inputs with one
 * packed copy and their results with one; when the same shape (B, C, q, k, R,
 * alpha, flags) repeats on a workspace, the call replays a CUDA graph of its
 * device work captured on the second such call (results are identical; the
 * graph runs on `stream`). */
ESPN_API int espn_gpu_rerank(espn_gpu_table* table, espn_gpu_workspace* ws,
                    const espn_rerank_args* args, espn_rerank_out* out, void* stream);

/* Prefetcher (the paper's prefetch worker):
 * stages the host-tier rows of the NEXT batch's needed candidates into the
 * workspace's spare HBM staging buffer on `side_stream`, overlapping the
 * current batch's scoring.  `next` describes the batch exactly as it will be
 * passed to espn_gpu_rerank (DEVICE_IO; offsets host or device per its flags);
 * that call must carry ESPN_RERANK_PREFETCHED and waits on this staging.  A
 * no-op for untiered tables. */
ESPN_API int espn_gpu_prefetch(espn_gpu_table* table, espn_gpu_workspace* ws, const espn_rerank_args* next,
                      void* side_stream);

/* Prefetch hints (run_query stages (1)-(2), SPEC.md:276,
 * pipeline.hpp:56-64): stages the host-tier rows of an APPROXIMATE id list --
 * the IVF cursor's snapshot after delta clusters (ivf.hpp:67-68) -- into the
 * workspace's spare staging buffer on `side_stream`, while the ANN search
 * finishes.  hint_ids: CSR over n_queries by hint_offsets; a device array
 * when flags has ESPN_RERANK_DEVICE_IO, else a host array (copied through
 * pinned staging); hint_offsets is a host array unless flags also has
 * ESPN_RERANK_DEVICE_OFFSETS.  Ids of other shards or
 * unknown ids are ignored (hints are advisory).  A doc hinted by several
 * queries is staged once.  The next espn_gpu_rerank of this workspace carrying
 * ESPN_RERANK_PREFETCHED consumes the staging with ANY candidate lists: needed
 * host-tier rows found staged are hits (espn_fetch_stats.prefetched), the
 * others are copied on the critical path (missed).  Results are identical to
 * an unprefetched call.  The hinted rows use at most half of the staging
 * buffer; the rest is kept for the critical-path misses.  A no-op for
 * untiered tables. */
ESPN_API int espn_gpu_prefetch_hints(espn_gpu_table* table, espn_gpu_workspace* ws, uint32_t n_queries,
                                     const uint32_t* hint_ids, const uint64_t* hint_offsets, uint32_t flags,
                                     void* side_stream);

/* The disk-tier prefetcher (ESPN_TABLE_DISK_TIER; PAPER.md's SSD tier): the
 * caller read the records of some docs from the store file (espn_store_fetch,
 * O_DIRECT, queue_depth reads in flight) and hands their BOW rows over --
 * plain row-major table codes, doc ids[j]'s t rows at byte row_byte_off[j]
 * (16-byte aligned) of `rows` (a HOST buffer of rows_bytes; pinned makes the
 * upload asynchronous).  ids: HOST CSR over n_queries by id_offsets (per-query
 * byte accounting).  The rows are uploaded on side_stream, tiled into a free
 * staging slot and keyed by doc exactly like espn_gpu_prefetch_hints; the next
 * espn_gpu_rerank carrying ESPN_RERANK_PREFETCHED finds them (hits).  HBM-
 * resident docs, other shards' and unknown ids are skipped.  Works for any
 * streamed tiered table (host-tier docs may be handed over too).  The rows
 * handed over must fit the workspace's staging slot (staging_bytes, all of
 * it -- host-tier hints use half), else INVALID_CONFIG. */
ESPN_API int espn_gpu_prefetch_rows(espn_gpu_table* table, espn_gpu_workspace* ws, uint32_t n_queries,
                                    const uint32_t* ids, const uint64_t* id_offsets, const void* rows,
                                    const uint64_t* row_byte_off, uint64_t rows_bytes, void* side_stream);

/* Completes an ASYNC batch on its stream and reports device-side errors
 * (unknown doc id -> DATA_INTEGRITY, non-finite query/cls -> INVALID_INPUT,
 * duplicate candidate -> INVALID_INPUT). */
ESPN_API int espn_gpu_workspace_sync(espn_gpu_workspace* ws, void* stream);

/* Per-candidate fetch status of the workspace's last completed batch (the
 * record-level accounting behind QueryStats, pipeline.hpp:45-53): for each of
 * the first n candidates of the batch, 0 = the row was in HBM, 1 = staged by
 * the prefetcher before scoring (hit), 2 = staged on the critical path
 * (missed), 3 = not staged (staging overflow / unknown id).  Only the needed
 * candidates (first min(R, n_b) of each query) are defined.  HOST array. */
ESPN_API int espn_gpu_workspace_cand_status(espn_gpu_workspace* ws, uint8_t* out, uint64_t n);

/* Gather (StoreHandle::fetch_batch, store.hpp:91-94): copies the token rows of
 * `ids` (request order, duplicates allowed) into out_rows as CSR with
 * out_row_ptr[n+1] (token offsets).  ids/out_* are device pointers.
 * capacity_tokens bounds out_rows.  Unknown id -> INVALID_INPUT. */
ESPN_API int espn_gpu_gather(espn_gpu_table* table, const uint32_t* ids, uint64_t n,
                    uint16_t* out_rows, uint64_t* out_row_ptr, uint64_t capacity_tokens,
                    void* stream);

/* Host-memory convenience form of espn_gpu_gather (the C++ Store::fetch_batch
 * uses it): `ids` and the outputs are HOST pointers; out_row_ptr[n+1] receives
 * the request-order token offsets and out_rows the plain row-major codes
 * (capacity_tokens rows of d codes).  Synchronous. */
ESPN_API int espn_gpu_gather_host(espn_gpu_table* table, const uint32_t* ids, uint64_t n,
                         uint16_t* out_rows, uint64_t* out_row_ptr, uint64_t capacity_tokens);

/* Merge per-shard ranked lists (multi-GPU, doc-id sharding): for each of
 * n_queries queries, `n_lists` ranked lists of up to k entries, merged into
 * the global top-k by (score desc, doc_id asc).  List l's arrays start at
 * ids + l*list_stride, scores + l*list_stride, counts + l*list_stride
 * (list_stride in 4-byte elements; ids/scores are [query][k], counts [query]),
 * so one packed all-gather buffer can be merged in place.  Device pointers. */
ESPN_API int espn_gpu_merge_topk(const uint32_t* ids, const float* scores, const uint32_t* counts,
                        uint32_t n_lists, uint64_t list_stride, uint32_t n_queries, uint32_t k,
                        uint32_t* out_ids, float* out_scores, uint32_t* out_counts, void* stream);

/* ---- Persistent re-rank server ---------------------------------
 * A long-lived tcgen05 MaxSim kernel (one CTA per SM) fed by a device-side
 * batch queue: a served espn_gpu_rerank enqueues only the plan kernel (which
 * submits the planned batch to the queue) and a one-thread wait kernel; the
 * server's CTAs outlive batches, so one batch's start-up (CTA launch, prologue,
 * first unit's dependent loads) overlaps the previous batch's tail.  Served
 * batches: untiered table, tcgen05, fused top-k (final_k <= 32), the query
 * precision the server was started with (flags: ESPN_RERANK_QUERY_*).  While
 * the server runs, a non-servable tcgen05 batch on this table fails with
 * INVALID_STATE (it could not get an SM).  The server exits by itself after
 * idle_us without work (0 = 50 ms) -- a device-wide synchronisation in the
 * process (cudaDeviceSynchronize, cudaFree) waits at most that long -- and is
 * relaunched by the next served call made outside a stream capture.  Results
 * are identical to unserved calls.  espn_gpu_table_close stops it. */
ESPN_API int espn_gpu_server_start(espn_gpu_table* table, uint32_t flags, uint32_t idle_us);
ESPN_API int espn_gpu_server_stop(espn_gpu_table* table);
/* Stop the kernel (once drained) but keep the table attached: calls stay in
 * served mode (captures record plan + wait), the next eager served call or
 * espn_gpu_server_start relaunches it.  CUDA-graph replays of served batches
 * need a running server (otherwise they fail with INVALID_STATE). */
ESPN_API int espn_gpu_server_pause(espn_gpu_table* table);
ESPN_API int espn_gpu_server_running(const espn_gpu_table* table);
/* Diagnostics: {state, stop_req, exited CTAs, idle_ns, slot0 ready, slot0 done,
   slot0 done|merge counts, alive | launches << 8}. */
ESPN_API int espn_gpu_server_debug(const espn_gpu_table* table, uint64_t* out8);

/* ---- Multi-GPU --------------------------------
 * One process (rank) per GPU, or one process driving several GPUs.  Every rank
 * passes the SAME global batch (global doc ids; the candidate generator's
 * top-K per query, as run_batch hands it over, pipeline.hpp:81-85) and gets
 * the SAME global ranked lists back.  The placement follows the table:
 *   SHARD   (espn_table_desc.shard_count = G > 1; rank g opened shard g):
 *           each rank scores its own candidates (doc_id % G == g) -- needed
 *           count = its share of the query's global top-R prefix -- and ranks
 *           them; one ncclAllGather of the packed local top-k lists; merge.
 *   REPLICA (shard_count <= 1, every rank holds the whole table): rank g
 *           scores queries [g*ceil(B/G), (g+1)*ceil(B/G)); one ncclAllGather
 *           reassembles the batch.
 * Packed per-rank block (int32 words): [err bits, 0, 0, 0 | ids BQ x k |
 * scores BQ x k (fp32 bits) | counts BQ], BQ = B (SHARD) or ceil(B/G)
 * (REPLICA).  All steps run on `stream` (graph-capturable with DEVICE_IO |
 * DEVICE_OFFSETS | ASYNC); errors of any rank surface on every rank.  Not
 * combinable with WRITE_BOW, PREFETCHED or fetch_stats.
 * NCCL is loaded at run time (dlopen "libnccl.so.2", reusing an already
 * loaded copy, e.g. torch's); a nccl_comm is an ncclComm_t passed as void*. */
typedef struct { uint8_t internal[128]; } espn_nccl_id;  /* ncclUniqueId */
ESPN_API int espn_nccl_get_unique_id(espn_nccl_id* out);
/* ncclCommInitRank on `device` (the caller exchanges the id, e.g. over torch.distributed). */
ESPN_API int espn_nccl_comm_init(int nranks, const espn_nccl_id* id, int rank, int device, void** comm);
/* ncclCommInitAll: one communicator per device for a single process driving ndev GPUs. */
ESPN_API int espn_nccl_comm_init_all(int ndev, const int* devices, void** comms);
ESPN_API int espn_nccl_comm_destroy(void* comm);

/* Pack + all-gather + merge on `stream`.  nccl_comm: this rank's communicator
 * (SHARD: nranks == shard_count, rank == shard_index). */
ESPN_API int espn_gpu_rerank_sharded(espn_gpu_table* table, espn_gpu_workspace* ws, const espn_rerank_args* args,
                                     espn_rerank_out* out, void* nccl_comm, void* stream);
/* Single process, n GPUs (tables[i] on its own device, comms from
 * espn_nccl_comm_init_all): the same batch on every device, the NCCL calls in
 * one group (required when one thread drives several ranks).  outs[i] gets
 * the global result on device i (DEVICE_IO) or a host copy. */
ESPN_API int espn_gpu_rerank_sharded_multi(uint32_t n, espn_gpu_table* const* tables, espn_gpu_workspace* const* ws,
                                           const espn_rerank_args* args, espn_rerank_out* outs,
                                           void* const* nccl_comms, void* const* streams);
/* The two local phases without NCCL (tests, custom transports): pack this
 * rank's block into the workspace's send buffer (*send, *words on return:
 * device pointer and int32 count), then -- after the caller gathered the G
 * blocks contiguously into `recv` (device) -- merge them into `out`. */
ESPN_API int espn_gpu_shard_pack(espn_gpu_table* table, espn_gpu_workspace* ws, const espn_rerank_args* args,
                                 uint32_t nranks, uint32_t rank, void* stream, const int32_t** send, uint64_t* words);
ESPN_API int espn_gpu_shard_merge(espn_gpu_table* table, espn_gpu_workspace* ws, const espn_rerank_args* args,
                                  const int32_t* recv, uint32_t nranks, espn_rerank_out* out, void* stream);

/* Cumulative counters of a workspace since creation.  Reading them
 * synchronizes the device (completes PROFILE timings still in flight). */
typedef struct {
  uint64_t batches;
  uint64_t queries;
  uint64_t pairs_scored;       /* (query, candidate) MaxSim evaluations */
  uint64_t kernel_launches;    /* kernels of this library launched by the workspace */
  uint64_t profiled_batches;   /* batches run with ESPN_RERANK_PROFILE */
  double maxsim_ms;            /* summed CUDA-event time of the MaxSim kernel (PROFILE) */
  double topk_ms;              /* summed CUDA-event time of the top-k kernel (PROFILE) */
  uint64_t maxsim_device_ns;   /* PROFILE, tcgen05 path: device-timed MaxSim duration summed over
                                  launches (globaltimer, first CTA start -> last CTA end); also
                                  counts launches replayed from CUDA graphs */
  uint64_t maxsim_device_launches;
} espn_counters;
ESPN_API int espn_gpu_get_counters(const espn_gpu_workspace* ws, espn_counters* out);

/* Profiling only (no reference counterpart): per-kernel device timeline of
   the re-rank step, recorded when ESPN_DEBUG has bit 256 set.  out8 = {plan
   start, plan end, MaxSim start, MaxSim end, top-k start, top-k end, 0, 0} (globaltimer ns; min over CTA starts, max over CTA ends).
   Synchronises the device; reset != 0 re-arms the recorder. */
ESPN_API int espn_gpu_debug_timeline(int device, uint64_t* out8, int reset);

/* Synthetic MS-MARCO-shaped table generation on the device (bench/tests):
 * t ~ U{t_min..t_max} per doc and i.i.d. N(0,1) rows L2-normalised per row,
 * rounded to dtype with subnormals flushed.  The RNG
 * is counter-based and keyed by the GLOBAL doc id (and token index), so the
 * corpus is identical for every shard count and any doc can be regenerated
 * independently (paper_2312_05417_b200/synth.py mirrors it on the host).
 * Rows are written in the HBM tile layout: open with ESPN_TABLE_ROWS_TILED.
 * Generates shard `shard_index` of `shard_count` (local doc i = global id
 * i*shard_count + shard_index) with n_local_docs docs.  Writes row_ptr
 * (n_local_docs+1) and rows (device pointers; rows must hold
 * row_ptr[n_local_docs]*d codes -- call with rows == NULL first to fill
 * row_ptr only). */
ESPN_API int espn_gpu_synth_table(uint64_t n_local_docs, uint32_t d, uint32_t dtype, uint32_t t_min,
                         uint32_t t_max, uint64_t seed, uint32_t shard_count, uint32_t shard_index,
                         uint64_t* row_ptr, uint16_t* rows, void* stream);

/* K1 copy stage only, asynchronous on `stream` (for kernel timing / ncu):
 * out_row_ptr must already hold the request-order token offsets (as produced by
 * espn_gpu_gather with out_rows == NULL); ids must be known.  Device pointers. */
ESPN_API int espn_gpu_gather_rows(espn_gpu_table* table, const uint32_t* ids, uint64_t n,
                         const uint64_t* out_row_ptr, uint16_t* out_rows, void* stream);

/* Reference scoring primitives on the device, HOST arrays, synchronous (the
 * unmodified-header definitions of scoring.hpp in csrc/host/espn_ref_api.cpp):
 *   espn_gpu_maxsim_f32  maxsim_score (scoring.hpp:7-10) of one fp32 query
 *                        (nq x d) and one fp32 document (t x d): dot over k
 *                        ascending, max over doc tokens, sum over query tokens
 *                        ascending -- bit-exact with the reference order
 *                        (dot_f32 = the nq = t = 1 case);
 *   espn_gpu_rank        rank (scoring.hpp:16-18): sort by (score desc,
 *                        doc_id asc); duplicate ids or non-finite scores ->
 *                        INVALID_INPUT. */
ESPN_API int espn_gpu_maxsim_f32(const float* q, uint32_t nq, const float* doc, uint32_t t, uint32_t d, float* out,
                                 int device);
ESPN_API int espn_gpu_rank(const uint32_t* ids, const float* scores, uint64_t n, uint32_t* out_ids,
                           float* out_scores, int device);

ESPN_API const char* espn_last_error(void);
ESPN_API int espn_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ESPN_GPU_H */
