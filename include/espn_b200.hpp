// espn_b200.hpp -- C++ host API of the B200 re-rank path (the drop-in for
// stages 3-6 of espn::run_query, proj/include/espn/pipeline.hpp:56-64).
//
// It is a thin layer over the C-ABI in espn_gpu.h: argument marshalling,
// QueryStats accounting and the error mapping of error.hpp:8-42 (status code
// -> exception class).  No compute happens here.
//
// Carrier types.  Built with -DESPN_B200_WITH_REFERENCE_HEADERS and the
// reference's include directory on the path, this header uses the reference's
// own espn::QueryEmbedding / CandidateList / PipelineConfig / QueryStats /
// RankedList / FetchResult / error classes (pipeline.hpp pulls types.hpp,
// ivf.hpp, store.hpp), so code written against the reference compiles
// unchanged.  Without it, source-compatible declarations of the same types
// (same names, members and defaults) are provided below.
//
// New seam: the reference has no "candidates in -> ranked
// out" function; espn::gpu::rerank_candidates / rerank_batch are that seam,
// and espn::gpu::Store is the HBM tier that replaces StoreHandle for the
// re-rank path (store.hpp:80-107).
#pragma once

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <istream>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "espn_gpu.h"
#include "espn_store.h"

#if defined(ESPN_B200_WITH_REFERENCE_HEADERS)
#include "espn/error.hpp"
#include "espn/pipeline.hpp"
#else
#include <algorithm>
#include <stdexcept>

namespace espn {

using DocId = std::uint32_t;
using QueryId = std::uint32_t;

// error.hpp:8-42
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
struct InvalidInputError : Error { using Error::Error; };
struct InvalidStateError : Error { using Error::Error; };
struct InvalidConfigError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DataIntegrityError : Error { using Error::Error; };

// types.hpp:16-55 (t x d / q x d row-major fp32)
struct EmbeddingMatrix {
  DocId doc_id = 0;
  std::uint32_t rows = 0;
  std::uint32_t cols = 0;
  std::vector<float> values;
};
struct ClsVector {
  DocId doc_id = 0;
  std::vector<float> values;
};
struct QueryEmbedding {
  QueryId query_id = 0;
  std::vector<float> cls;
  std::uint32_t rows = 0;
  std::uint32_t cols = 0;
  std::vector<float> tokens;
};
struct ScoredDoc {
  DocId doc_id = 0;
  float score = 0.0f;
};
struct RankedList {
  std::vector<ScoredDoc> entries;  // (score desc, doc_id asc), unique ids
};

// ivf.hpp:40-50
struct Candidate {
  DocId doc_id = 0;
  float cls_score = 0.0f;
};
struct CandidateList {
  std::vector<Candidate> entries;  // (cls_score desc, doc_id asc), deduplicated
  std::size_t clusters_visited = 0;
};

// pipeline.hpp:11-29
struct PipelineConfig {
  std::uint32_t nprobe = 0;
  double prefetch_step_pct = 10.0;
  std::uint32_t rerank_count = 0;
  std::uint32_t final_k = 10;
  std::uint32_t prefetch_top_k = 0;
  std::uint32_t candidate_k = 0;
  float alpha = 1.0f;
  bool prefetch_enabled = true;
  bool partial_rerank_enabled = false;

  std::uint32_t effective_prefetch_top_k() const { return prefetch_top_k ? prefetch_top_k : rerank_count; }
  std::uint32_t effective_candidate_k() const { return candidate_k ? candidate_k : std::max(rerank_count, final_k); }
};

// pipeline.hpp:36-54
struct QueryStats {
  QueryId query_id = 0;
  double ann_time = 0.0;
  double prefetch_time = 0.0;
  double early_rerank_time = 0.0;
  double critical_fetch_time = 0.0;
  double rerank_time = 0.0;
  double total_time = 0.0;
  std::uint64_t prefetched_count = 0;
  std::uint64_t needed_count = 0;
  std::uint64_t missed_count = 0;
  double hit_rate = 0.0;
  std::uint64_t prefetch_bytes = 0;
  std::uint64_t critical_fetch_bytes = 0;
  std::uint64_t critical_blocks_read = 0;
  std::uint64_t needed_payload_bytes = 0;
};

// pipeline.hpp:66-79
struct BatchStats {
  std::size_t n_queries = 0;
  double mean_latency = 0.0;
  double p50_latency = 0.0;
  double p99_latency = 0.0;
  double wall_time = 0.0;
  std::uint64_t total_critical_fetch_bytes = 0;
};
struct BatchResult {
  std::vector<RankedList> rankings;
  std::vector<QueryStats> stats;
  BatchStats batch;
};

// store.hpp:61-71
struct FetchedDoc {
  ClsVector cls;
  EmbeddingMatrix bow;
};
struct FetchResult {
  std::vector<FetchedDoc> docs;
  std::uint64_t bytes_read = 0;
  std::uint64_t blocks_read = 0;
  double wall_time = 0.0;
};

// types.hpp:57-62
using Qrels = std::map<QueryId, std::set<DocId>>;
using ResultsByQuery = std::map<QueryId, RankedList>;

}  // namespace espn
#endif

namespace espn::gpu {

enum class Dtype : std::uint32_t { f16 = ESPN_DTYPE_F16, bf16 = ESPN_DTYPE_BF16 };
enum class Kernel : std::uint32_t { automatic = ESPN_KERNEL_AUTO, tcgen05 = ESPN_KERNEL_TCGEN05, simt = ESPN_KERNEL_SIMT,
                                        small = ESPN_KERNEL_SMALL };

// Throws the espn:: exception class matching an espn_status (error.hpp:8-42).
void throw_status(int status);
void throw_status(int status, const std::string& message);

// Record layout of the reference store (store.hpp:25-34), used only for the
// QueryStats / FetchResult byte counters.
struct RecordLayout {
  std::uint32_t d_cls = 128;
  std::uint32_t value_width = 2;
  std::uint32_t alignment = 4096;
};

// The HBM tier of the embedding table: the re-rank path's StoreHandle.
// Built from CSR token rows (doc i = rows[row_ptr[i]*d, row_ptr[i+1]*d), 2-byte
// codes of `dtype`) or from reference EmbeddingMatrix docs (fp32, rounded to
// dtype).  Move-only; shareable read-only across threads.
class Store {
 public:
  // resident (optional, n_docs flags): docs with resident[i] == 0 live in a
  // pinned-host tier and are staged into HBM per batch (prefetched through
  // Reranker::prefetch_hints, or on the critical path).
  Store(std::span<const std::uint64_t> row_ptr, std::span<const std::uint16_t> rows, std::uint32_t d,
        Dtype dtype = Dtype::f16, RecordLayout layout = {}, int device = 0,
        std::span<const std::uint8_t> resident = {});
  // docs[i].doc_id must equal i (dense ids, store.hpp:20)
  static Store from_documents(const std::vector<EmbeddingMatrix>& docs, Dtype dtype = Dtype::f16,
                              RecordLayout layout = {}, int device = 0);
  // open_store (store.hpp:111-112) for the GPU table, streamed from a .espn
  // store (include/espn_store.h): allocated from the manifest -- only the
  // resident docs in HBM when `resident` is given -- and filled in chunks of
  // chunk_bytes, so the store is never read whole; the record layout comes
  // from the manifest.
  // disk_tier (with `resident`): the non-resident docs stay ONLY in the file
  // (ESPN_TABLE_DISK_TIER, the paper's SSD tier); batches that need them are
  // staged by Reranker::prefetch_from_file and re-ranked with prefetched = true.
  static Store open_store(const std::string& base, Dtype dtype = Dtype::f16, int device = 0,
                          std::span<const std::uint8_t> resident = {}, std::uint64_t chunk_bytes = 64ull << 20,
                          bool disk_tier = false);
  // ESPN_TABLE_STREAMED: an empty table allocated from row_ptr (+ resident),
  // filled in doc order by load_rows (plain 2-byte codes of the next docs).
  static Store streamed(std::span<const std::uint64_t> row_ptr, std::uint32_t d, Dtype dtype = Dtype::f16,
                        RecordLayout layout = {}, int device = 0, std::span<const std::uint8_t> resident = {},
                        bool disk_tier = false);
  void load_rows(std::uint64_t doc_begin, std::uint64_t n_docs, std::span<const std::uint16_t> codes);
  ~Store();
  Store(Store&&) noexcept;
  Store& operator=(Store&&) noexcept;
  Store(const Store&) = delete;
  Store& operator=(const Store&) = delete;

  espn_gpu_table* handle() const { return table_; }
  std::uint32_t d() const { return d_; }
  Dtype dtype() const { return dtype_; }
  const RecordLayout& layout() const { return layout_; }
  std::uint64_t n_docs() const { return row_ptr_.empty() ? 0 : row_ptr_.size() - 1; }
  std::uint32_t token_count(DocId id) const;
  std::uint64_t record_bytes(std::uint32_t token_count) const;

  // StoreHandle::fetch_batch (store.hpp:91-94): request order, duplicates
  // allowed, unknown ids -> InvalidInputError; values decoded to fp32.
  FetchResult fetch_batch(std::span<const DocId> doc_ids) const;

  // Per-record I/O of the reference store (store.hpp:61-65): payload bytes
  // and ceil(bytes / 4096) blocks of doc `id`'s record (buffered reads).
  std::pair<std::uint64_t, std::uint64_t> record_io(DocId id) const;

  // The calling thread's cached workspace, at least this large (the free
  // rerank_batch / rerank_candidates reuse it instead of allocating one per
  // call; one per thread, so concurrent callers never share scratch).
  class Reranker& thread_reranker(std::uint32_t max_queries, std::uint32_t max_candidates,
                                  std::uint32_t max_query_tokens) const;

  // Tier of doc `id` (tiered stores): true = HBM-resident.
  bool resident(DocId id) const { return resident_.empty() || resident_[id] != 0; }

 private:
  struct WorkspaceCache;
  struct StreamedTag {};
  Store(StreamedTag, std::span<const std::uint64_t> row_ptr, std::uint32_t d, Dtype dtype, RecordLayout layout,
        int device, std::span<const std::uint8_t> resident, bool disk_tier);
  std::unique_ptr<WorkspaceCache> cache_;
  espn_gpu_table* table_ = nullptr;
  std::uint32_t d_ = 0;
  Dtype dtype_ = Dtype::f16;
  RecordLayout layout_;
  int device_ = 0;
  std::vector<std::uint64_t> row_ptr_;  // host copy for byte accounting
  std::vector<std::uint8_t> resident_;  // tiered stores: the residency mask
};

// A reusable batch context (one workspace = per-stream scratch).  Not
// thread-safe: one in-flight batch per Reranker.
class Reranker {
 public:
  Reranker(const Store& store, std::uint32_t max_queries, std::uint32_t max_candidates,
           std::uint32_t max_query_tokens = 32, std::uint64_t staging_bytes = 0);
  ~Reranker();
  Reranker(const Reranker&) = delete;
  Reranker& operator=(const Reranker&) = delete;

  // run_batch (pipeline.hpp:81-85) restricted to stages 3-6: one device pass
  // for the whole batch, per-query results identical to single-query calls.
  // prefetched: the batch consumes the staging of the last prefetch_hints
  // call (tiered stores).  QueryStats follow the reference exactly
  // (pipeline.hpp:45-53, the oracle's eo_rerank_query): prefetched = the
  // query's snapshot ids given to prefetch_hints (none when !prefetched),
  // hits = needed ∩ prefetched, per-record byte / block counters.  The tier
  // view (rows resident in HBM vs staged over PCIe) is last_fetch_stats().
  BatchResult rerank(std::span<const QueryEmbedding> queries, std::span<const CandidateList> candidates,
                     const PipelineConfig& config, Kernel kernel = Kernel::automatic, bool prefetched = false);

  // Device fetch accounting of the last rerank, per query (espn_fetch_stats).
  const std::vector<espn_fetch_stats>& last_fetch_stats() const { return last_fs_; }
  std::uint32_t max_queries() const { return max_queries_; }
  std::uint32_t max_candidates() const { return max_candidates_; }
  std::uint32_t max_query_tokens() const { return max_nq_; }

  // run_query stages (1)-(2) (pipeline.hpp:56-64): stage the host-tier rows of
  // the cursors' snapshots after delta clusters (SearchCursor::snapshot,
  // ivf.hpp:67-68; the first top_k entries of each, 0 = all) on side_stream,
  // while the search finishes.  The next rerank(..., prefetched = true)
  // resolves its needed rows against them.  No-op for an all-HBM store.
  void prefetch_hints(std::span<const CandidateList> snapshots, std::uint32_t top_k = 0,
                      void* side_stream = nullptr);

  // The disk tier's prefetcher (ESPN_TABLE_DISK_TIER stores): reads the
  // records of each list's first `top_k` entries (0 = all) that are not in
  // HBM from the store file through `reader` (espn_store_fetch: O_DIRECT /
  // buffered / mmap, queue_depth reads in flight -- the reference's own
  // StoreHandle::fetch_batch) into a pinned buffer and stages their rows
  // (espn_gpu_prefetch_rows) on side_stream.  Pass the final lists with
  // top_k = rerank_count so every needed doc is staged; the next
  // rerank(..., prefetched = true) finds them.  Returns the bytes read.
  std::uint64_t prefetch_from_file(std::span<const CandidateList> lists, std::uint32_t top_k,
                                   espn_store_reader* reader, void* side_stream = nullptr);

  espn_counters counters() const;

 private:
  const Store* store_;
  espn_gpu_workspace* ws_ = nullptr;
  std::uint32_t max_queries_ = 0, max_candidates_ = 0, max_nq_ = 0;
  std::vector<std::uint32_t> hint_ids_;   // last prefetch_hints snapshot (CSR)
  std::vector<std::uint64_t> hint_off_;
  std::vector<espn_fetch_stats> last_fs_;
  std::uint8_t* pinned_ = nullptr;  // prefetch_from_file: record payloads (cudaHostAlloc, grown)
  std::uint64_t pinned_cap_ = 0;
};

// QueryStats of one query exactly as the reference computes them
// (pipeline.hpp:45-53): needed = the first n_needed candidates, prefetched =
// the ids the prefetcher fetched; record sizes from the store's manifest layout.
QueryStats query_stats(const Store& store, QueryId query_id, std::span<const DocId> candidates, std::uint64_t n_needed,
                       std::span<const DocId> prefetched);

// build_store (store.hpp:48-51) from a CSR of fp32 rows (+ n_docs * d_cls CLS
// values, or empty for zeros): writes <base>.espn / .manifest / .manifest.json.
void build_store(const std::string& base, std::span<const std::uint64_t> row_ptr, std::span<const float> rows,
                 std::uint32_t d, std::span<const float> cls = {}, RecordLayout layout = {});

// The seam: stages 3-6 of run_query for one query (SPEC.md:276 (3)-(6)).
std::pair<RankedList, QueryStats> rerank_candidates(const QueryEmbedding& query, const CandidateList& candidates,
                                                    const Store& store, const PipelineConfig& config);

// Batched form (run_batch restricted to stages 3-6).
BatchResult rerank_batch(std::span<const QueryEmbedding> queries, std::span<const CandidateList> candidates,
                         const Store& store, const PipelineConfig& config);

// Quality harness (metrics.hpp:10-20), to
// check that re-ranking on the GPU preserves retrieval quality.  Same
// definitions as the reference's espn::mrr_at_k / recall_at_k / load_qrels:
// averages run over the qrels queries in id order, a query without results
// (or without relevant docs) contributes 0, k < 1 -> InvalidInputError.
double mrr_at_k(const ResultsByQuery& results, const Qrels& qrels, int k);
double recall_at_k(const ResultsByQuery& results, const Qrels& qrels, int k);
// TREC qrels: `query_id 0 doc_id relevance` per line, relevance > 0 marks a
// relevant doc; blank lines skipped; anything else -> FormatError.
Qrels load_qrels(std::istream& in);
Qrels load_qrels(const std::filesystem::path& path);

}  // namespace espn::gpu
