// espn_b200.cpp -- C++ host API (include/espn_b200.hpp) over the C-ABI.
// Marshalling, byte accounting and exception mapping only; every score is
// computed by libespn_gpu.so.
#include "espn_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <unordered_set>

namespace espn::gpu {
namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void check(int status) {
  if (status != ESPN_OK) throw_status(status);
}

std::uint16_t encode(float x, Dtype dt) {
  if (dt == Dtype::f16) {
    const _Float16 h = static_cast<_Float16>(x);  // IEEE binary16, round to nearest even
    std::uint16_t u;
    std::memcpy(&u, &h, 2);
    return u;
  }
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<std::uint16_t>((u >> 16) | 0x40u);  // quiet NaN
  return static_cast<std::uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

float decode(std::uint16_t c, Dtype dt) {
  if (dt == Dtype::f16) {
    _Float16 h;
    std::memcpy(&h, &c, 2);
    return static_cast<float>(h);
  }
  const std::uint32_t u = static_cast<std::uint32_t>(c) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

double percentile(std::vector<double> v, double p) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double r = p / 100.0 * static_cast<double>(v.size() - 1);
  const std::size_t lo = static_cast<std::size_t>(r);
  const std::size_t hi = std::min(lo + 1, v.size() - 1);
  return v[lo] + (v[hi] - v[lo]) * (r - static_cast<double>(lo));
}

}  // namespace

void throw_status(int status) { throw_status(status, espn_last_error()); }

void throw_status(int status, const std::string& msg) {
  switch (status) {
    case ESPN_E_INVALID_INPUT: throw InvalidInputError(msg);
    case ESPN_E_INVALID_STATE: throw InvalidStateError(msg);
    case ESPN_E_INVALID_CONFIG: throw InvalidConfigError(msg);
    case ESPN_E_FORMAT: throw FormatError(msg);
    case ESPN_E_IO: throw IoError(msg);
    case ESPN_E_DATA_INTEGRITY: throw DataIntegrityError(msg);
    default: throw Error(msg.empty() ? std::string("espn_gpu failure ") + std::to_string(status) : msg);
  }
}

// ---------------------------------------------------------------- Store
struct Store::WorkspaceCache {
  std::mutex mu;
  std::unordered_map<std::thread::id, std::unique_ptr<Reranker>> by_thread;
};

Reranker& Store::thread_reranker(std::uint32_t max_queries, std::uint32_t max_candidates,
                                 std::uint32_t max_query_tokens) const {
  std::lock_guard<std::mutex> lk(cache_->mu);
  auto& slot = cache_->by_thread[std::this_thread::get_id()];
  if (!slot || slot->max_queries() < max_queries || slot->max_candidates() < max_candidates ||
      slot->max_query_tokens() < max_query_tokens) {
    // grow geometrically so a slowly growing workload does not reallocate every call
    std::uint32_t q = max_queries, c = max_candidates, t = max_query_tokens;
    if (slot) {
      q = std::max(q, slot->max_queries());
      c = std::max(c, slot->max_candidates());
      t = std::max(t, slot->max_query_tokens());
    }
    slot.reset();
    slot = std::make_unique<Reranker>(*this, q, c, std::min<std::uint32_t>(t, 32));
  }
  return *slot;
}

std::pair<std::uint64_t, std::uint64_t> Store::record_io(DocId id) const {
  const std::uint64_t b = record_bytes(token_count(id));
  return {b, (b + 4095) / 4096};
}

QueryStats query_stats(const Store& store, QueryId query_id, std::span<const DocId> candidates, std::uint64_t n_needed,
                       std::span<const DocId> prefetched) {
  QueryStats st;
  st.query_id = query_id;
  st.needed_count = n_needed;
  st.prefetched_count = prefetched.size();
  std::unordered_set<DocId> pf(prefetched.begin(), prefetched.end());
  for (DocId id : prefetched) st.prefetch_bytes += store.record_io(id).first;
  std::uint64_t hits = 0;
  for (std::uint64_t j = 0; j < n_needed; ++j) {
    const DocId id = candidates[j];
    const auto [bytes, blocks] = store.record_io(id);
    st.needed_payload_bytes += bytes;
    if (pf.count(id)) {
      ++hits;
    } else {
      st.critical_fetch_bytes += bytes;
      st.critical_blocks_read += blocks;
    }
  }
  st.missed_count = n_needed - hits;
  st.hit_rate = n_needed ? static_cast<double>(hits) / static_cast<double>(n_needed) : 0.0;
  return st;
}

Store::Store(std::span<const std::uint64_t> row_ptr, std::span<const std::uint16_t> rows, std::uint32_t d,
             Dtype dtype, RecordLayout layout, int device, std::span<const std::uint8_t> resident)
    : cache_(std::make_unique<WorkspaceCache>()), d_(d), dtype_(dtype), layout_(layout), device_(device),
      row_ptr_(row_ptr.begin(), row_ptr.end()) {
  if (row_ptr.size() < 2) throw InvalidInputError("empty table");
  espn_table_desc desc{};
  desc.n_docs = row_ptr.size() - 1;
  desc.d = d;
  desc.dtype = static_cast<std::uint32_t>(dtype);
  desc.d_cls = layout.d_cls;
  desc.value_width = layout.value_width;
  desc.alignment = layout.alignment;
  desc.row_ptr = row_ptr.data();
  desc.rows = rows.data();
  desc.device = device;
  if (!resident.empty()) {
    if (resident.size() != desc.n_docs) throw InvalidInputError("resident mask size != n_docs");
    desc.resident = resident.data();
  }
  if (rows.size() < row_ptr.back() * d) throw InvalidInputError("rows shorter than row_ptr[n_docs] * d");
  check(espn_gpu_table_open(&desc, &table_));
}

Store Store::from_documents(const std::vector<EmbeddingMatrix>& docs, Dtype dtype, RecordLayout layout, int device) {
  if (docs.empty()) throw InvalidInputError("no documents");
  const std::uint32_t d = docs[0].cols;
  std::vector<std::uint64_t> rp(docs.size() + 1, 0);
  for (std::size_t i = 0; i < docs.size(); ++i) {
    const auto& m = docs[i];
    if (m.doc_id != i) throw InvalidInputError("doc ids must be dense [0, n) in order (store.hpp:20)");
    if (m.cols != d) throw InvalidInputError("inconsistent embedding dims");
    if (m.rows < 1) throw InvalidInputError("doc with t < 1 (types.hpp:64-68)");
    if (m.values.size() != static_cast<std::size_t>(m.rows) * m.cols) throw InvalidInputError("values size != rows*cols");
    rp[i + 1] = rp[i] + m.rows;
  }
  std::vector<std::uint16_t> codes(rp.back() * d);
  for (std::size_t i = 0; i < docs.size(); ++i) {
    const auto& v = docs[i].values;
    for (std::size_t j = 0; j < v.size(); ++j) {
      if (!std::isfinite(v[j])) throw InvalidInputError("non-finite embedding value (types.hpp:64-68)");
      codes[rp[i] * d + j] = encode(v[j], dtype);
    }
  }
  return Store(rp, codes, d, dtype, layout, device);
}

Store::Store(StreamedTag, std::span<const std::uint64_t> row_ptr, std::uint32_t d, Dtype dtype, RecordLayout layout,
             int device, std::span<const std::uint8_t> resident, bool disk_tier)
    : cache_(std::make_unique<WorkspaceCache>()), d_(d), dtype_(dtype), layout_(layout), device_(device),
      row_ptr_(row_ptr.begin(), row_ptr.end()), resident_(resident.begin(), resident.end()) {
  if (row_ptr.size() < 2) throw InvalidInputError("empty table");
  espn_table_desc desc{};
  desc.n_docs = row_ptr.size() - 1;
  desc.d = d;
  desc.dtype = static_cast<std::uint32_t>(dtype);
  desc.d_cls = layout.d_cls;
  desc.value_width = layout.value_width;
  desc.alignment = layout.alignment;
  desc.flags = ESPN_TABLE_STREAMED | (disk_tier ? ESPN_TABLE_DISK_TIER : 0u);
  desc.row_ptr = row_ptr.data();
  desc.rows = nullptr;
  desc.device = device;
  if (!resident.empty()) {
    if (resident.size() != desc.n_docs) throw InvalidInputError("resident mask size != n_docs");
    desc.resident = resident.data();
  }
  check(espn_gpu_table_open(&desc, &table_));
}

Store Store::streamed(std::span<const std::uint64_t> row_ptr, std::uint32_t d, Dtype dtype, RecordLayout layout,
                      int device, std::span<const std::uint8_t> resident, bool disk_tier) {
  return Store(StreamedTag{}, row_ptr, d, dtype, layout, device, resident, disk_tier);
}

void Store::load_rows(std::uint64_t doc_begin, std::uint64_t n_docs, std::span<const std::uint16_t> codes) {
  if (doc_begin + n_docs > this->n_docs()) throw InvalidInputError("load_rows: doc range beyond the table");
  if (codes.size() < (row_ptr_[doc_begin + n_docs] - row_ptr_[doc_begin]) * d_)
    throw InvalidInputError("load_rows: codes shorter than the docs' rows");
  check(espn_gpu_table_load_rows(table_, doc_begin, n_docs, codes.data()));
}

Store Store::open_store(const std::string& base, Dtype dtype, int device, std::span<const std::uint8_t> resident,
                        std::uint64_t chunk_bytes, bool disk_tier) {
  auto check_store = [](int st) {
    if (st != ESPN_OK) throw_status(st, espn_store_last_error());
  };
  espn_store_reader* rd = nullptr;
  espn_store_header h{};
  check_store(espn_store_open(base.c_str(), ESPN_READ_BUFFERED, 16, &rd, &h));
  std::unique_ptr<espn_store_reader, int (*)(espn_store_reader*)> guard(rd, espn_store_close);
  std::vector<espn_manifest_record> recs(h.count);
  check_store(espn_store_records(rd, recs.data()));
  std::vector<std::uint64_t> rp(h.count + 1, 0);
  for (std::uint64_t i = 0; i < h.count; ++i) rp[i + 1] = rp[i] + recs[i].token_count;
  Store s = streamed(rp, h.d, dtype, RecordLayout{h.d_cls, h.value_width, h.alignment}, device, resident, disk_tier);
  const std::uint64_t max_tok = std::max<std::uint64_t>(chunk_bytes / (2ull * h.d), 1);
  std::vector<std::uint16_t> codes;
  std::vector<std::uint64_t> lrp;
  for (std::uint64_t i = 0; i < h.count;) {
    std::uint64_t j = i + 1;
    while (j < h.count && rp[j + 1] - rp[i] <= max_tok) ++j;
    codes.resize((rp[j] - rp[i]) * h.d);
    lrp.resize(j - i + 1);
    check_store(espn_store_read_rows(rd, i, j - i, static_cast<std::uint32_t>(dtype), lrp.data(), codes.data()));
    s.load_rows(i, j - i, codes);
    i = j;
  }
  return s;
}

void build_store(const std::string& base, std::span<const std::uint64_t> row_ptr, std::span<const float> rows,
                 std::uint32_t d, std::span<const float> cls, RecordLayout layout) {
  if (row_ptr.empty()) throw InvalidInputError("row_ptr must hold n_docs + 1 offsets");
  const std::uint64_t n = row_ptr.size() - 1;
  if (rows.size() != row_ptr.back() * d) throw InvalidInputError("rows size != row_ptr[n] * d");
  if (!cls.empty() && cls.size() != n * layout.d_cls) throw InvalidInputError("cls size != n_docs * d_cls");
  const int st = espn_store_build(base.c_str(), n, d, layout.d_cls, layout.value_width, layout.alignment,
                                  row_ptr.data(), rows.data(), cls.empty() ? nullptr : cls.data());
  if (st != ESPN_OK) throw_status(st, espn_store_last_error());
}

Store::~Store() {
  cache_.reset();  // workspaces first: they belong to the table
  if (table_) espn_gpu_table_close(table_);
}
Store::Store(Store&& o) noexcept
    : cache_(std::make_unique<WorkspaceCache>()), table_(std::exchange(o.table_, nullptr)), d_(o.d_),
      dtype_(o.dtype_), layout_(o.layout_), device_(o.device_), row_ptr_(std::move(o.row_ptr_)) {
  o.cache_.reset();  // its workspaces point at the moved-from object
}
Store& Store::operator=(Store&& o) noexcept {
  if (this != &o) {
    cache_ = std::make_unique<WorkspaceCache>();
    o.cache_.reset();
    if (table_) espn_gpu_table_close(table_);
    table_ = std::exchange(o.table_, nullptr);
    d_ = o.d_;
    dtype_ = o.dtype_;
    layout_ = o.layout_;
    device_ = o.device_;
    row_ptr_ = std::move(o.row_ptr_);
  }
  return *this;
}

std::uint32_t Store::token_count(DocId id) const {
  if (id >= n_docs()) throw InvalidInputError("unknown doc id " + std::to_string(id));
  return static_cast<std::uint32_t>(row_ptr_[id + 1] - row_ptr_[id]);
}

std::uint64_t Store::record_bytes(std::uint32_t t) const {
  return (static_cast<std::uint64_t>(layout_.d_cls) + static_cast<std::uint64_t>(t) * d_) * layout_.value_width;
}

FetchResult Store::fetch_batch(std::span<const DocId> doc_ids) const {
  const double t0 = now_s();
  FetchResult res;
  const std::uint64_t n = doc_ids.size();
  std::vector<DocId> bad;
  for (DocId id : doc_ids)
    if (id >= n_docs()) bad.push_back(id);
  if (!bad.empty()) {
    std::string m = "unknown doc ids:";
    for (std::size_t i = 0; i < std::min<std::size_t>(bad.size(), 16); ++i) m += " " + std::to_string(bad[i]);
    throw InvalidInputError(m);  // store.hpp:92-93
  }
  if (n == 0) return res;
  // device buffers through the CUDA runtime the library links
  std::uint64_t tokens = 0;
  std::vector<std::uint64_t> out_rp(n + 1, 0);
  for (std::uint64_t i = 0; i < n; ++i) out_rp[i + 1] = out_rp[i] + token_count(doc_ids[i]);
  tokens = out_rp[n];
  std::vector<std::uint16_t> codes(tokens * d_);
  check(espn_gpu_gather_host(table_, doc_ids.data(), n, codes.data(), out_rp.data(), tokens));
  res.docs.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    auto& doc = res.docs[i].bow;
    doc.doc_id = doc_ids[i];
    doc.rows = static_cast<std::uint32_t>(out_rp[i + 1] - out_rp[i]);
    doc.cols = d_;
    doc.values.resize(static_cast<std::size_t>(doc.rows) * d_);
    for (std::size_t j = 0; j < doc.values.size(); ++j) doc.values[j] = decode(codes[out_rp[i] * d_ + j], dtype_);
    res.docs[i].cls.doc_id = doc_ids[i];
    const std::uint64_t pb = record_bytes(doc.rows);
    res.bytes_read += pb;
    res.blocks_read += (pb + 4095) / 4096;  // block = 4096 outside direct mode (store.hpp:63-65)
  }
  res.wall_time = now_s() - t0;
  return res;
}

// ---------------------------------------------------------------- Reranker
Reranker::Reranker(const Store& store, std::uint32_t max_queries, std::uint32_t max_candidates,
                   std::uint32_t max_query_tokens, std::uint64_t staging_bytes)
    : store_(&store) {
  espn_workspace_desc desc{};
  desc.staging_bytes = staging_bytes;
  desc.max_queries = std::max(max_queries, 1u);
  desc.max_candidates = std::max(max_candidates, 1u);
  desc.max_query_tokens = max_query_tokens;
  max_queries_ = desc.max_queries;
  max_candidates_ = desc.max_candidates;
  max_nq_ = max_query_tokens;
  check(espn_gpu_workspace_create(store.handle(), &desc, &ws_));
}

Reranker::~Reranker() {
  if (ws_) espn_gpu_workspace_destroy(ws_);
  if (pinned_) cudaFreeHost(pinned_);
}

std::uint64_t Reranker::prefetch_from_file(std::span<const CandidateList> lists, std::uint32_t top_k,
                                           espn_store_reader* reader, void* side_stream) {
  if (!reader) throw InvalidInputError("prefetch_from_file: null store reader");
  if (store_->layout().value_width != 2 || store_->dtype() != Dtype::f16)
    throw InvalidConfigError("prefetch_from_file: the file's values must be the table's codes "
                             "(value_width 2 store, f16 table)");
  const std::uint32_t B = static_cast<std::uint32_t>(lists.size());
  if (B == 0) return 0;
  // the needed docs of each list that are not in HBM (store.hpp:91-94 order)
  std::vector<std::uint64_t> off(B + 1, 0);
  std::vector<std::uint32_t> ids;
  for (std::uint32_t b = 0; b < B; ++b) {
    const std::size_t n = lists[b].entries.size();
    const std::size_t m = top_k ? std::min<std::size_t>(n, top_k) : n;
    for (std::size_t j = 0; j < m; ++j) {
      const DocId id = lists[b].entries[j].doc_id;
      if (id < store_->n_docs() && !store_->resident(id)) ids.push_back(static_cast<std::uint32_t>(id));
    }
    off[b + 1] = ids.size();
  }
  auto check_store = [](int st) {
    if (st != ESPN_OK) throw_status(st, espn_store_last_error());
  };
  const std::uint64_t n = ids.size();
  std::vector<std::uint64_t> rec_off(n + 1, 0);
  std::uint64_t br = 0, bl = 0;
  double secs = 0;
  check_store(espn_store_fetch(reader, ids.data(), n, nullptr, rec_off.data(), 0, &br, &bl, &secs));  // sizes
  if (rec_off[n] > pinned_cap_) {
    if (pinned_) cudaFreeHost(pinned_);
    pinned_ = nullptr;
    pinned_cap_ = 0;
    if (cudaHostAlloc(reinterpret_cast<void**>(&pinned_), rec_off[n], cudaHostAllocDefault) != cudaSuccess)
      throw espn::Error("prefetch_from_file: pinned buffer allocation failed");
    pinned_cap_ = rec_off[n];
  }
  check_store(espn_store_fetch(reader, ids.data(), n, pinned_, rec_off.data(), pinned_cap_, &br, &bl, &secs));
  // each record is [CLS d_cls x value_width | BOW rows]: the rows follow the CLS
  std::vector<std::uint64_t> row_off(n);
  const std::uint64_t cls_bytes = static_cast<std::uint64_t>(store_->layout().d_cls) * store_->layout().value_width;
  for (std::uint64_t j = 0; j < n; ++j) row_off[j] = rec_off[j] + cls_bytes;
  check(espn_gpu_prefetch_rows(store_->handle(), ws_, B, ids.data(), off.data(), pinned_, row_off.data(), rec_off[n],
                               side_stream));
  hint_ids_ = std::move(ids);  // the prefetched ids of the next prefetched rerank (QueryStats)
  hint_off_ = std::move(off);
  return br;
}

espn_counters Reranker::counters() const {
  espn_counters c{};
  check(espn_gpu_get_counters(ws_, &c));
  return c;
}

void Reranker::prefetch_hints(std::span<const CandidateList> snapshots, std::uint32_t top_k, void* side_stream) {
  const std::uint32_t B = static_cast<std::uint32_t>(snapshots.size());
  if (B == 0) return;
  std::vector<std::uint64_t> off(B + 1, 0);
  for (std::uint32_t b = 0; b < B; ++b) {
    const std::size_t n = snapshots[b].entries.size();
    off[b + 1] = off[b] + (top_k ? std::min<std::size_t>(n, top_k) : n);
  }
  std::vector<std::uint32_t> ids(off[B]);
  for (std::uint32_t b = 0; b < B; ++b)
    for (std::uint64_t j = 0; j < off[b + 1] - off[b]; ++j) ids[off[b] + j] = snapshots[b].entries[j].doc_id;
  check(espn_gpu_prefetch_hints(store_->handle(), ws_, B, ids.data(), off.data(), 0u, side_stream));
  hint_ids_ = std::move(ids);  // the prefetched ids of the next prefetched rerank (QueryStats)
  hint_off_ = std::move(off);
}

BatchResult Reranker::rerank(std::span<const QueryEmbedding> queries, std::span<const CandidateList> candidates,
                             const PipelineConfig& config, Kernel kernel, bool prefetched) {
  if (queries.size() != candidates.size()) throw InvalidInputError("queries and candidate lists differ in length");
  BatchResult res;
  const std::uint32_t B = static_cast<std::uint32_t>(queries.size());
  if (B == 0) return res;
  const std::uint32_t d = store_->d();
  const std::uint32_t nq = queries[0].rows;
  std::vector<float> qt(static_cast<std::size_t>(B) * nq * d);
  std::vector<std::uint64_t> off(B + 1, 0);
  for (std::uint32_t b = 0; b < B; ++b) {
    const auto& q = queries[b];
    if (q.cols != d) throw InvalidInputError("query dim " + std::to_string(q.cols) + " != table dim " + std::to_string(d));
    if (q.rows != nq) throw InvalidInputError("all queries of a batch must have the same token count");
    if (q.tokens.size() != static_cast<std::size_t>(q.rows) * q.cols) throw InvalidInputError("tokens size != rows*cols");
    std::copy(q.tokens.begin(), q.tokens.end(), qt.begin() + static_cast<std::size_t>(b) * nq * d);
    off[b + 1] = off[b] + candidates[b].entries.size();
  }
  std::vector<std::uint32_t> ids(off[B]);
  std::vector<float> cls(off[B]);
  for (std::uint32_t b = 0; b < B; ++b)
    for (std::size_t j = 0; j < candidates[b].entries.size(); ++j) {
      ids[off[b] + j] = candidates[b].entries[j].doc_id;
      cls[off[b] + j] = candidates[b].entries[j].cls_score;
    }
  const std::uint32_t k = config.final_k;
  std::vector<std::uint32_t> out_ids(static_cast<std::size_t>(B) * k), out_n(B);
  std::vector<float> out_sc(static_cast<std::size_t>(B) * k);
  espn_rerank_args a{};
  a.n_queries = B;
  a.n_query_tokens = nq;
  a.query_tokens = qt.data();
  a.cand_ids = ids.data();
  a.cand_cls = cls.data();
  a.cand_offsets = off.data();
  a.rerank_count = config.rerank_count;
  a.final_k = k;
  a.alpha = config.alpha;
  a.flags = (config.partial_rerank_enabled ? ESPN_RERANK_PARTIAL : 0u) | (prefetched ? ESPN_RERANK_PREFETCHED : 0u);
  a.kernel = static_cast<std::uint32_t>(kernel);
  std::vector<espn_fetch_stats> fs(B);
  espn_rerank_out o{};
  o.ids = out_ids.data();
  o.scores = out_sc.data();
  o.counts = out_n.data();
  o.fetch_stats = fs.data();
  const double t0 = now_s();
  check(espn_gpu_rerank(store_->handle(), ws_, &a, &o, nullptr));
  const double wall = now_s() - t0;
  res.rankings.resize(B);
  res.stats.resize(B);
  std::vector<double> lat(B, wall);
  for (std::uint32_t b = 0; b < B; ++b) {
    auto& rl = res.rankings[b];
    rl.entries.resize(out_n[b]);
    for (std::uint32_t i = 0; i < out_n[b]; ++i)
      rl.entries[i] = ScoredDoc{out_ids[static_cast<std::size_t>(b) * k + i], out_sc[static_cast<std::size_t>(b) * k + i]};
    // QueryStats (pipeline.hpp:36-54) as the reference defines them: the
    // prefetched ids are the query's snapshot hints (prefetched batches only)
    const std::uint64_t n = off[b + 1] - off[b];
    std::span<const DocId> pf;
    if (prefetched && b + 1 < hint_off_.size())
      pf = std::span<const DocId>(hint_ids_.data() + hint_off_[b], hint_off_[b + 1] - hint_off_[b]);
    auto& st = res.stats[b];
    st = query_stats(*store_, queries[b].query_id, std::span<const DocId>(ids.data() + off[b], n),
                     std::min<std::uint64_t>(n, config.rerank_count), pf);
    st.rerank_time = wall;
    st.total_time = wall;
  }
  last_fs_ = std::move(fs);
  res.batch.n_queries = B;
  res.batch.mean_latency = wall;
  res.batch.p50_latency = percentile(lat, 50);
  res.batch.p99_latency = percentile(lat, 99);
  res.batch.wall_time = wall;
  for (const auto& st : res.stats) res.batch.total_critical_fetch_bytes += st.critical_fetch_bytes;
  return res;
}

// ---------------------------------------------------------------- free functions
BatchResult rerank_batch(std::span<const QueryEmbedding> queries, std::span<const CandidateList> candidates,
                         const Store& store, const PipelineConfig& config) {
  std::uint64_t c = 0;
  std::uint32_t nq = 1;
  for (const auto& cl : candidates) c += cl.entries.size();
  if (!queries.empty()) nq = std::max<std::uint32_t>(queries[0].rows, 1);
  Reranker& rr = store.thread_reranker(static_cast<std::uint32_t>(queries.size()),
                                       static_cast<std::uint32_t>(std::max<std::uint64_t>(c, 1)),
                                       std::min<std::uint32_t>(nq, 32));
  return rr.rerank(queries, candidates, config);
}

std::pair<RankedList, QueryStats> rerank_candidates(const QueryEmbedding& query, const CandidateList& candidates,
                                                    const Store& store, const PipelineConfig& config) {
  BatchResult r = rerank_batch(std::span<const QueryEmbedding>(&query, 1),
                               std::span<const CandidateList>(&candidates, 1), store, config);
  return {std::move(r.rankings[0]), r.stats[0]};
}

// ---------------------------------------------------------------- quality harness (metrics.hpp:10-20)
double mrr_at_k(const ResultsByQuery& results, const Qrels& qrels, int k) {
  if (k < 1) throw InvalidInputError("k must be >= 1 (SPEC.md:74)");
  if (qrels.empty()) return 0.0;
  double sum = 0.0;
  for (const auto& [qid, rel] : qrels) {
    auto it = results.find(qid);
    if (it == results.end()) continue;
    const auto& e = it->second.entries;
    const std::size_t n = std::min<std::size_t>(e.size(), static_cast<std::size_t>(k));
    for (std::size_t r = 0; r < n; ++r)
      if (rel.count(e[r].doc_id)) {
        sum += 1.0 / static_cast<double>(r + 1);
        break;
      }
  }
  return sum / static_cast<double>(qrels.size());
}

double recall_at_k(const ResultsByQuery& results, const Qrels& qrels, int k) {
  if (k < 1) throw InvalidInputError("k must be >= 1 (SPEC.md:82)");
  if (qrels.empty()) return 0.0;
  double sum = 0.0;
  for (const auto& [qid, rel] : qrels) {
    auto it = results.find(qid);
    if (it == results.end() || rel.empty()) continue;
    const auto& e = it->second.entries;
    const std::size_t n = std::min<std::size_t>(e.size(), static_cast<std::size_t>(k));
    std::size_t hit = 0;
    for (std::size_t r = 0; r < n; ++r) hit += rel.count(e[r].doc_id);
    sum += static_cast<double>(hit) / static_cast<double>(rel.size());
  }
  return sum / static_cast<double>(qrels.size());
}

Qrels load_qrels(std::istream& in) {
  Qrels q;
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ls(line);
    long long qid, iter, did, relv;
    std::string extra;
    if (!(ls >> qid >> iter >> did >> relv) || (ls >> extra) || qid < 0 || did < 0 || qid > 0xFFFFFFFFLL ||
        did > 0xFFFFFFFFLL)
      throw FormatError("qrels line " + std::to_string(lineno) + ": expected `query_id 0 doc_id relevance`");
    if (relv > 0) q[static_cast<QueryId>(qid)].insert(static_cast<DocId>(did));
  }
  return q;
}

Qrels load_qrels(const std::filesystem::path& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open qrels file " + path.string());
  return load_qrels(f);
}

}  // namespace espn::gpu

// ---------------------------------------------------------------- serving loop (include/espn_host.h)
#include <cuda_runtime_api.h>
#include <deque>

#include "espn_host.h"

extern "C" int espn_host_run_batches(espn_gpu_table* table, espn_gpu_workspace* const* ws, void* const* streams,
                                     uint32_t lanes, uint32_t depth, const espn_rerank_args* batches,
                                     espn_rerank_out* outs, uint32_t n, double* seconds) {
  if (!table || !ws || !streams || !batches || !outs || lanes == 0) return ESPN_E_INVALID_INPUT;
  depth = std::max(depth, 1u);
  std::vector<std::deque<cudaEvent_t>> inflight(lanes);
  std::vector<cudaEvent_t> pool;
  auto get_event = [&]() -> cudaEvent_t {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
  };
  int status = ESPN_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t i = 0; i < n && status == ESPN_OK; ++i) {
    const uint32_t l = i % lanes;
    auto& q = inflight[l];
    if (q.size() >= depth) {  // the lane's oldest batch must finish before its buffers are reused
      cudaEventSynchronize(q.front());
      pool.push_back(q.front());
      q.pop_front();
    }
    espn_rerank_args a = batches[i];
    a.flags |= ESPN_RERANK_ASYNC;
    status = espn_gpu_rerank(table, ws[l], &a, &outs[i], streams[l]);
    if (status == ESPN_OK) {
      cudaEvent_t e = get_event();
      cudaEventRecord(e, static_cast<cudaStream_t>(streams[l]));
      q.push_back(e);
    }
  }
  for (uint32_t l = 0; l < lanes; ++l) {
    const int st = espn_gpu_workspace_sync(ws[l], streams[l]);  // completes the lane, reports device errors
    if (status == ESPN_OK) status = st;
  }
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto& q : inflight)
    for (cudaEvent_t e : q) cudaEventDestroy(e);
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
  return status;
}
