// espn_ref_api.cpp -- the reference's own C++ API, compiled against its
// UNMODIFIED headers (/root/reference/proj/include/espn/*.hpp), defined over
// the B200 path.  The reference ships declarations only; a
// program written against them links lib/libespn_refapi.so instead.
//
//   types.hpp:64-68      validate_embedding / validate_cls / validate_query   host checks
//   scoring.hpp:7-21     maxsim_score, dot_f32 -> espn_gpu_maxsim_f32 (device, the reference's fp32 order)
//                        rank            -> espn_gpu_rank (device sort + duplicate / finite checks)
//                        aggregate_score -> one fp32 multiply then add (this TU: -ffp-contract=off)
//   store.hpp:13-112     store_paths, build_store, save/load_manifest -> libespn_store.so;
//                        open_store + StoreHandle::fetch_batch -> the file-backed reader (direct /
//                        buffered / mmap, queue_depth reads in flight, the reference's counters),
//                        values decoded with the reference's own half.hpp
//   kmeans.hpp, ivf.hpp  k-means++ / Lloyd, IVF, SearchCursor: host (the candidate generator runs
//                        on the CPU, as in the paper; it feeds the hot path, it is not on it)
//   pipeline.hpp         run_query / run_batch / measure_hit_rate: the IVF stages on the host, the
//                        delta-snapshot as prefetch hints, stages 3-6 on the GPU (espn::gpu::Reranker);
//                        QueryStats with the reference's exact semantics
//   metrics.hpp          mrr_at_k / recall_at_k / load_qrels -> espn::gpu
//
// Built with -DESPN_B200_WITH_REFERENCE_HEADERS so espn_b200.hpp reuses the
// reference's carrier types.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <cmath>
#include <cstring>
#include <fstream>
#include <mutex>
#include <numeric>
#include <queue>
#include <random>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "espn/error.hpp"
#include "espn/half.hpp"
#include "espn/ivf.hpp"
#include "espn/kmeans.hpp"
#include "espn/metrics.hpp"
#include "espn/pipeline.hpp"
#include "espn/scoring.hpp"
#include "espn/store.hpp"
#include "espn/types.hpp"
#include "espn_b200.hpp"
#include "espn_gpu.h"
#include "espn_store.h"

namespace espn {
int espn_ref_device();  // the CUDA runtime's current device (defined at the end)
namespace {

int current_device() { return espn_ref_device(); }

void throw_gpu(int st) {
  if (st != ESPN_OK) gpu::throw_status(st);
}

void throw_store(int st) {
  if (st != ESPN_OK) gpu::throw_status(st, espn_store_last_error());
}

bool all_finite(const std::vector<float>& v) {
  for (float x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

}  // namespace

// ============================================================ types.hpp:64-68
void validate_embedding(const EmbeddingMatrix& doc) {
  if (doc.rows < 1) throw InvalidInputError("document " + std::to_string(doc.doc_id) + " has t < 1");
  if (doc.cols < 1) throw InvalidInputError("document " + std::to_string(doc.doc_id) + " has d < 1");
  if (doc.values.size() != std::size_t(doc.rows) * doc.cols)
    throw InvalidInputError("document " + std::to_string(doc.doc_id) + ": values size != rows * cols");
  if (!all_finite(doc.values)) throw InvalidInputError("document " + std::to_string(doc.doc_id) + ": non-finite value");
}

void validate_cls(const ClsVector& cls) {
  if (cls.values.empty()) throw InvalidInputError("CLS vector of doc " + std::to_string(cls.doc_id) + " is empty");
  if (!all_finite(cls.values)) throw InvalidInputError("CLS vector of doc " + std::to_string(cls.doc_id) + ": non-finite value");
}

void validate_query(const QueryEmbedding& q) {
  if (q.rows < 1 || q.cols < 1) throw InvalidInputError("query " + std::to_string(q.query_id) + " has no tokens");
  if (q.tokens.size() != std::size_t(q.rows) * q.cols)
    throw InvalidInputError("query " + std::to_string(q.query_id) + ": tokens size != rows * cols");
  if (!all_finite(q.tokens) || !all_finite(q.cls))
    throw InvalidInputError("query " + std::to_string(q.query_id) + ": non-finite value");
}

// ============================================================ scoring.hpp:7-21
float maxsim_score(const QueryEmbedding& query, const EmbeddingMatrix& doc) {
  if (query.cols != doc.cols) throw InvalidInputError("maxsim_score: query dim != document dim");
  if (query.tokens.size() != std::size_t(query.rows) * query.cols || doc.values.size() != std::size_t(doc.rows) * doc.cols)
    throw InvalidInputError("maxsim_score: matrix sizes inconsistent with rows * cols");
  float out = 0.0f;
  throw_gpu(espn_gpu_maxsim_f32(query.tokens.data(), query.rows, doc.values.data(), doc.rows, doc.cols, &out,
                                current_device()));
  return out;
}

float aggregate_score(float cls_score, float bow_score, float alpha) {
  const float a = alpha * cls_score;  // no contraction in this TU (-ffp-contract=off): mul, then add
  return a + bow_score;
}

RankedList rank(std::vector<ScoredDoc> scored) {
  RankedList out;
  const std::size_t n = scored.size();
  if (!n) return out;
  std::vector<std::uint32_t> ids(n), oid(n);
  std::vector<float> sc(n), osc(n);
  for (std::size_t i = 0; i < n; ++i) {
    ids[i] = scored[i].doc_id;
    sc[i] = scored[i].score;
  }
  throw_gpu(espn_gpu_rank(ids.data(), sc.data(), n, oid.data(), osc.data(), current_device()));
  out.entries.resize(n);
  for (std::size_t i = 0; i < n; ++i) out.entries[i] = ScoredDoc{oid[i], osc[i]};
  return out;
}

float dot_f32(std::span<const float> a, std::span<const float> b) {
  if (a.size() != b.size()) throw InvalidInputError("dot_f32: length mismatch");
  if (a.empty()) return 0.0f;
  float out = 0.0f;
  throw_gpu(espn_gpu_maxsim_f32(a.data(), 1, b.data(), 1, static_cast<std::uint32_t>(a.size()), &out,
                                current_device()));
  return out;
}

// ============================================================ metrics.hpp:10-20
double mrr_at_k(const ResultsByQuery& results, const Qrels& qrels, int k) { return gpu::mrr_at_k(results, qrels, k); }
double recall_at_k(const ResultsByQuery& results, const Qrels& qrels, int k) {
  return gpu::recall_at_k(results, qrels, k);
}
Qrels load_qrels(const std::filesystem::path& path) { return gpu::load_qrels(path); }
Qrels load_qrels(std::istream& in) { return gpu::load_qrels(in); }

// ============================================================ store.hpp:37-112
StorePaths store_paths(const std::filesystem::path& base) {
  StorePaths p;
  p.data = base.string() + ".espn";
  p.manifest = base.string() + ".manifest";
  p.manifest_json = base.string() + ".manifest.json";
  return p;
}

namespace {
std::string base_of_manifest(const std::filesystem::path& manifest_path) {
  const std::string s = manifest_path.string();
  const std::string ext = ".manifest";
  if (s.size() > ext.size() && s.compare(s.size() - ext.size(), ext.size(), ext) == 0) return s.substr(0, s.size() - ext.size());
  throw InvalidInputError("manifest path must end in .manifest: " + s);
}

StoreManifest manifest_from(const espn_store_header& h, const std::vector<espn_manifest_record>& recs) {
  StoreManifest m;
  m.version = h.version;
  m.d = h.d;
  m.d_cls = h.d_cls;
  m.value_width = h.value_width;
  m.alignment = h.alignment;
  m.records.resize(recs.size());
  for (std::size_t i = 0; i < recs.size(); ++i)
    m.records[i] = ManifestRecord{recs[i].byte_offset, recs[i].byte_length, recs[i].token_count};
  return m;
}
}  // namespace

StoreManifest load_manifest(const std::filesystem::path& manifest_path) {
  const std::string base = base_of_manifest(manifest_path);
  espn_store_header h{};
  throw_store(espn_store_load_manifest(base.c_str(), &h, nullptr));
  std::vector<espn_manifest_record> recs(h.count);
  throw_store(espn_store_load_manifest(base.c_str(), &h, recs.data()));
  return manifest_from(h, recs);
}

void save_manifest(const StoreManifest& m, const StorePaths& paths) {
  const std::string base = base_of_manifest(paths.manifest);
  espn_store_header h{m.version, m.d, m.d_cls, m.value_width, m.alignment, m.count()};
  std::vector<espn_manifest_record> recs(m.records.size());
  for (std::size_t i = 0; i < recs.size(); ++i)
    recs[i] = espn_manifest_record{m.records[i].byte_offset, m.records[i].byte_length, m.records[i].token_count};
  throw_store(espn_store_save_manifest(base.c_str(), &h, recs.data()));
}

StoreManifest build_store(const std::vector<ClsVector>& cls, const std::vector<EmbeddingMatrix>& docs,
                          const std::filesystem::path& base, std::uint32_t alignment, std::uint32_t value_width) {
  const std::size_t n = docs.size();
  if (cls.size() != n) throw InvalidInputError("build_store: one CLS vector per document");
  if (alignment != 1 && alignment != 512 && alignment != 4096) throw InvalidInputError("alignment must be 1, 512 or 4096");
  if (value_width != 2 && value_width != 4) throw InvalidInputError("value_width must be 2 or 4");
  // dense ids [0, n) (store.hpp:20): place documents by id
  std::vector<const EmbeddingMatrix*> by_id(n, nullptr);
  std::vector<const ClsVector*> cls_by_id(n, nullptr);
  const std::uint32_t d = n ? docs[0].cols : 0;
  const std::uint32_t d_cls = n ? static_cast<std::uint32_t>(cls[0].values.size()) : 0;
  for (std::size_t i = 0; i < n; ++i) {
    validate_embedding(docs[i]);
    validate_cls(cls[i]);
    if (docs[i].doc_id >= n || by_id[docs[i].doc_id]) throw InvalidInputError("doc ids must be dense [0, n) and unique");
    if (cls[i].doc_id >= n || cls_by_id[cls[i].doc_id]) throw InvalidInputError("CLS doc ids must be dense [0, n)");
    if (docs[i].cols != d || cls[i].values.size() != d_cls) throw InvalidInputError("inconsistent dimensions");
    by_id[docs[i].doc_id] = &docs[i];
    cls_by_id[cls[i].doc_id] = &cls[i];
  }
  std::vector<std::uint64_t> rp(n + 1, 0);
  for (std::size_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + by_id[i]->rows;
  std::vector<float> rows(rp[n] * d), cv(n * std::size_t(d_cls));
  for (std::size_t i = 0; i < n; ++i) {
    std::copy(by_id[i]->values.begin(), by_id[i]->values.end(), rows.begin() + rp[i] * d);
    std::copy(cls_by_id[i]->values.begin(), cls_by_id[i]->values.end(), cv.begin() + i * d_cls);
  }
  throw_store(espn_store_build(base.c_str(), n, d, d_cls, value_width, alignment, rp.data(), rows.data(),
                               n ? cv.data() : nullptr));
  return load_manifest(store_paths(base).manifest);
}

// StoreHandle's private state is the reference's (manifest, options, fd,
// map, file size); the library's side -- the file reader and, for the
// pipeline, the HBM table -- is kept in a registry keyed by the handle's
// manifest address, re-keyed by the moves below.
namespace {
struct StoreState {
  std::string base;
  espn_store_reader* reader = nullptr;
  std::mutex mu;
  std::unique_ptr<gpu::Store> table;  // lazily opened by the pipeline
  ~StoreState() { espn_store_close(reader); }
  gpu::Store& gpu_table() {
    std::lock_guard<std::mutex> lk(mu);
    if (!table) table = std::make_unique<gpu::Store>(gpu::Store::open_store(base, gpu::Dtype::f16, current_device()));
    return *table;
  }
};
std::mutex g_reg_mu;
std::unordered_map<const StoreManifest*, std::shared_ptr<StoreState>> g_reg;

std::shared_ptr<StoreState> state_of(const StoreHandle& h) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto it = g_reg.find(&h.manifest());
  if (it == g_reg.end()) throw InvalidStateError("store handle is not open");
  return it->second;
}
int g_next_fd = 1;
}  // namespace

StoreHandle::~StoreHandle() {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_reg.erase(&manifest_);
}

StoreHandle::StoreHandle(StoreHandle&& o) noexcept
    : manifest_(std::move(o.manifest_)), options_(o.options_), fd_(o.fd_), map_(o.map_), file_size_(o.file_size_) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto it = g_reg.find(&o.manifest_);
  if (it != g_reg.end()) {
    g_reg[&manifest_] = std::move(it->second);
    g_reg.erase(it);
  }
  o.fd_ = -1;
  o.map_ = nullptr;
}

StoreHandle& StoreHandle::operator=(StoreHandle&& o) noexcept {
  if (this == &o) return *this;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_reg.erase(&manifest_);
  manifest_ = std::move(o.manifest_);
  options_ = o.options_;
  fd_ = o.fd_;
  map_ = o.map_;
  file_size_ = o.file_size_;
  auto it = g_reg.find(&o.manifest_);
  if (it != g_reg.end()) {
    g_reg[&manifest_] = std::move(it->second);
    g_reg.erase(it);
  }
  o.fd_ = -1;
  o.map_ = nullptr;
  return *this;
}

StoreHandle open_store(const std::filesystem::path& base, const StoreOptions& options) {
  auto st = std::make_shared<StoreState>();
  st->base = base.string();
  const std::uint32_t mode = options.mode == ReadMode::direct ? ESPN_READ_DIRECT
                             : options.mode == ReadMode::mmap ? ESPN_READ_MMAP
                                                              : ESPN_READ_BUFFERED;
  espn_store_header h{};
  throw_store(espn_store_open(st->base.c_str(), mode, static_cast<std::uint32_t>(options.queue_depth), &st->reader, &h));
  std::vector<espn_manifest_record> recs(h.count);
  throw_store(espn_store_records(st->reader, recs.data()));
  StoreHandle sh;
  sh.manifest_ = manifest_from(h, recs);
  sh.options_ = options;
  sh.fd_ = g_next_fd++;  // the reader owns the descriptor; this is the handle's identity
  sh.map_ = nullptr;
  sh.file_size_ = recs.empty() ? 0 : recs.back().byte_offset + recs.back().byte_length;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_reg[&sh.manifest_] = st;
  }
  return sh;
}

FetchResult StoreHandle::fetch_batch(std::span<const DocId> doc_ids) const {
  auto st = state_of(*this);
  FetchResult res;
  const std::uint64_t n = doc_ids.size();
  std::vector<std::uint64_t> off(n + 1, 0);
  std::uint64_t bytes = 0, blocks = 0;
  double wall = 0.0;
  throw_store(espn_store_fetch(st->reader, doc_ids.data(), n, nullptr, off.data(), 0, &bytes, &blocks, nullptr));
  std::vector<std::uint8_t> buf(std::max<std::uint64_t>(off[n], 1));
  throw_store(espn_store_fetch(st->reader, doc_ids.data(), n, buf.data(), off.data(), buf.size(), &bytes, &blocks, &wall));
  const StoreManifest& m = manifest_;
  res.docs.resize(n);
  auto value = [&](const std::uint8_t* p, std::size_t j) -> float {
    if (m.value_width == 2) {
      std::uint16_t c;
      std::memcpy(&c, p + 2 * j, 2);
      return half_to_float(c);  // the reference's own decoder (half.hpp:47-73)
    }
    float x;
    std::memcpy(&x, p + 4 * j, 4);
    return x;
  };
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::uint8_t* p = buf.data() + off[i];
    const ManifestRecord& r = m.records[doc_ids[i]];
    FetchedDoc& fd = res.docs[i];
    fd.cls.doc_id = doc_ids[i];
    fd.cls.values.resize(m.d_cls);
    for (std::uint32_t j = 0; j < m.d_cls; ++j) fd.cls.values[j] = value(p, j);
    fd.bow.doc_id = doc_ids[i];
    fd.bow.rows = r.token_count;
    fd.bow.cols = m.d;
    fd.bow.values.resize(std::size_t(r.token_count) * m.d);
    for (std::size_t j = 0; j < fd.bow.values.size(); ++j) fd.bow.values[j] = value(p, m.d_cls + j);
  }
  res.bytes_read = bytes;
  res.blocks_read = blocks;
  res.wall_time = wall;
  return res;
}

// ============================================================ kmeans.hpp
namespace {
float sq_l2(const float* a, const float* b, std::size_t d) {
  float s = 0.0f;
  for (std::size_t k = 0; k < d; ++k) {
    const float t = a[k] - b[k];
    s += t * t;
  }
  return s;
}
float ip(const float* a, const float* b, std::size_t d) {  // ascending-order fp32 inner product
  float s = 0.0f;
  for (std::size_t k = 0; k < d; ++k) s += a[k] * b[k];
  return s;
}
}  // namespace

std::uint32_t nearest_centroid(const float* vec, const float* centroids, std::size_t k, std::size_t dim) {
  std::uint32_t best = 0;
  float bd = INFINITY;
  for (std::size_t c = 0; c < k; ++c) {
    const float dd = sq_l2(vec, centroids + c * dim, dim);
    if (dd < bd) {  // ties resolve to the lowest index
      bd = dd;
      best = static_cast<std::uint32_t>(c);
    }
  }
  return best;
}

KMeansResult kmeans(const float* data, std::size_t n, std::size_t dim, std::size_t k, std::size_t max_iters,
                    std::uint64_t seed) {
  if (k < 1 || n < k) throw InvalidInputError("kmeans: need 1 <= k <= n");
  if (max_iters < 1) throw InvalidInputError("kmeans: max_iters must be >= 1");
  KMeansResult r;
  r.centroids.assign(k * dim, 0.0f);
  std::mt19937_64 rng(seed);
  // k-means++ seeding (squared-distance weighted)
  std::vector<float> dmin(n, INFINITY);
  std::size_t first = std::uniform_int_distribution<std::size_t>(0, n - 1)(rng);
  std::copy(data + first * dim, data + (first + 1) * dim, r.centroids.begin());
  for (std::size_t c = 1; c < k; ++c) {
    double tot = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
      dmin[i] = std::min(dmin[i], sq_l2(data + i * dim, r.centroids.data() + (c - 1) * dim, dim));
      tot += dmin[i];
    }
    std::size_t pick = 0;
    if (tot > 0.0) {
      const double u = std::uniform_real_distribution<double>(0.0, tot)(rng);
      double acc = 0.0;
      for (pick = 0; pick + 1 < n; ++pick) {
        acc += dmin[pick];
        if (acc > u) break;
      }
    } else {
      pick = std::uniform_int_distribution<std::size_t>(0, n - 1)(rng);
    }
    std::copy(data + pick * dim, data + (pick + 1) * dim, r.centroids.begin() + c * dim);
  }
  // Lloyd iterations; empty clusters repaired by splitting the largest one
  r.assignment.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i) r.assignment[i] = nearest_centroid(data + i * dim, r.centroids.data(), k, dim);
  for (r.iterations = 1; r.iterations <= max_iters; ++r.iterations) {
    std::vector<double> sums(k * dim, 0.0);
    std::vector<std::size_t> cnt(k, 0);
    for (std::size_t i = 0; i < n; ++i) {
      ++cnt[r.assignment[i]];
      for (std::size_t j = 0; j < dim; ++j) sums[r.assignment[i] * dim + j] += data[i * dim + j];
    }
    for (std::size_t c = 0; c < k; ++c) {
      if (cnt[c]) {
        for (std::size_t j = 0; j < dim; ++j) r.centroids[c * dim + j] = static_cast<float>(sums[c * dim + j] / cnt[c]);
      } else {
        const std::size_t big = static_cast<std::size_t>(std::max_element(cnt.begin(), cnt.end()) - cnt.begin());
        for (std::size_t j = 0; j < dim; ++j) r.centroids[c * dim + j] = r.centroids[big * dim + j] * (1.0f + 1e-3f);
      }
    }
    bool changed = false;
    for (std::size_t i = 0; i < n; ++i) {
      const std::uint32_t a = nearest_centroid(data + i * dim, r.centroids.data(), k, dim);
      changed |= a != r.assignment[i];
      r.assignment[i] = a;
    }
    if (!changed) {
      r.converged = true;
      break;
    }
  }
  r.iterations = std::min(r.iterations, max_iters);
  return r;
}

// ============================================================ ivf.hpp
std::size_t IvfIndex::size() const {
  std::size_t s = 0;
  for (const auto& l : lists) s += l.ids.size();
  return s;
}

IvfIndex train_ivf(const std::vector<ClsVector>& vectors, std::size_t nlist, std::size_t max_iters, std::uint64_t seed) {
  if (nlist < 1 || vectors.size() < nlist) throw InvalidInputError("train_ivf needs at least nlist vectors");
  const std::size_t d = vectors[0].values.size();
  std::vector<float> data(vectors.size() * d);
  for (std::size_t i = 0; i < vectors.size(); ++i) {
    validate_cls(vectors[i]);
    if (vectors[i].values.size() != d) throw InvalidInputError("train_ivf: inconsistent CLS dimensions");
    std::copy(vectors[i].values.begin(), vectors[i].values.end(), data.begin() + i * d);
  }
  KMeansResult km = kmeans(data.data(), vectors.size(), d, nlist, max_iters, seed);
  IvfIndex ix;
  ix.d_cls = static_cast<std::uint32_t>(d);
  ix.centroids = std::move(km.centroids);
  ix.lists.resize(nlist);
  for (std::size_t i = 0; i < vectors.size(); ++i) {
    auto& l = ix.lists[km.assignment[i]];
    l.ids.push_back(vectors[i].doc_id);
    l.vectors.insert(l.vectors.end(), vectors[i].values.begin(), vectors[i].values.end());
  }
  return ix;
}

void save_ivf(const IvfIndex& index, const std::filesystem::path& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot write " + path.string());
  const char magic[8] = {'E', 'S', 'P', 'N', 'I', 'V', 'F', '1'};
  const std::uint32_t ver = 1, dcls = index.d_cls;
  const std::uint64_t nlist = index.nlist();
  f.write(magic, 8);
  f.write(reinterpret_cast<const char*>(&ver), 4);
  f.write(reinterpret_cast<const char*>(&dcls), 4);
  f.write(reinterpret_cast<const char*>(&nlist), 8);
  f.write(reinterpret_cast<const char*>(index.centroids.data()), index.centroids.size() * 4);
  for (const auto& l : index.lists) {
    const std::uint64_t len = l.ids.size();
    f.write(reinterpret_cast<const char*>(&len), 8);
    f.write(reinterpret_cast<const char*>(l.ids.data()), len * 4);
    f.write(reinterpret_cast<const char*>(l.vectors.data()), l.vectors.size() * 4);
  }
  if (!f) throw IoError("write failed: " + path.string());
}

IvfIndex load_ivf(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot read " + path.string());
  char magic[8];
  std::uint32_t ver = 0, dcls = 0;
  std::uint64_t nlist = 0;
  f.read(magic, 8);
  f.read(reinterpret_cast<char*>(&ver), 4);
  f.read(reinterpret_cast<char*>(&dcls), 4);
  f.read(reinterpret_cast<char*>(&nlist), 8);
  if (!f || std::memcmp(magic, "ESPNIVF1", 8) != 0 || ver != 1 || dcls == 0 || nlist == 0)
    throw FormatError("not an ESPNIVF1 file: " + path.string());
  IvfIndex ix;
  ix.d_cls = dcls;
  ix.centroids.resize(nlist * dcls);
  f.read(reinterpret_cast<char*>(ix.centroids.data()), ix.centroids.size() * 4);
  ix.lists.resize(nlist);
  for (auto& l : ix.lists) {
    std::uint64_t len = 0;
    f.read(reinterpret_cast<char*>(&len), 8);
    if (!f || len > (1ull << 32)) throw FormatError("truncated IVF list header");
    l.ids.resize(len);
    l.vectors.resize(len * dcls);
    f.read(reinterpret_cast<char*>(l.ids.data()), len * 4);
    f.read(reinterpret_cast<char*>(l.vectors.data()), l.vectors.size() * 4);
    if (!f) throw FormatError("truncated IVF list block");
  }
  f.peek();
  if (!f.eof()) throw FormatError("trailing bytes after the last IVF list");
  return ix;
}

namespace {
bool cand_better(const Candidate& a, const Candidate& b) {  // (cls_score desc, doc_id asc)
  return a.cls_score != b.cls_score ? a.cls_score > b.cls_score : a.doc_id < b.doc_id;
}
}  // namespace

SearchCursor::SearchCursor(const IvfIndex& index, std::span<const float> query_cls, std::size_t nprobe, std::size_t k)
    : index_(&index), query_(query_cls.begin(), query_cls.end()), capacity_(k) {
  if (nprobe < 1 || nprobe > index.nlist()) throw InvalidInputError("nprobe outside [1, nlist]");
  if (k < 1) throw InvalidInputError("k must be >= 1");
  if (query_.size() != index.d_cls) throw InvalidInputError("query CLS dimension != index d_cls");
  std::vector<std::pair<float, std::uint32_t>> cs(index.nlist());
  for (std::size_t c = 0; c < index.nlist(); ++c)
    cs[c] = {ip(index.centroids.data() + c * index.d_cls, query_.data(), index.d_cls), static_cast<std::uint32_t>(c)};
  std::stable_sort(cs.begin(), cs.end(), [](auto& a, auto& b) { return a.first > b.first; });  // ties: centroid index
  plan_.resize(nprobe);
  for (std::size_t i = 0; i < nprobe; ++i) plan_[i] = cs[i].second;
}

void SearchCursor::advance(std::size_t n_clusters) {
  if (visited_ + n_clusters > plan_.size()) throw InvalidInputError("advance past nprobe");
  // heap_: min-heap on cand_better (the worst candidate on top), at most capacity_ entries
  auto worse = [](const Candidate& a, const Candidate& b) { return cand_better(a, b); };
  for (std::size_t s = 0; s < n_clusters; ++s) {
    const auto& l = index_->lists[plan_[visited_ + s]];
    for (std::size_t i = 0; i < l.ids.size(); ++i) {
      const Candidate c{l.ids[i], ip(l.vectors.data() + i * index_->d_cls, query_.data(), index_->d_cls)};
      if (heap_.size() < capacity_) {
        heap_.push_back(c);
        std::push_heap(heap_.begin(), heap_.end(), worse);
      } else if (cand_better(c, heap_.front())) {
        std::pop_heap(heap_.begin(), heap_.end(), worse);
        heap_.back() = c;
        std::push_heap(heap_.begin(), heap_.end(), worse);
      }
    }
  }
  visited_ += n_clusters;
}

CandidateList SearchCursor::snapshot(std::size_t top_k) const {
  if (top_k < 1) throw InvalidInputError("top_k must be >= 1");
  CandidateList out;
  out.entries = heap_;
  std::sort(out.entries.begin(), out.entries.end(), cand_better);
  if (out.entries.size() > top_k) out.entries.resize(top_k);
  out.clusters_visited = visited_;
  return out;
}

CandidateList SearchCursor::finish(std::size_t k) const {
  if (visited_ != plan_.size()) throw InvalidStateError("finish before the cursor is fully advanced");
  return snapshot(std::max<std::size_t>(k, 1));
}

SearchCursor begin_search(const IvfIndex& index, std::span<const float> query_cls, std::size_t nprobe, std::size_t k) {
  return SearchCursor(index, query_cls, nprobe, k);
}

// ============================================================ pipeline.hpp
std::uint32_t PipelineConfig::delta() const {
  const std::uint32_t d = static_cast<std::uint32_t>(std::floor(nprobe * prefetch_step_pct / 100.0 + 0.5));
  return std::max<std::uint32_t>(1, d);
}

void validate_config(const PipelineConfig& c, const IvfIndex& index) {
  if (!(c.prefetch_step_pct > 0.0 && c.prefetch_step_pct <= 100.0))
    throw InvalidInputError("prefetch_step_pct must be in (0, 100]");
  if (c.nprobe < 1 || c.nprobe > index.nlist()) throw InvalidInputError("nprobe outside [1, nlist]");
  if (c.delta() > c.nprobe) throw InvalidInputError("delta > nprobe");
  if (c.final_k < 1) throw InvalidInputError("final_k must be >= 1");
  if (c.rerank_count < c.final_k && !c.partial_rerank_enabled)
    throw InvalidInputError("rerank_count < final_k requires partial re-ranking");
}

namespace {
struct Staged {  // stages (1)-(3) of one query on the host
  CandidateList snapshot, finals;
  double ann_time = 0.0;
};

Staged ivf_stages(const QueryEmbedding& q, const IvfIndex& index, const PipelineConfig& c) {
  const auto t0 = std::chrono::steady_clock::now();
  Staged s;
  const std::size_t K = c.effective_candidate_k();
  SearchCursor cur = begin_search(index, q.cls, c.nprobe, std::max<std::size_t>(K, c.effective_prefetch_top_k()));
  cur.advance(c.delta());
  if (c.prefetch_enabled) s.snapshot = cur.snapshot(std::max<std::uint32_t>(c.effective_prefetch_top_k(), 1));
  cur.advance(c.nprobe - c.delta());
  s.finals = cur.finish(K);
  s.ann_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return s;
}
}  // namespace

BatchResult run_batch(std::span<const QueryEmbedding> queries, const IvfIndex& index, const StoreHandle& store,
                      const PipelineConfig& config, std::size_t concurrency) {
  if (concurrency < 1) throw InvalidInputError("concurrency must be >= 1");
  validate_config(config, index);
  const std::size_t B = queries.size();
  BatchResult res;
  if (B == 0) return res;
  for (const auto& q : queries) validate_query(q);
  const auto t0 = std::chrono::steady_clock::now();
  // stages (1)-(3) on host threads, at most `concurrency` queries in flight
  std::vector<Staged> st(B);
  {
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex em;
    auto worker = [&] {
      for (std::size_t i; (i = next.fetch_add(1)) < B;) {
        try {
          st[i] = ivf_stages(queries[i], index, config);
        } catch (...) {
          std::lock_guard<std::mutex> lk(em);
          if (!err) err = std::current_exception();
        }
      }
    };
    std::vector<std::thread> pool;
    const std::size_t nt = std::min(concurrency, B);
    for (std::size_t t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
  }
  // the snapshot hints and stages 3-6 of the whole batch on the GPU
  gpu::Store& table = state_of(store)->gpu_table();
  std::uint64_t c_total = 0;
  for (const auto& s : st) c_total += s.finals.entries.size();
  const std::uint32_t nq = queries[0].rows;
  gpu::Reranker& rr = table.thread_reranker(static_cast<std::uint32_t>(B),
                                            static_cast<std::uint32_t>(std::max<std::uint64_t>(c_total, 1)),
                                            std::min<std::uint32_t>(nq, 32));
  std::vector<CandidateList> finals(B), snaps(B);
  for (std::size_t i = 0; i < B; ++i) {
    finals[i] = std::move(st[i].finals);
    snaps[i] = std::move(st[i].snapshot);
  }
  if (config.prefetch_enabled) rr.prefetch_hints(snaps);
  BatchResult r = rr.rerank(queries, finals, config, gpu::Kernel::automatic, config.prefetch_enabled);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<double> lat(B);
  for (std::size_t i = 0; i < B; ++i) {
    r.stats[i].ann_time = st[i].ann_time;
    r.stats[i].total_time = st[i].ann_time + r.stats[i].rerank_time;
    lat[i] = r.stats[i].total_time;
  }
  std::sort(lat.begin(), lat.end());
  auto pct = [&](double p) {
    const double x = p / 100.0 * static_cast<double>(B - 1);
    const std::size_t lo = static_cast<std::size_t>(x), hi = std::min(lo + 1, B - 1);
    return lat[lo] + (lat[hi] - lat[lo]) * (x - static_cast<double>(lo));
  };
  r.batch.n_queries = B;
  r.batch.mean_latency = std::accumulate(lat.begin(), lat.end(), 0.0) / static_cast<double>(B);
  r.batch.p50_latency = pct(50);
  r.batch.p99_latency = pct(99);
  r.batch.wall_time = wall;
  r.batch.total_critical_fetch_bytes = 0;
  for (const auto& s : r.stats) r.batch.total_critical_fetch_bytes += s.critical_fetch_bytes;
  return r;
}

std::pair<RankedList, QueryStats> run_query(const QueryEmbedding& query, const IvfIndex& index,
                                            const StoreHandle& store, const PipelineConfig& config) {
  BatchResult r = run_batch(std::span<const QueryEmbedding>(&query, 1), index, store, config, 1);
  return {std::move(r.rankings[0]), r.stats[0]};
}

std::vector<HitRatePoint> measure_hit_rate(std::span<const QueryEmbedding> queries, const IvfIndex& index,
                                           const StoreHandle& store, const PipelineConfig& base,
                                           std::span<const double> steps) {
  if (steps.empty()) throw InvalidInputError("measure_hit_rate needs at least one step");
  std::vector<HitRatePoint> out;
  for (double s : steps) {
    if (!(s > 0.0 && s <= 100.0)) throw InvalidInputError("prefetch steps must be in (0, 100]");
    PipelineConfig c = base;
    c.prefetch_step_pct = s;
    c.prefetch_enabled = true;
    BatchResult r = run_batch(queries, index, store, c, std::max<std::size_t>(1, std::thread::hardware_concurrency()));
    double sum = 0.0;
    for (const auto& st : r.stats) sum += st.hit_rate;
    out.push_back(HitRatePoint{s, queries.empty() ? 0.0 : sum / static_cast<double>(queries.size())});
  }
  return out;
}

}  // namespace espn

// the device the reference API uses: the CUDA runtime's current device
#include <cuda_runtime_api.h>
int espn::espn_ref_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
