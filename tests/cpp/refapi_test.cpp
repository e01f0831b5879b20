// refapi_test.cpp -- a program written against the reference's OWN headers
// (/root/reference/proj/include/espn/*.hpp, unmodified), linked with
// lib/libespn_refapi.so (the B200 definitions) and checked against the CPU
// oracle (test infrastructure: oracle/_build/libespn_oracle.so).
//
// Covers the declarations the reference never defined: types.hpp:64-68,
// scoring.hpp:7-21, store.hpp:37-112 (build / manifests / open_store in the
// three read modes / fetch_batch with its counters), kmeans.hpp, ivf.hpp,
// pipeline.hpp (run_query / run_batch / measure_hit_rate, QueryStats field
// for field), metrics.hpp.  Built here (the reference tree exists only in
// the build container), run on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <set>
#include <vector>

#include "espn/error.hpp"
#include "espn/half.hpp"
#include "espn/ivf.hpp"
#include "espn/kmeans.hpp"
#include "espn/metrics.hpp"
#include "espn/pipeline.hpp"
#include "espn/scoring.hpp"
#include "espn/store.hpp"
#include "espn/types.hpp"

extern "C" {
#include "espn_oracle.h"
}

static int failures = 0;
#define CHECK(cond, ...)                                \
  do {                                                  \
    if (!(cond)) {                                      \
      ++failures;                                       \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__);  \
      std::printf(__VA_ARGS__);                         \
      std::printf("\n");                                \
    }                                                   \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  const std::uint32_t n_docs = 3000, d = 32, d_cls = 64, nq = 32;
  std::mt19937_64 rng(42);
  std::normal_distribution<float> nd(0.0f, 1.0f);
  std::uniform_int_distribution<std::uint32_t> tlen(1, 63);
  // ---- corpus: unit rows, fp16-representable (so the store round-trips exactly) ----
  std::vector<espn::EmbeddingMatrix> docs(n_docs);
  std::vector<espn::ClsVector> cls(n_docs);
  std::vector<std::vector<float>> centers(16, std::vector<float>(d_cls));
  for (auto& c : centers)
    for (auto& x : c) x = nd(rng);
  for (std::uint32_t i = 0; i < n_docs; ++i) {
    auto& m = docs[i];
    m.doc_id = i;
    m.rows = tlen(rng);
    m.cols = d;
    m.values.resize(std::size_t(m.rows) * d);
    for (std::uint32_t j = 0; j < m.rows; ++j) {
      float s = 0;
      for (std::uint32_t k = 0; k < d; ++k) s += (m.values[j * d + k] = nd(rng)) * m.values[j * d + k];
      for (std::uint32_t k = 0; k < d; ++k) {
        float v = espn::half_round_trip(m.values[j * d + k] / std::sqrt(s));
        if (std::fabs(v) < 6.2e-5f) v = 0.0f;  // no fp16 subnormals
        m.values[j * d + k] = v;
      }
    }
    cls[i].doc_id = i;
    cls[i].values.resize(d_cls);
    const auto& c = centers[i % 16];
    for (std::uint32_t k = 0; k < d_cls; ++k) cls[i].values[k] = espn::half_round_trip(c[k] + 0.3f * nd(rng));
  }
  // ---- types.hpp:64-68 ----
  {
    espn::EmbeddingMatrix bad = docs[0];
    bad.values[0] = NAN;
    CHECK(throws<espn::InvalidInputError>([&] { espn::validate_embedding(bad); }), "validate_embedding NaN");
    bad = docs[0];
    bad.rows = 0;
    bad.values.clear();
    CHECK(throws<espn::InvalidInputError>([&] { espn::validate_embedding(bad); }), "validate_embedding t=0");
    espn::validate_embedding(docs[1]);
    espn::validate_cls(cls[1]);
  }
  // ---- scoring.hpp on the device: bit-exact with the reference order ----
  espn::QueryEmbedding q0;
  q0.query_id = 7;
  q0.rows = nq;
  q0.cols = d;
  q0.cls = cls[5].values;
  q0.tokens.resize(nq * d);
  for (std::uint32_t i = 0; i < nq; ++i)
    for (std::uint32_t k = 0; k < d; ++k) q0.tokens[i * d + k] = docs[5].values[(i % docs[5].rows) * d + k] + 0.05f * nd(rng);
  for (std::uint32_t j : {0u, 5u, 77u, 2999u}) {
    const float g = espn::maxsim_score(q0, docs[j]);
    const float o = eo_maxsim_score(q0.tokens.data(), nq, docs[j].values.data(), docs[j].rows, d);
    CHECK(std::memcmp(&g, &o, 4) == 0, "maxsim_score doc %u: %.9g vs %.9g", j, g, o);
  }
  {
    const float g = espn::dot_f32(docs[9].values, docs[9].values);
    const float o = eo_dot_f32(docs[9].values.data(), docs[9].values.data(), (std::uint32_t)docs[9].values.size());
    CHECK(std::memcmp(&g, &o, 4) == 0, "dot_f32 %.9g vs %.9g", g, o);
    CHECK(espn::aggregate_score(2.0f, 1.0f, 0.5f) == eo_aggregate_score(2.0f, 1.0f, 0.5f), "aggregate_score");
    std::vector<espn::ScoredDoc> sd = {{5, 1.0f}, {3, 2.0f}, {9, 1.0f}, {1, -4.0f}};
    espn::RankedList rl = espn::rank(sd);
    const std::uint32_t want[4] = {3, 5, 9, 1};
    for (int i = 0; i < 4; ++i) CHECK(rl.entries[i].doc_id == want[i], "rank order %d", i);
    sd.push_back({3, 0.5f});
    CHECK(throws<espn::InvalidInputError>([&] { espn::rank(sd); }), "rank duplicate");
    sd.pop_back();
    sd.push_back({11, INFINITY});
    CHECK(throws<espn::InvalidInputError>([&] { espn::rank(sd); }), "rank non-finite");
    espn::QueryEmbedding q1 = q0;
    q1.cols = 16;
    CHECK(throws<espn::InvalidInputError>([&] { espn::maxsim_score(q1, docs[0]); }), "maxsim dim mismatch");
  }
  // ---- store.hpp: build, manifests, three read modes, fetch_batch + counters ----
  const std::string base = "/tmp/espn_refapi_store";
  espn::StoreManifest m = espn::build_store(cls, docs, base, 4096, 2);
  CHECK(m.count() == n_docs && m.d == d && m.d_cls == d_cls && m.value_width == 2 && m.alignment == 4096, "manifest");
  espn::StorePaths paths = espn::store_paths(base);
  espn::StoreManifest m2 = espn::load_manifest(paths.manifest);
  CHECK(m2.records.size() == n_docs && m2.records[17].byte_length == m.record_bytes(docs[17].rows), "load_manifest");
  espn::save_manifest(m2, paths);
  CHECK(espn::load_manifest(paths.manifest).records[2999].byte_offset == m.records[2999].byte_offset, "save_manifest");
  std::vector<espn::DocId> req = {17, 0, 17, 2999, 1234};
  std::uint64_t want_blocks = 0, want_bytes = 0;
  for (auto id : req) {
    want_bytes += m.records[id].byte_length;
    want_blocks += (m.records[id].byte_length + 4095) / 4096;
  }
  int modes_run = 0;
  for (auto mode : {espn::ReadMode::buffered, espn::ReadMode::mmap, espn::ReadMode::direct}) {
    espn::StoreOptions opt;
    opt.mode = mode;
    opt.queue_depth = 8;
    bool opened = true;
    espn::FetchResult fr;
    try {
      espn::StoreHandle h = espn::open_store(base, opt);
      fr = h.fetch_batch(req);
      CHECK(throws<espn::InvalidInputError>([&] { std::vector<espn::DocId> bad = {5, n_docs}; h.fetch_batch(bad); }),
            "unknown id");
      CHECK(h.fetch_batch(std::vector<espn::DocId>{}).docs.empty(), "empty request");
    } catch (const espn::IoError& e) {  // a filesystem without O_DIRECT (tmpfs / overlay)
      opened = mode != espn::ReadMode::direct;
      std::printf("note: direct mode unavailable here: %s\n", e.what());
    }
    if (!opened || fr.docs.empty()) continue;
    ++modes_run;
    CHECK(fr.docs.size() == req.size(), "fetch size");
    for (std::size_t i = 0; i < req.size(); ++i) {
      CHECK(fr.docs[i].bow.doc_id == req[i] && fr.docs[i].bow.values == docs[req[i]].values, "fetch bow %zu", i);
      CHECK(fr.docs[i].cls.values == cls[req[i]].values, "fetch cls %zu", i);
    }
    // store.hpp:61-65 / SPEC "Block accounting": per record; aligned-rounded bytes in direct mode
    CHECK(fr.blocks_read == want_blocks, "blocks_read %llu vs %llu", (unsigned long long)fr.blocks_read,
          (unsigned long long)want_blocks);
    const std::uint64_t wb = mode == espn::ReadMode::direct ? want_blocks * 4096 : want_bytes;
    CHECK(fr.bytes_read == wb, "bytes_read %llu vs %llu", (unsigned long long)fr.bytes_read, (unsigned long long)wb);
  }
  CHECK(modes_run >= 2, "read modes run: %d", modes_run);
  {
    const std::string b1 = "/tmp/espn_refapi_store_a1";
    espn::build_store(cls, docs, b1, 1, 2);
    espn::StoreOptions opt;
    opt.mode = espn::ReadMode::direct;
    CHECK(throws<espn::InvalidConfigError>([&] { espn::open_store(b1, opt); }), "direct on alignment 1");
  }
  // ---- kmeans / ivf ----
  std::vector<float> cdata(std::size_t(n_docs) * d_cls);
  for (std::uint32_t i = 0; i < n_docs; ++i) std::copy(cls[i].values.begin(), cls[i].values.end(), cdata.begin() + i * d_cls);
  espn::KMeansResult km = espn::kmeans(cdata.data(), n_docs, d_cls, 16, 20, 3);
  CHECK(km.centroids.size() == 16 * d_cls && km.assignment.size() == n_docs, "kmeans sizes");
  for (std::uint32_t i = 0; i < n_docs; i += 97)
    CHECK(km.assignment[i] == espn::nearest_centroid(cdata.data() + i * d_cls, km.centroids.data(), 16, d_cls),
          "kmeans assignment %u", i);
  espn::IvfIndex ix = espn::train_ivf(cls, 32, 15, 5);
  CHECK(ix.nlist() == 32 && ix.size() == n_docs, "train_ivf");
  espn::save_ivf(ix, "/tmp/espn_refapi.ivf");
  espn::IvfIndex ix2 = espn::load_ivf("/tmp/espn_refapi.ivf");
  CHECK(ix2.size() == ix.size() && ix2.centroids == ix.centroids, "ivf round trip");
  {  // exhaustive search == brute-force top-k by inner product (ties by id)
    espn::SearchCursor c = espn::begin_search(ix, q0.cls, 32, 50);
    c.advance(10);
    c.advance(22);
    espn::CandidateList f = c.finish(50);
    std::vector<std::pair<float, std::uint32_t>> all;
    for (std::uint32_t i = 0; i < n_docs; ++i) {
      float s = 0;
      for (std::uint32_t k = 0; k < d_cls; ++k) s += cls[i].values[k] * q0.cls[k];
      all.push_back({-s, i});
    }
    std::sort(all.begin(), all.end());
    CHECK(f.entries.size() == 50, "finish size");
    for (int i = 0; i < 50; ++i) CHECK(f.entries[i].doc_id == all[i].second, "exhaustive top-k %d", i);
    espn::SearchCursor c2 = espn::begin_search(ix, q0.cls, 4, 50);
    CHECK(throws<espn::InvalidStateError>([&] { c2.finish(10); }), "finish before advance");
  }
  // ---- pipeline.hpp: run_batch / run_query vs the oracle, QueryStats field for field ----
  espn::StoreHandle store = espn::open_store(base);
  std::vector<espn::QueryEmbedding> qs(6);
  for (std::uint32_t b = 0; b < 6; ++b) {
    const std::uint32_t src = 100 + 377 * b;
    qs[b].query_id = 1000 + b;
    qs[b].rows = nq;
    qs[b].cols = d;
    qs[b].cls = cls[src].values;
    qs[b].tokens.resize(nq * d);
    for (std::uint32_t i = 0; i < nq; ++i)
      for (std::uint32_t k = 0; k < d; ++k)
        qs[b].tokens[i * d + k] = docs[src].values[(i % docs[src].rows) * d + k] + 0.1f * nd(rng);
  }
  espn::PipelineConfig cfg;
  cfg.nprobe = 16;
  cfg.prefetch_step_pct = 25.0;
  cfg.rerank_count = 200;
  cfg.final_k = 10;
  cfg.candidate_k = 400;
  cfg.partial_rerank_enabled = true;
  cfg.alpha = 0.5f;
  espn::BatchResult on = espn::run_batch(qs, ix, store, cfg, 4);
  espn::PipelineConfig cfg_off = cfg;
  cfg_off.prefetch_enabled = false;
  espn::BatchResult off = espn::run_batch(qs, ix, store, cfg_off, 1);
  // the oracle table: the store's fp16 codes
  std::vector<std::uint64_t> rp(n_docs + 1, 0);
  for (std::uint32_t i = 0; i < n_docs; ++i) rp[i + 1] = rp[i] + docs[i].rows;
  std::vector<std::uint16_t> codes(rp[n_docs] * d);
  for (std::uint32_t i = 0; i < n_docs; ++i)
    for (std::size_t j = 0; j < docs[i].values.size(); ++j) codes[rp[i] * d + j] = espn::float_to_half(docs[i].values[j]);
  eo_table ot{};
  ot.n_docs = n_docs;
  ot.d = d;
  ot.dtype = EO_DTYPE_F16;
  ot.row_ptr = rp.data();
  ot.rows = codes.data();
  ot.d_cls = d_cls;
  ot.value_width = 2;
  ot.alignment = 4096;
  for (std::uint32_t b = 0; b < 6; ++b) {
    // stages (1)-(3) again (deterministic cursor): snapshot and final candidates
    espn::SearchCursor c = espn::begin_search(ix, qs[b].cls, cfg.nprobe, 400);
    c.advance(cfg.delta());
    espn::CandidateList snap = c.snapshot(cfg.effective_prefetch_top_k());
    c.advance(cfg.nprobe - cfg.delta());
    espn::CandidateList fin = c.finish(400);
    std::vector<std::uint32_t> ids, pf;
    std::vector<float> cs;
    for (auto& e : fin.entries) { ids.push_back(e.doc_id); cs.push_back(e.cls_score); }
    for (auto& e : snap.entries) pf.push_back(e.doc_id);
    eo_config oc{cfg.rerank_count, cfg.final_k, cfg.alpha, 1, 1};
    std::uint32_t oid[10], on_n = 0;
    float osc[10];
    eo_stats ost{};
    const int st = eo_rerank_query(&ot, qs[b].tokens.data(), nq, ids.data(), cs.data(), (std::uint32_t)ids.size(),
                                   pf.data(), (std::uint32_t)pf.size(), &oc, oid, osc, &on_n, &ost);
    CHECK(st == 0, "oracle status %d", st);
    const auto& got = on.rankings[b].entries;
    CHECK(got.size() == on_n, "q%u count", b);
    for (std::uint32_t i = 0; i < on_n && i < got.size(); ++i)
      CHECK(std::fabs(got[i].score - osc[i]) <= 1e-3f * std::max(1.0f, std::fabs(osc[i])), "q%u rank %u score", b, i);
    CHECK(off.rankings[b].entries.size() == got.size(), "prefetch on/off count q%u", b);
    for (std::size_t i = 0; i < got.size() && i < off.rankings[b].entries.size(); ++i)
      CHECK(off.rankings[b].entries[i].doc_id == got[i].doc_id && off.rankings[b].entries[i].score == got[i].score,
            "prefetch on/off identical q%u pos %zu", b, i);
    const espn::QueryStats& s = on.stats[b];
    CHECK(s.query_id == qs[b].query_id && s.needed_count == ost.needed_count && s.prefetched_count == ost.prefetched_count &&
              s.missed_count == ost.missed_count && s.hit_rate == ost.hit_rate && s.prefetch_bytes == ost.prefetch_bytes &&
              s.critical_fetch_bytes == ost.critical_fetch_bytes && s.critical_blocks_read == ost.critical_blocks_read &&
              s.needed_payload_bytes == ost.needed_payload_bytes,
          "q%u QueryStats: pf %llu/%llu miss %llu/%llu crit %llu/%llu", b, (unsigned long long)s.prefetched_count,
          (unsigned long long)ost.prefetched_count, (unsigned long long)s.missed_count,
          (unsigned long long)ost.missed_count, (unsigned long long)s.critical_fetch_bytes,
          (unsigned long long)ost.critical_fetch_bytes);
  }
  {
    auto [rl, st1] = espn::run_query(qs[2], ix, store, cfg);
    CHECK(rl.entries.size() == on.rankings[2].entries.size() && rl.entries[0].doc_id == on.rankings[2].entries[0].doc_id,
          "run_query == run_batch");
    std::vector<double> steps = {10.0, 100.0};
    auto pts = espn::measure_hit_rate(qs, ix, store, cfg, steps);
    CHECK(pts.size() == 2 && pts[1].mean_hit_rate == 1.0 && pts[0].mean_hit_rate <= 1.0, "hit rate endpoint");
    espn::PipelineConfig badc = cfg;
    badc.prefetch_step_pct = 0.0;
    CHECK(throws<espn::InvalidInputError>([&] { espn::validate_config(badc, ix); }), "validate_config step");
  }
  {  // metrics.hpp
    espn::Qrels qr = {{1000, {100}}, {1001, {477}}};
    espn::ResultsByQuery res;
    res[1000] = on.rankings[0];
    res[1001] = on.rankings[1];
    const double mrr = espn::mrr_at_k(res, qr, 10);
    CHECK(mrr >= 0.0 && mrr <= 1.0, "mrr range");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
