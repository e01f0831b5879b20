// host_api_test -- drives the C++ espn::gpu API (include/espn_b200.hpp) on the
// GPU and checks it against the CPU oracle (oracle/espn_oracle.h; test
// infrastructure).  Exit code 0 = all checks passed.  Run by
// tests/test_cpp_api.py under -m gpu.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "espn_b200.hpp"
#include "espn_oracle.h"

namespace {
int failures = 0;
#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                \
      std::printf("\n");                       \
      ++failures;                              \
    }                                          \
  } while (0)

float half_round(float x) { return eo_half_to_float(eo_float_to_half(x)); }

std::vector<float> unit_vector(std::mt19937_64& rng, std::uint32_t d) {
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> v(d);
  double s = 0;
  for (auto& x : v) { x = nd(rng); s += (double)x * x; }
  for (auto& x : v) x = half_round(x / (float)std::sqrt(s));
  for (auto& x : v)  // no fp16 subnormals in generated tables
    if (std::fabs(x) < 6.103515625e-05f) x = 0.f;
  return v;
}
}  // namespace

int main() {
  const std::uint32_t n_docs = 4000, d = 32, nq = 32, B = 6, K = 500;
  std::mt19937_64 rng(2024);
  // ---- corpus as reference EmbeddingMatrix docs ----
  std::vector<espn::EmbeddingMatrix> docs(n_docs);
  std::vector<std::uint64_t> rp(n_docs + 1, 0);
  for (std::uint32_t i = 0; i < n_docs; ++i) {
    const std::uint32_t t = 1 + rng() % 63;
    docs[i].doc_id = i;
    docs[i].rows = t;
    docs[i].cols = d;
    for (std::uint32_t j = 0; j < t; ++j) {
      auto v = unit_vector(rng, d);
      docs[i].values.insert(docs[i].values.end(), v.begin(), v.end());
    }
    rp[i + 1] = rp[i] + t;
  }
  espn::gpu::Store store = espn::gpu::Store::from_documents(docs);
  // ---- queries: perturbed rows of a source doc; candidates sorted (cls desc, id asc) ----
  std::vector<espn::QueryEmbedding> qs(B);
  std::vector<espn::CandidateList> cl(B);
  std::vector<std::uint32_t> src(B);
  for (std::uint32_t b = 0; b < B; ++b) {
    src[b] = rng() % n_docs;
    qs[b].query_id = 100 + b;
    qs[b].rows = nq;
    qs[b].cols = d;
    for (std::uint32_t i = 0; i < nq; ++i) {
      auto v = unit_vector(rng, d);
      const auto& sd = docs[src[b]];
      const std::uint32_t j = rng() % sd.rows;
      for (std::uint32_t k = 0; k < d; ++k) v[k] = half_round(sd.values[j * d + k] + 0.1f * v[k]);
      qs[b].tokens.insert(qs[b].tokens.end(), v.begin(), v.end());
    }
    std::vector<std::uint32_t> ids;
    std::vector<char> used(n_docs, 0);
    ids.push_back(src[b]);
    used[src[b]] = 1;
    while (ids.size() < K) {
      const std::uint32_t c = rng() % n_docs;
      if (!used[c]) { used[c] = 1; ids.push_back(c); }
    }
    std::uniform_real_distribution<float> u01(0.f, 1.f);
    for (std::uint32_t c : ids) cl[b].entries.push_back({c, c == src[b] ? 1.0f : u01(rng)});
    std::sort(cl[b].entries.begin(), cl[b].entries.end(), [](const espn::Candidate& x, const espn::Candidate& y) {
      return x.cls_score != y.cls_score ? x.cls_score > y.cls_score : x.doc_id < y.doc_id;
    });
  }
  // ---- oracle table (same fp16 codes) ----
  std::vector<std::uint16_t> codes(rp.back() * d);
  for (std::uint32_t i = 0; i < n_docs; ++i)
    for (std::size_t j = 0; j < docs[i].values.size(); ++j) codes[rp[i] * d + j] = eo_float_to_half(docs[i].values[j]);
  eo_table ot{};
  ot.n_docs = n_docs;
  ot.d = d;
  ot.dtype = EO_DTYPE_F16;
  ot.row_ptr = rp.data();
  ot.rows = codes.data();
  ot.d_cls = 128;
  ot.value_width = 2;
  ot.alignment = 4096;

  for (int partial = 0; partial < 2; ++partial) {
    espn::PipelineConfig cfg;
    cfg.rerank_count = partial ? 64 : K;
    cfg.final_k = 10;
    cfg.alpha = partial ? 0.5f : 1.0f;
    cfg.partial_rerank_enabled = partial != 0;
    espn::BatchResult r = espn::gpu::rerank_batch(qs, cl, store, cfg);
    CHECK(r.rankings.size() == B, "batch size");
    eo_config oc{cfg.rerank_count, cfg.final_k, cfg.alpha, 1, partial};
    for (std::uint32_t b = 0; b < B; ++b) {
      std::vector<std::uint32_t> ids;
      std::vector<float> cls;
      for (auto& c : cl[b].entries) { ids.push_back(c.doc_id); cls.push_back(c.cls_score); }
      std::uint32_t oid[10], on = 0;
      float osc[10];
      eo_stats ost{};
      const int st = eo_rerank_query(&ot, qs[b].tokens.data(), nq, ids.data(), cls.data(), (std::uint32_t)ids.size(),
                                     nullptr, 0, &oc, oid, osc, &on, &ost);
      CHECK(st == 0, "oracle status %d", st);
      const auto& got = r.rankings[b].entries;
      CHECK(got.size() == on, "query %u: count %zu vs %u", b, got.size(), on);
      for (std::uint32_t i = 0; i < on && i < got.size(); ++i) {
        CHECK(std::fabs(got[i].score - osc[i]) <= 1e-3f * std::max(1.0f, std::fabs(osc[i])),
              "query %u rank %u: score %g vs %g", b, i, got[i].score, osc[i]);
        if (got[i].doc_id != oid[i])  // allowed only at a stated tie
          CHECK(std::fabs(got[i].score - osc[i]) <= 1e-3f * std::max(1.0f, std::fabs(osc[i])), "order at %u", i);
      }
      if (!partial) CHECK(!got.empty() && got[0].doc_id == src[b], "query %u: source doc not first", b);
      // QueryStats field for field with the oracle (pipeline.hpp:45-53)
      const auto& qs_b = r.stats[b];
      CHECK(qs_b.query_id == qs[b].query_id, "query id");
      CHECK(qs_b.needed_count == ost.needed_count, "needed_count %llu vs %llu",
            (unsigned long long)qs_b.needed_count, (unsigned long long)ost.needed_count);
      CHECK(qs_b.prefetched_count == ost.prefetched_count && qs_b.missed_count == ost.missed_count &&
                qs_b.hit_rate == ost.hit_rate, "q%u counts / hit rate", b);
      CHECK(qs_b.prefetch_bytes == ost.prefetch_bytes && qs_b.critical_fetch_bytes == ost.critical_fetch_bytes &&
                qs_b.critical_blocks_read == ost.critical_blocks_read &&
                qs_b.needed_payload_bytes == ost.needed_payload_bytes,
            "q%u bytes %llu/%llu blocks %llu/%llu", b, (unsigned long long)qs_b.critical_fetch_bytes,
            (unsigned long long)ost.critical_fetch_bytes, (unsigned long long)qs_b.critical_blocks_read,
            (unsigned long long)ost.critical_blocks_read);
    }
  }
  // ---- the single-query seam ----
  {
    espn::PipelineConfig cfg;
    cfg.rerank_count = K;
    auto [rl, qst] = espn::gpu::rerank_candidates(qs[0], cl[0], store, cfg);
    CHECK(!rl.entries.empty() && rl.entries[0].doc_id == src[0], "rerank_candidates top-1");
    CHECK(qst.hit_rate == 0.0 && qst.missed_count == qst.needed_count, "no prefetch: every needed doc is fetched");
  }
  // ---- fetch_batch: request order, duplicates, decoded fp32 (store.hpp:91-94) ----
  {
    std::vector<espn::DocId> req = {5, 17, 5, 3999};
    espn::FetchResult fr = store.fetch_batch(req);
    CHECK(fr.docs.size() == req.size(), "fetch size");
    for (std::size_t i = 0; i < req.size(); ++i) {
      const auto& got = fr.docs[i].bow;
      CHECK(got.doc_id == req[i] && got.rows == docs[req[i]].rows, "fetch doc %zu", i);
      CHECK(got.values == docs[req[i]].values, "fetch values of doc %u", req[i]);
    }
  }
  // ---- build_store -> open_store: same rows, same rankings (store.hpp:48-54, 111-112) ----
  {
    std::vector<float> rows;
    for (const auto& m : docs) rows.insert(rows.end(), m.values.begin(), m.values.end());
    const std::string base = "/tmp/espn_host_api_test_store";
    espn::gpu::build_store(base, rp, rows, d);
    espn::gpu::Store disk = espn::gpu::Store::open_store(base);
    CHECK(disk.n_docs() == n_docs && disk.d() == d, "open_store dims");
    CHECK(disk.record_bytes(10) == (128 + 10 * d) * 2, "record layout from the manifest");
    std::vector<espn::DocId> req = {0, 77, 3999};
    espn::FetchResult fa = disk.fetch_batch(req), fb = store.fetch_batch(req);
    for (std::size_t i = 0; i < req.size(); ++i) CHECK(fa.docs[i].bow.values == fb.docs[i].bow.values, "store doc %u", req[i]);
    espn::PipelineConfig cfg;
    cfg.rerank_count = K;
    espn::BatchResult ra = espn::gpu::rerank_batch(qs, cl, disk, cfg), rb = espn::gpu::rerank_batch(qs, cl, store, cfg);
    for (std::uint32_t b = 0; b < B; ++b) {
      CHECK(ra.rankings[b].entries.size() == rb.rankings[b].entries.size(), "open_store ranking size");
      for (std::size_t j = 0; j < ra.rankings[b].entries.size() && j < rb.rankings[b].entries.size(); ++j)
        CHECK(ra.rankings[b].entries[j].doc_id == rb.rankings[b].entries[j].doc_id &&
                  ra.rankings[b].entries[j].score == rb.rankings[b].entries[j].score,
              "open_store ranking q%u pos %zu", b, j);
    }
    bool thrown = false;
    try { espn::gpu::Store::open_store("/tmp/espn_no_such_store"); } catch (const espn::Error&) { thrown = true; }
    CHECK(thrown, "open_store of a missing store must throw");
  }
  // ---- tiered store + prefetch hints (run_query stages 1-2): same rankings, exact accounting ----
  {
    std::vector<std::uint8_t> resident(n_docs);
    for (std::uint32_t i = 0; i < n_docs; ++i) resident[i] = (i * 2654435761u >> 7) % 3 == 0;  // ~1/3 in HBM
    espn::gpu::Store tiered(rp, codes, d, espn::gpu::Dtype::f16, {}, 0, resident);
    espn::gpu::Reranker rt(tiered, B, B * K, nq);
    espn::gpu::Reranker rh(store, B, B * K, nq);
    espn::PipelineConfig cfg;
    cfg.rerank_count = 200;
    cfg.partial_rerank_enabled = true;
    const std::uint32_t P = 120;  // snapshot: the first P entries of each final list
    rt.prefetch_hints(cl, P);
    espn::BatchResult on = rt.rerank(qs, cl, cfg, espn::gpu::Kernel::automatic, /*prefetched=*/true);
    const std::vector<espn_fetch_stats> on_fs = rt.last_fetch_stats();
    espn::BatchResult off = rt.rerank(qs, cl, cfg);
    const std::vector<espn_fetch_stats> off_fs = rt.last_fetch_stats();
    // the same arithmetic as the tiered calls (AUTO may pick the single-launch
    // CUDA-core kernel for a small HBM-resident batch; tiered batches run tcgen05)
    espn::BatchResult hbm = rh.rerank(qs, cl, cfg, espn::gpu::Kernel::tcgen05);
    std::vector<char> hinted(n_docs, 0);
    for (const auto& c : cl)
      for (std::uint32_t j = 0; j < P && j < c.entries.size(); ++j) hinted[c.entries[j].doc_id] = 1;
    for (std::uint32_t b = 0; b < B; ++b) {
      const auto &x = on.rankings[b].entries, &y = off.rankings[b].entries, &z = hbm.rankings[b].entries;
      CHECK(x.size() == z.size() && y.size() == z.size(), "tiered ranking size q%u", b);
      for (std::size_t j = 0; j < x.size() && j < z.size() && j < y.size(); ++j)
        CHECK(x[j].doc_id == z[j].doc_id && x[j].score == z[j].score && y[j].doc_id == z[j].doc_id &&
                  y[j].score == z[j].score, "tiered ranking q%u pos %zu", b, j);
      // device tier view: host-tier needed rows not hinted are staged on the critical path
      std::uint64_t miss = 0, miss_off = 0, hint_miss = 0;
      for (std::uint32_t j = 0; j < cfg.rerank_count; ++j) {
        const std::uint32_t id = cl[b].entries[j].doc_id;
        if (!resident[id]) { ++miss_off; if (!hinted[id]) ++miss; }
        if (j >= P) ++hint_miss;
      }
      CHECK(on_fs[b].missed == miss, "q%u tier missed %llu vs %llu", b, (unsigned long long)on_fs[b].missed,
            (unsigned long long)miss);
      CHECK(off_fs[b].missed == miss_off, "q%u unprefetched tier missed", b);
      // QueryStats (reference semantics): prefetched = the P snapshot ids, missed = needed minus snapshot
      CHECK(on.stats[b].prefetched_count == P && on.stats[b].missed_count == hint_miss, "q%u reference counts", b);
      CHECK(off.stats[b].prefetched_count == 0 && off.stats[b].missed_count == cfg.rerank_count, "q%u no prefetch", b);
      CHECK(hbm.stats[b].hit_rate == 0.0, "no prefetch, hit rate 0");
    }
  }
  // ---- the disk tier: only ~1/3 of the docs in HBM, the rest read from the file per batch ----
  {
    std::vector<float> rows;
    for (const auto& m : docs) rows.insert(rows.end(), m.values.begin(), m.values.end());
    const std::string base = "/tmp/espn_host_api_test_disk";
    espn::gpu::build_store(base, rp, rows, d, {}, espn::gpu::RecordLayout{16, 2, 512});
    std::vector<std::uint8_t> resident(n_docs);
    for (std::uint32_t i = 0; i < n_docs; ++i) resident[i] = (i * 2654435761u >> 9) % 3 == 0;
    espn::gpu::Store disk = espn::gpu::Store::open_store(base, espn::gpu::Dtype::f16, 0, resident, 64ull << 20,
                                                         /*disk_tier=*/true);
    espn_store_reader* rd = nullptr;
    espn_store_header hh{};
    CHECK(espn_store_open(base.c_str(), ESPN_READ_DIRECT, 16, &rd, &hh) == ESPN_OK, "store open (direct)");
    espn::gpu::Reranker rd_r(disk, B, B * K, nq);
    espn::gpu::Reranker rh(store, B, B * K, nq);
    espn::PipelineConfig cfg;
    cfg.rerank_count = K;
    bool thrown = false;  // not prefetched: the rows exist only in the file
    try { rd_r.rerank(qs, cl, cfg, espn::gpu::Kernel::tcgen05); } catch (const espn::InvalidStateError&) { thrown = true; }
    CHECK(thrown, "disk tier without prefetch must throw InvalidStateError");
    const std::uint64_t got_bytes = rd_r.prefetch_from_file(cl, cfg.rerank_count, rd);
    CHECK(got_bytes > 0, "prefetch_from_file read the misses");
    espn::BatchResult a = rd_r.rerank(qs, cl, cfg, espn::gpu::Kernel::tcgen05, /*prefetched=*/true);
    espn::BatchResult h = rh.rerank(qs, cl, cfg, espn::gpu::Kernel::tcgen05);
    for (std::uint32_t b = 0; b < B; ++b) {
      CHECK(a.rankings[b].entries.size() == h.rankings[b].entries.size(), "disk ranking size q%u", b);
      for (std::size_t j = 0; j < a.rankings[b].entries.size() && j < h.rankings[b].entries.size(); ++j)
        CHECK(a.rankings[b].entries[j].doc_id == h.rankings[b].entries[j].doc_id &&
                  a.rankings[b].entries[j].score == h.rankings[b].entries[j].score,
              "disk ranking q%u pos %zu", b, j);
      std::uint64_t miss = 0;
      for (std::uint32_t j = 0; j < cfg.rerank_count && j < cl[b].entries.size(); ++j) miss += !resident[cl[b].entries[j].doc_id];
      CHECK(rd_r.last_fetch_stats()[b].prefetched == miss && rd_r.last_fetch_stats()[b].missed == 0,
            "q%u disk-tier hits %llu vs %llu", b, (unsigned long long)rd_r.last_fetch_stats()[b].prefetched,
            (unsigned long long)miss);
    }
    espn_store_close(rd);
  }
  // ---- error mapping (error.hpp:8-42) ----
  {
    espn::PipelineConfig cfg;
    cfg.rerank_count = K;
    auto bad = cl[0];
    bad.entries[3].doc_id = bad.entries[7].doc_id;  // duplicate -> InvalidInputError (scoring.hpp:16-18)
    bool thrown = false;
    try { espn::gpu::rerank_candidates(qs[0], bad, store, cfg); } catch (const espn::InvalidInputError&) { thrown = true; }
    CHECK(thrown, "duplicate id must throw InvalidInputError");
    auto unk = cl[0];
    unk.entries[2].doc_id = n_docs + 5;  // store lacks a candidate -> DataIntegrityError
    thrown = false;
    try { espn::gpu::rerank_candidates(qs[0], unk, store, cfg); } catch (const espn::DataIntegrityError&) { thrown = true; }
    CHECK(thrown, "unknown id must throw DataIntegrityError");
    thrown = false;
    std::vector<espn::DocId> req = {n_docs};
    try { store.fetch_batch(req); } catch (const espn::InvalidInputError&) { thrown = true; }
    CHECK(thrown, "fetch of an unknown id must throw InvalidInputError");
    espn::PipelineConfig c2;
    c2.rerank_count = 5;  // R < final_k without partial
    thrown = false;
    try { espn::gpu::rerank_candidates(qs[0], cl[0], store, c2); } catch (const espn::InvalidInputError&) { thrown = true; }
    CHECK(thrown, "R < final_k must throw InvalidInputError");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
