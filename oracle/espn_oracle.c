/*
 * espn_oracle.c -- CPU restatement of the ESPN re-ranking contract.
 * TEST INFRASTRUCTURE ONLY (see espn_oracle.h).  Built with -ffp-contract=off.
 *
 * Follows, function by function:
 *   codecs        proj/include/espn/half.hpp:11-76 (IEEE semantics; the reference's
 *                 subnormal defects are documented in SURVEY.md §8(a3) and pinned
 *                 by tests/test_oracle.py against tests/golden/half_ref_codec.npz)
 *   dot/maxsim    proj/include/espn/scoring.hpp:7-10, 20-21
 *   aggregate     scoring.hpp:12-14
 *   rank          scoring.hpp:16-18; types.hpp:51-55
 *   gather        store.hpp:56-94
 *   rerank        pipeline.hpp:34-64; SPEC.md:273-281, 301-311 (stages 3-6)
 *   batch         pipeline.hpp:81-85
 */
#include "espn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t f2u(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static inline float u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* IEEE binary32 -> binary16, round to nearest even (half.hpp:11-45 contract). */
uint16_t eo_float_to_half(float f) {
  const uint32_t x = f2u(f);
  const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  const uint32_t a = x & 0x7fffffffu;
  if (a > 0x7f800000u) return (uint16_t)(sign | 0x7e00u | ((a >> 13) & 0x03ffu)); /* NaN, quiet */
  if (a >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 rounds to inf */
  if (a >= 0x38800000u) {                                  /* normal half */
    uint32_t h = (((a >> 23) - 112u) << 10) | ((a >> 13) & 0x03ffu);
    const uint32_t rem = a & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
  }
  if (a <= 0x33000000u) return sign; /* |x| <= 2^-25 rounds to zero (tie -> even) */
  /* subnormal half: units of 2^-24 */
  const uint32_t e = a >> 23;                 /* biased, 102..112 */
  const uint32_t m = (a & 0x007fffffu) | 0x00800000u;
  const uint32_t shift = 126u - e;            /* 14..24 */
  uint32_t q = m >> shift;
  const uint32_t rem = m & ((1u << shift) - 1u);
  const uint32_t half = 1u << (shift - 1u);
  if (rem > half || (rem == half && (q & 1u))) ++q;
  return (uint16_t)(sign | q);
}

float eo_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu;
  const uint32_t m = h & 0x03ffu;
  if (e == 0) {
    const float v = (float)m * 5.9604644775390625e-8f; /* m * 2^-24, exact */
    return sign ? -v : v;
  }
  if (e == 31) return u2f(sign | 0x7f800000u | (m << 13));
  return u2f(sign | ((e + 112u) << 23) | (m << 13));
}

uint16_t eo_float_to_bf16(float f) {
  const uint32_t x = f2u(f);
  if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((x >> 16) | 0x0040u);
  return (uint16_t)((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
}

float eo_bf16_to_float(uint16_t h) { return u2f((uint32_t)h << 16); }

void eo_encode(const float* in, uint16_t* out, size_t n, int dtype) {
  for (size_t i = 0; i < n; ++i)
    out[i] = dtype == EO_DTYPE_BF16 ? eo_float_to_bf16(in[i]) : eo_float_to_half(in[i]);
}

void eo_decode(const uint16_t* in, float* out, size_t n, int dtype) {
  for (size_t i = 0; i < n; ++i)
    out[i] = dtype == EO_DTYPE_BF16 ? eo_bf16_to_float(in[i]) : eo_half_to_float(in[i]);
}

/* dot_f32 (scoring.hpp:20-21): fp32, ascending index order, no contraction. */
float eo_dot_f32(const float* a, const float* b, uint32_t d) {
  float acc = 0.0f;
  for (uint32_t k = 0; k < d; ++k) {
    const float p = a[k] * b[k];
    acc = acc + p;
  }
  return acc;
}

/* maxsim_score (scoring.hpp:7-10): sum over query tokens, in
 * ascending order, of the max dot product over doc tokens. */
float eo_maxsim_score(const float* q, uint32_t nq, const float* doc, uint32_t t,
                      uint32_t d) {
  float s = 0.0f;
  for (uint32_t i = 0; i < nq; ++i) {
    float m = -INFINITY;
    for (uint32_t j = 0; j < t; ++j) {
      const float v = eo_dot_f32(q + (size_t)i * d, doc + (size_t)j * d, d);
      if (v > m) m = v;
    }
    s = s + m;
  }
  return s;
}

/* aggregate_score (scoring.hpp:12-14): alpha*cls + bow. */
float eo_aggregate_score(float cls_score, float bow_score, float alpha) {
  const float p = alpha * cls_score;
  return p + bow_score;
}

typedef struct {
  uint32_t id;
  float score;
} scored_t;

static int cmp_rank(const void* pa, const void* pb) {
  const scored_t* a = (const scored_t*)pa;
  const scored_t* b = (const scored_t*)pb;
  if (a->score > b->score) return -1;
  if (a->score < b->score) return 1;
  return (a->id > b->id) - (a->id < b->id);
}

static int cmp_u32(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  return (a > b) - (a < b);
}

/* rank (scoring.hpp:16-18): (score desc, doc_id asc); duplicates and
 * non-finite scores rejected. */
int eo_rank(const uint32_t* ids, const float* scores, size_t n, uint32_t* out_ids,
            float* out_scores) {
  scored_t* v = (scored_t*)malloc((n ? n : 1) * sizeof(scored_t));
  uint32_t* sid = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  int st = EO_OK;
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(scores[i])) st = EO_INVALID_INPUT;
    v[i].id = ids[i];
    v[i].score = scores[i];
    sid[i] = ids[i];
  }
  if (st == EO_OK) {
    qsort(sid, n, sizeof(uint32_t), cmp_u32);
    for (size_t i = 1; i < n; ++i)
      if (sid[i] == sid[i - 1]) st = EO_INVALID_INPUT;
  }
  if (st == EO_OK) {
    qsort(v, n, sizeof(scored_t), cmp_rank);
    for (size_t i = 0; i < n; ++i) {
      out_ids[i] = v[i].id;
      out_scores[i] = v[i].score;
    }
  }
  free(v);
  free(sid);
  return st;
}

uint64_t eo_record_bytes(const eo_table* t, uint64_t doc) {
  const uint64_t tok = t->row_ptr[doc + 1] - t->row_ptr[doc];
  return ((uint64_t)t->d_cls + tok * t->d) * t->value_width;
}

/* Bytes a read of this record transfers and blocks it touches (store.hpp:61-65):
 * aligned-rounded in direct mode (block = alignment), payload otherwise (block =
 * 4096).  Records start on `alignment` boundaries (store.hpp:21-22), so with
 * alignment >= block the first block offset is 0. */
static void record_io(const eo_table* t, uint64_t doc, uint64_t* bytes, uint64_t* blocks) {
  const uint64_t len = eo_record_bytes(t, doc);
  const uint64_t align = t->alignment ? t->alignment : 1;
  const uint64_t block = t->direct_io ? align : 4096u;
  if (t->direct_io) {
    *bytes = (len + align - 1) / align * align;
  } else {
    *bytes = len;
  }
  *blocks = (len + block - 1) / block;
}

int eo_gather(const eo_table* t, const uint32_t* ids, size_t n, uint64_t* out_row_ptr,
              uint16_t* out_rows) {
  for (size_t i = 0; i < n; ++i)
    if (ids[i] >= t->n_docs) return EO_INVALID_INPUT;
  out_row_ptr[0] = 0;
  for (size_t i = 0; i < n; ++i)
    out_row_ptr[i + 1] = out_row_ptr[i] + (t->row_ptr[ids[i] + 1] - t->row_ptr[ids[i]]);
  if (out_rows) {
    for (size_t i = 0; i < n; ++i) {
      const uint64_t tok = out_row_ptr[i + 1] - out_row_ptr[i];
      memcpy(out_rows + out_row_ptr[i] * t->d, t->rows + t->row_ptr[ids[i]] * t->d,
             tok * t->d * sizeof(uint16_t));
    }
  }
  return EO_OK;
}

int eo_validate_config(const eo_config* cfg) {
  if (cfg->final_k < 1) return EO_INVALID_INPUT;
  if (!isfinite(cfg->alpha)) return EO_INVALID_INPUT;
  if (!cfg->partial_rerank_enabled && cfg->rerank_count < cfg->final_k) return EO_INVALID_INPUT;
  return EO_OK;
}

/* MaxSim of one query against one table doc (decodes the doc's rows). */
static float score_doc(const eo_table* t, const float* q, uint32_t nq, uint32_t id,
                       float* scratch) {
  const uint64_t r0 = t->row_ptr[id];
  const uint32_t tok = (uint32_t)(t->row_ptr[id + 1] - r0);
  eo_decode(t->rows + r0 * t->d, scratch, (size_t)tok * t->d, (int)t->dtype);
  return eo_maxsim_score(q, nq, scratch, tok, t->d);
}

static uint32_t max_tokens(const eo_table* t, const uint32_t* ids, uint32_t n) {
  uint32_t m = 1;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t tok = (uint32_t)(t->row_ptr[ids[i] + 1] - t->row_ptr[ids[i]]);
    if (tok > m) m = tok;
  }
  return m;
}

int eo_rerank_query(const eo_table* t, const float* q_tokens, uint32_t nq,
                    const uint32_t* cand_ids, const float* cand_cls, uint32_t n_cand,
                    const uint32_t* prefetched_ids, uint32_t n_prefetched,
                    const eo_config* cfg, uint32_t* out_ids, float* out_scores,
                    uint32_t* out_n, eo_stats* stats) {
  int st = eo_validate_config(cfg);
  if (st) return st;
  if (nq < 1) return EO_INVALID_INPUT;
  for (size_t i = 0; i < (size_t)nq * t->d; ++i)
    if (!isfinite(q_tokens[i])) return EO_INVALID_INPUT; /* validate_query */
  for (uint32_t i = 0; i < n_cand; ++i) {
    if (cand_ids[i] >= t->n_docs) return EO_DATA_INTEGRITY;
    if (!isfinite(cand_cls[i])) return EO_INVALID_INPUT;
  }
  /* (3) needed = top R of the final candidates; missed = needed \ prefetched. */
  const uint32_t n_needed = n_cand < cfg->rerank_count ? n_cand : cfg->rerank_count;
  const uint32_t n_pf = cfg->prefetch_enabled ? n_prefetched : 0;
  uint32_t* pf_sorted = (uint32_t*)malloc((n_pf ? n_pf : 1) * sizeof(uint32_t));
  if (n_pf) memcpy(pf_sorted, prefetched_ids, n_pf * sizeof(uint32_t));
  qsort(pf_sorted, n_pf, sizeof(uint32_t), cmp_u32);

  eo_stats s;
  memset(&s, 0, sizeof s);
  s.prefetched_count = n_pf;
  s.needed_count = n_needed;
  for (uint32_t i = 0; i < n_pf; ++i) {
    if (pf_sorted[i] >= t->n_docs) { free(pf_sorted); return EO_DATA_INTEGRITY; }
    uint64_t b, k;
    record_io(t, pf_sorted[i], &b, &k);
    s.prefetch_bytes += b;
  }
  uint32_t hits = 0;
  for (uint32_t i = 0; i < n_needed; ++i) {
    const uint32_t id = cand_ids[i];
    s.needed_payload_bytes += eo_record_bytes(t, id);
    if (n_pf && bsearch(&id, pf_sorted, n_pf, sizeof(uint32_t), cmp_u32)) {
      ++hits;
    } else {
      uint64_t b, k;
      record_io(t, id, &b, &k);
      s.critical_fetch_bytes += b;
      s.critical_blocks_read += k;
    }
  }
  s.missed_count = n_needed - hits;
  s.hit_rate = n_needed ? (double)hits / (double)n_needed : 0.0;
  free(pf_sorted);

  /* (4)+(5): MaxSim + aggregate for every needed doc (early or critical path:
   * the same arithmetic, so prefetch on/off is bit-identical);
   * tail beyond R gets alpha*cls under partial re-rank (SPEC.md:276 (5), 311). */
  const uint32_t n_scored = cfg->partial_rerank_enabled ? n_cand : n_needed;
  uint32_t* ids = (uint32_t*)malloc((n_scored ? n_scored : 1) * sizeof(uint32_t));
  float* sc = (float*)malloc((n_scored ? n_scored : 1) * sizeof(float));
  float* scratch = (float*)malloc((size_t)max_tokens(t, cand_ids, n_needed) * t->d * sizeof(float));
  for (uint32_t i = 0; i < n_needed; ++i) {
    ids[i] = cand_ids[i];
    sc[i] = eo_aggregate_score(cand_cls[i], score_doc(t, q_tokens, nq, cand_ids[i], scratch),
                               cfg->alpha);
  }
  for (uint32_t i = n_needed; i < n_scored; ++i) {
    ids[i] = cand_ids[i];
    sc[i] = eo_aggregate_score(cand_cls[i], 0.0f, cfg->alpha);
  }
  free(scratch);
  /* (6) rank + truncate to final_k. */
  uint32_t* rid = (uint32_t*)malloc((n_scored ? n_scored : 1) * sizeof(uint32_t));
  float* rsc = (float*)malloc((n_scored ? n_scored : 1) * sizeof(float));
  st = eo_rank(ids, sc, n_scored, rid, rsc);
  if (st == EO_OK) {
    const uint32_t k = n_scored < cfg->final_k ? n_scored : cfg->final_k;
    memcpy(out_ids, rid, k * sizeof(uint32_t));
    memcpy(out_scores, rsc, k * sizeof(float));
    *out_n = k;
    if (stats) *stats = s;
  }
  free(ids);
  free(sc);
  free(rid);
  free(rsc);
  return st;
}

/* ---- run_batch: queries in parallel, each result identical to serial ---- */
typedef struct {
  const eo_table* t;
  const float* q;
  uint32_t nb, nq;
  const uint32_t* ids;
  const float* cls;
  const uint64_t* off;
  const eo_config* cfg;
  uint32_t* out_ids;
  float* out_scores;
  uint32_t* out_n;
  float* out_bow; /* maxsim-only mode when non-NULL */
  volatile int next;
  volatile int status;
  pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int b = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (b >= (int)j->nb) break;
    const float* qb = j->q + (size_t)b * j->nq * j->t->d;
    const uint64_t o0 = j->off[b], o1 = j->off[b + 1];
    int st;
    if (j->out_bow) {
      st = EO_OK;
      float* scratch = (float*)malloc((size_t)max_tokens(j->t, j->ids + o0, (uint32_t)(o1 - o0)) *
                                      j->t->d * sizeof(float));
      for (uint64_t c = o0; c < o1; ++c) {
        if (j->ids[c] >= j->t->n_docs) { st = EO_DATA_INTEGRITY; break; }
        j->out_bow[c] = score_doc(j->t, qb, j->nq, j->ids[c], scratch);
      }
      free(scratch);
    } else {
      st = eo_rerank_query(j->t, qb, j->nq, j->ids + o0, j->cls + o0, (uint32_t)(o1 - o0), NULL, 0,
                           j->cfg, j->out_ids + (size_t)b * j->cfg->final_k,
                           j->out_scores + (size_t)b * j->cfg->final_k, j->out_n + b, NULL);
    }
    if (st) {
      pthread_mutex_lock(&j->mu);
      if (!j->status) j->status = st;
      pthread_mutex_unlock(&j->mu);
    }
  }
  return NULL;
}

static int run_jobs(batch_job* j, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_mutex_init(&j->mu, NULL);
  j->next = 0;
  j->status = EO_OK;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, batch_worker, j);
  batch_worker(j);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&j->mu);
  return j->status;
}

int eo_rerank_batch(const eo_table* t, const float* q_tokens, uint32_t n_queries,
                    uint32_t nq, const uint32_t* cand_ids, const float* cand_cls,
                    const uint64_t* cand_offsets, const eo_config* cfg, uint32_t* out_ids,
                    float* out_scores, uint32_t* out_n, int nthreads) {
  batch_job j;
  memset(&j, 0, sizeof j);
  j.t = t; j.q = q_tokens; j.nb = n_queries; j.nq = nq; j.ids = cand_ids; j.cls = cand_cls;
  j.off = cand_offsets; j.cfg = cfg; j.out_ids = out_ids; j.out_scores = out_scores;
  j.out_n = out_n;
  return run_jobs(&j, nthreads);
}

int eo_maxsim_batch(const eo_table* t, const float* q_tokens, uint32_t n_queries,
                    uint32_t nq, const uint32_t* cand_ids, const uint64_t* cand_offsets,
                    float* out_scores, int nthreads) {
  batch_job j;
  memset(&j, 0, sizeof j);
  j.t = t; j.q = q_tokens; j.nb = n_queries; j.nq = nq; j.ids = cand_ids;
  j.off = cand_offsets; j.out_bow = out_scores;
  return run_jobs(&j, nthreads);
}
