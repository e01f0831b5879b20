/*
 * espn_oracle.h -- CPU restatement of the ESPN re-ranking contract.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2312_05417_b200/,
 * include/, libespn_gpu.so) links, loads or calls this code.  It is used by
 * tests/ as the parity checker, by __graft_entry__.smoke() as the checker, and by
 * bench.py's cpu_baseline / --impl reference legs as "the reference's CPU
 * re-ranker" (kind "port": the reference ships headers only).
 *
 * Every function cites the reference contract it restates (paths relative to
 * the upstream tree: proj/include/espn/<name>.hpp and SPEC.md).  Build flags must
 * keep -ffp-contract=off so a*b+c is never fused.
 *
 * Parity pinning: the fp16 codec is checked against the reference's own
 * half.hpp compiled in oracle/_ref (all 65,536 codes; recipe `make -C oracle ref`,
 * fixture tests/golden/half_ref_codec.npz made by tests/golden/make_golden.py,
 * checked in tests/test_oracle.py), and scoring/rank/aggregate against SPEC.md's known-answer
 * examples.
 */
#ifndef ESPN_ORACLE_H
#define ESPN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numbering as include/espn_gpu.h, one per error class of
 * proj/include/espn/error.hpp:14-42. */
enum {
  EO_OK = 0,
  EO_INVALID_INPUT = 1,
  EO_INVALID_STATE = 2,
  EO_INVALID_CONFIG = 3,
  EO_FORMAT = 4,
  EO_IO = 5,
  EO_DATA_INTEGRITY = 6
};

enum { EO_DTYPE_F16 = 0, EO_DTYPE_BF16 = 1, EO_DTYPE_F32 = 2 };

/* ---- L0: codecs (half.hpp:11-76, IEEE-correct incl. subnormals) ---- */
uint16_t eo_float_to_half(float f);
float eo_half_to_float(uint16_t h);
uint16_t eo_float_to_bf16(float f);
float eo_bf16_to_float(uint16_t h);
void eo_encode(const float* in, uint16_t* out, size_t n, int dtype);
void eo_decode(const uint16_t* in, float* out, size_t n, int dtype);

/* ---- L1: scoring (scoring.hpp:7-21) ---- */
float eo_dot_f32(const float* a, const float* b, uint32_t d);
float eo_maxsim_score(const float* q, uint32_t nq, const float* doc, uint32_t t,
                      uint32_t d);
float eo_aggregate_score(float cls_score, float bow_score, float alpha);
/* rank (scoring.hpp:16-18): sort by (score desc, doc_id asc); rejects duplicate
 * ids and non-finite scores with EO_INVALID_INPUT. */
int eo_rank(const uint32_t* ids, const float* scores, size_t n, uint32_t* out_ids,
            float* out_scores);

/* ---- L2b: the HBM-tier table restated as CSR (store.hpp:13-35 layout) ----
 * rows[row_ptr[i] .. row_ptr[i+1]) hold doc i's t_i token rows, d values each,
 * encoded as `dtype` (2-byte codes; F32 not used for tables).  d_cls and
 * value_width are the on-disk record parameters (store.hpp:25-34) used only for
 * QueryStats byte accounting. */
typedef struct {
  uint64_t n_docs;
  uint32_t d;
  uint32_t dtype;
  const uint64_t* row_ptr; /* n_docs + 1 */
  const uint16_t* rows;    /* row_ptr[n_docs] * d */
  uint32_t d_cls;          /* record layout, for byte accounting */
  uint32_t value_width;    /* 2 or 4 */
  uint32_t alignment;      /* 1, 512, 4096 */
  uint32_t direct_io;      /* 1: counters as ReadMode::direct */
} eo_table;

/* record_bytes (store.hpp:32-34): exact payload (d_cls + t*d) * value_width. */
uint64_t eo_record_bytes(const eo_table* t, uint64_t doc);
/* gather (StoreHandle::fetch_batch, store.hpp:91-94): request order, duplicates
 * allowed, unknown id -> EO_INVALID_INPUT.  out_row_ptr[n+1]; out_rows is
 * sum(t)*d codes.  Pass out_rows == NULL to only fill out_row_ptr. */
int eo_gather(const eo_table* t, const uint32_t* ids, size_t n, uint64_t* out_row_ptr,
              uint16_t* out_rows);

/* ---- L3: PipelineConfig subset used by stages 3-6 (pipeline.hpp:11-29) ---- */
typedef struct {
  uint32_t rerank_count;  /* R */
  uint32_t final_k;       /* k */
  float alpha;
  int32_t prefetch_enabled;
  int32_t partial_rerank_enabled;
} eo_config;

/* QueryStats byte/count fields (pipeline.hpp:45-53). */
typedef struct {
  uint64_t prefetched_count;
  uint64_t needed_count;
  uint64_t missed_count;
  double hit_rate;
  uint64_t prefetch_bytes;
  uint64_t critical_fetch_bytes;
  uint64_t critical_blocks_read;
  uint64_t needed_payload_bytes;
} eo_stats;

/* validate_config restricted to the re-rank knobs (pipeline.hpp:31-32,
 * SPEC.md:264-265): final_k >= 1, R >= final_k unless partial re-rank. */
int eo_validate_config(const eo_config* cfg);

/* Stages 3-6 of run_query (SPEC.md:276 (3)-(6), pipeline.hpp:56-64) for one
 * query whose final candidate list (ivf.hpp:45-50, sorted (cls desc, id asc))
 * is given.  needed = first min(R, n_cand) candidates; missed = needed \
 * prefetched; every needed doc is scored maxsim+aggregate (the prefetched ones
 * "early", the missed ones on the critical path -- identical arithmetic);
 * tail [R, n) scored alpha*cls when partial re-rank is on, else absent;
 * rank; truncate to final_k.  q_tokens are fp32 (types.hpp:33-44); callers that
 * compare against a reduced-precision GPU path pass them already rounded.
 * out_ids/out_scores need room for final_k entries.  stats may be NULL. */
int eo_rerank_query(const eo_table* t, const float* q_tokens, uint32_t nq,
                    const uint32_t* cand_ids, const float* cand_cls, uint32_t n_cand,
                    const uint32_t* prefetched_ids, uint32_t n_prefetched,
                    const eo_config* cfg, uint32_t* out_ids, float* out_scores,
                    uint32_t* out_n, eo_stats* stats);

/* Same for every query of a batch (run_batch, pipeline.hpp:81-85): queries in
 * parallel on `nthreads` host threads, results identical to serial calls.
 * q_tokens: B*nq*d; cand_offsets: B+1 (CSR over cand_ids/cand_cls); outputs are
 * B*final_k (out_n[B]).  Returns the first failing query's status. */
int eo_rerank_batch(const eo_table* t, const float* q_tokens, uint32_t n_queries,
                    uint32_t nq, const uint32_t* cand_ids, const float* cand_cls,
                    const uint64_t* cand_offsets, const eo_config* cfg, uint32_t* out_ids,
                    float* out_scores, uint32_t* out_n, int nthreads);

/* Scores only: bow MaxSim of every (query, candidate) pair of a batch, no
 * aggregation -- used to check the GPU MaxSim stage in isolation. */
int eo_maxsim_batch(const eo_table* t, const float* q_tokens, uint32_t n_queries,
                    uint32_t nq, const uint32_t* cand_ids, const uint64_t* cand_offsets,
                    float* out_scores, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
