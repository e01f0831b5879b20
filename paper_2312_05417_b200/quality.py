"""Quality harness (metrics.hpp:10-20).

Checks that re-ranking on the GPU preserves retrieval quality, not only
scores: MRR@k / Recall@k of the device re-ranker over an R sweep (the paper's
partial re-ranking trade-off, PAPER §4.4 "maintain 99.3-99.7% of the MRR@10
score").  The metrics themselves are api.mrr_at_k / recall_at_k /
load_qrels (C++: espn::gpu::mrr_at_k ...).

Synthetic evaluation set (no network for MS MARCO): every query's relevant
doc is its source doc (queries are perturbed copies of its rows, synth.py);
the first-stage candidate list places that doc at a geometric rank
(mean `mean_rank`, default 10: a CLS-only first stage with MRR@10 ~0.2) and
drops it for a fraction `miss` of the queries, like a first-stage retriever
with imperfect recall.  Real qrels plug in through
load_qrels.

    python -m paper_2312_05417_b200.quality [--docs 200000 --queries 512 --K 1000]
"""
from __future__ import annotations

import argparse
import json
from typing import Dict, Sequence

import numpy as np

from . import api, synth


def make_eval_set(n_docs: int = 20000, d: int = 32, n_queries: int = 64, K: int = 1000, t_min: int = 1,
                  t_max: int = 63, nq: int = 32, dtype: str = "f16", mean_rank: float = 10.0, miss: float = 0.1,
                  seed: int = 5):
    """(row_ptr, codes, q, ids, cls, off, qrels): CSR candidates sorted
    (cls desc, id asc) with the relevant doc at a geometric first-stage rank."""
    row_ptr, codes = synth.make_table(n_docs, d, t_min, t_max, dtype=dtype, seed=seed)
    q, src = synth.make_queries(row_ptr, codes, d, n_queries, nq=nq, dtype=dtype, seed=seed + 1)
    rng = np.random.default_rng(seed + 2)
    K = min(K, n_docs)
    ids = np.empty((n_queries, K), np.uint32)
    cls = np.empty((n_queries, K), np.float32)
    for b in range(n_queries):
        others = rng.permutation(n_docs - 1)[:K].astype(np.int64)
        others[others >= src[b]] += 1  # K distinct ids != src
        s = np.sort(rng.random(K, dtype=np.float32))[::-1]
        c = others.copy()
        if rng.random() >= miss:
            pos = min(int(rng.geometric(1.0 / mean_rank)) - 1, K - 1)
            c[pos] = src[b]
        order = np.lexsort((c, -s))  # cls desc, id asc (ivf.hpp:45-46)
        ids[b], cls[b] = c[order], s[order]
    off = np.arange(n_queries + 1, dtype=np.uint64) * K
    qrels = {b: {int(src[b])} for b in range(n_queries)}
    return row_ptr, codes, q, ids.ravel(), cls.ravel(), off, qrels


def results_from_arrays(ids: np.ndarray, counts: np.ndarray) -> Dict[int, list]:
    return {b: [int(x) for x in ids[b, :int(counts[b])]] for b in range(ids.shape[0])}


def first_stage_results(ids, off, k: int) -> Dict[int, list]:
    return {b: [int(x) for x in ids[int(off[b]):int(off[b + 1])][:k]] for b in range(len(off) - 1)}


def rerank_sweep(store: api.GpuStore, q, ids, cls, off, qrels, Rs: Sequence[int] = (16, 64, 256, 1000),
                 k: int = 10, alpha: float = 1.0, kernel: str = "auto") -> dict:
    """MRR@k / Recall@k of the device re-ranker at each R (partial re-ranking:
    the tail keeps alpha*cls), plus the first-stage order."""
    B = len(off) - 1
    rr = api.Reranker(store, B, max(int(off[-1]), 1), q.shape[1])
    out = {"k": k, "first_stage": {"mrr": api.mrr_at_k(first_stage_results(ids, off, k), qrels, k),
                                   "recall": api.recall_at_k(first_stage_results(ids, off, k), qrels, k)},
           "R": {}}
    try:
        for R in Rs:
            cfg = api.PipelineConfig(rerank_count=int(R), final_k=k, alpha=alpha, partial_rerank_enabled=True)
            gi, _, gc, _ = rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kernel)
            res = results_from_arrays(gi, gc)
            out["R"][int(R)] = {"mrr": api.mrr_at_k(res, qrels, k), "recall": api.recall_at_k(res, qrels, k)}
    finally:
        rr.close()
    Rmax = max(out["R"])
    out["mrr_ratio_vs_Rmax"] = {R: (v["mrr"] / out["R"][Rmax]["mrr"] if out["R"][Rmax]["mrr"] else None)
                                for R, v in out["R"].items()}
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--docs", type=int, default=200000)
    ap.add_argument("--queries", type=int, default=512)
    ap.add_argument("--K", type=int, default=1000)
    ap.add_argument("--d", type=int, default=32)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--R", default="16,64,256,1000")
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--qrels", default=None, help="TREC qrels file (replaces the synthetic relevance)")
    a = ap.parse_args(argv)
    rp, codes, q, ids, cls, off, qrels = make_eval_set(a.docs, a.d, a.queries, a.K, dtype=a.dtype)
    if a.qrels:
        qrels = api.load_qrels(a.qrels)
    store = api.GpuStore(rp, codes, a.d, a.dtype)
    try:
        r = rerank_sweep(store, q, ids, cls, off, qrels, [int(x) for x in a.R.split(",")], a.k)
    finally:
        store.close()
    r["workload"] = {"docs": a.docs, "queries": a.queries, "K": a.K, "d": a.d, "dtype": a.dtype}
    print(json.dumps(r))


if __name__ == "__main__":
    main()
