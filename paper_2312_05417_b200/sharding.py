"""Doc-id sharding of a re-rank batch across G devices.

owner(doc) = doc_id % G.  Each query's final candidate list (sorted cls desc,
id asc; ivf.hpp:45-46) is split stably by owner, so every shard's sub-list is
still sorted.  The needed set of the query is the global top-R prefix
(SPEC.md:276 (3)); a shard's needed count is how many of ITS candidates fall in
that prefix -- its needed set is then a prefix of its sub-list, which is what
espn_rerank_args.needed_counts expresses.  Each shard returns its local top-k;
the global top-k is contained in the union of the local top-k lists, so one
all-gather of G x (B x k) entries plus a merge (espn_gpu_merge_topk) recovers
exactly the unsharded result.
"""
from __future__ import annotations

import numpy as np


def split_by_owner(ids: np.ndarray, cls: np.ndarray, offsets: np.ndarray, rerank_count: int,
                   n_shards: int, shard: int):
    """Returns (ids, cls, offsets, needed_counts) of shard `shard`."""
    ids = np.asarray(ids, np.uint32)
    cls = np.asarray(cls, np.float32)
    off = np.asarray(offsets, np.int64)
    n = off[1:] - off[:-1]
    pos = np.arange(ids.size, dtype=np.int64) - np.repeat(off[:-1], n)
    mine = (ids % n_shards) == shard
    in_r = pos < rerank_count
    cm = np.concatenate([[0], np.cumsum(mine)])
    cn = np.concatenate([[0], np.cumsum(mine & in_r)])
    local_off = cm[off].astype(np.uint64)
    needed = (cn[off[1:]] - cn[off[:-1]]).astype(np.uint32)
    return ids[mine].copy(), cls[mine].copy(), local_off, needed


def merge_ranked(lists_ids, lists_scores, lists_counts, k: int):
    """Host restatement of espn_gpu_merge_topk for one query: the union of the
    per-shard ranked lists, ranked by (score desc, doc_id asc), first k."""
    ent = []
    for ids, sc, c in zip(lists_ids, lists_scores, lists_counts):
        ent += [(float(sc[i]), int(ids[i])) for i in range(int(c))]
    ent.sort(key=lambda e: (-e[0], e[1]))
    ent = ent[:k]
    return np.asarray([e[1] for e in ent], np.uint32), np.asarray([e[0] for e in ent], np.float32)
