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


# ---- the packed exchange block of espn_gpu_rerank_sharded (shard.cuh) ------------
PACK_HEADER_WORDS = 4


def pack_words(bq: int, k: int) -> int:
    """int32 words of one rank's block: header + ids + scores + counts."""
    return PACK_HEADER_WORDS + bq * (2 * k + 1)


def pack_block(err: int, ids, scores, counts, k: int) -> np.ndarray:
    """Host restatement of a rank's packed block: [err, 0, 0, 0 | ids BQ x k |
    scores BQ x k (fp32 bits) | counts BQ] (int32 words)."""
    ids = np.asarray(ids, np.uint32).reshape(-1, k)
    bq = ids.shape[0]
    blk = np.zeros(pack_words(bq, k), np.int32)
    blk[0] = np.int32(np.uint32(err).view(np.int32))
    blk[PACK_HEADER_WORDS:PACK_HEADER_WORDS + bq * k] = ids.ravel().view(np.int32)
    blk[PACK_HEADER_WORDS + bq * k:PACK_HEADER_WORDS + 2 * bq * k] = \
        np.asarray(scores, np.float32).reshape(-1).view(np.int32)
    blk[PACK_HEADER_WORDS + 2 * bq * k:] = np.asarray(counts, np.uint32).view(np.int32)
    return blk


def unpack_block(blk: np.ndarray, bq: int, k: int):
    """(err, ids[BQ,k], scores[BQ,k], counts[BQ]) of one packed block."""
    blk = np.asarray(blk, np.int32)
    h = PACK_HEADER_WORDS
    return (int(blk[0].view(np.uint32)), blk[h:h + bq * k].view(np.uint32).reshape(bq, k),
            blk[h + bq * k:h + 2 * bq * k].view(np.float32).reshape(bq, k),
            blk[h + 2 * bq * k:h + 2 * bq * k + bq].view(np.uint32))


def merge_packed(recv: np.ndarray, n_ranks: int, n_queries: int, k: int, replica: bool = False):
    """Host restatement of the device merge of the all-gathered blocks: SHARD
    -> per query the union of the ranks' ranked lists by (score desc, doc_id
    asc), first k; REPLICA -> query b from the block of the rank that owns its
    slice.  Returns (err OR of all ranks, ids[B,k], scores[B,k], counts[B])."""
    bq = -(-n_queries // n_ranks) if replica else n_queries
    P = pack_words(bq, k)
    blocks = [unpack_block(np.asarray(recv, np.int32)[r * P:(r + 1) * P], bq, k) for r in range(n_ranks)]
    err = 0
    for e, *_ in blocks:
        err |= e
    ids = np.zeros((n_queries, k), np.uint32)
    sc = np.zeros((n_queries, k), np.float32)
    cnt = np.zeros(n_queries, np.uint32)
    for b in range(n_queries):
        if replica:
            r, i = divmod(b, bq)
            _, bi, bs, bc = blocks[r]
            c = int(bc[i])
            ids[b, :c], sc[b, :c], cnt[b] = bi[i, :c], bs[i, :c], c
        else:
            mi, ms = merge_ranked([bl[1][b] for bl in blocks], [bl[2][b] for bl in blocks],
                                  [bl[3][b] for bl in blocks], k)
            c = mi.shape[0]
            ids[b, :c], sc[b, :c], cnt[b] = mi, ms, c
    return err, ids, sc, cnt


def shard_table(row_ptr, codes, d: int, n_shards: int, shard: int):
    """The CSR of doc-id shard `shard` (local doc i = global id i*G + shard)."""
    row_ptr = np.asarray(row_ptr, np.uint64)
    n = row_ptr.shape[0] - 1
    gids = np.arange(shard, n, n_shards, dtype=np.int64)
    t = (row_ptr[gids + 1] - row_ptr[gids]).astype(np.int64)
    lrp = np.zeros(gids.size + 1, np.uint64)
    lrp[1:] = np.cumsum(t)
    idx = np.concatenate([np.arange(int(row_ptr[g]), int(row_ptr[g + 1])) for g in gids]) if gids.size else \
        np.zeros(0, np.int64)
    rows = np.asarray(codes).reshape(-1, d)[idx]
    return lrp, rows.reshape(-1)
