"""Multi-GPU host logic on CPU with the gloo backend,
world_size 2, through the EXACT exchange layout of espn_gpu_rerank_sharded
(shard.cuh; restated in sharding.pack_block / merge_packed):

  SHARD   each rank keeps its own candidates (owner = id % G, stable), needed =
          its share of the global top-R prefix, ranks them (the CPU oracle
          stands in for the GPU here), packs [err | ids | scores | counts],
          ONE all-gather, merge -> must equal the unsharded re-rank exactly;
  REPLICA each rank ranks its slice of the queries, the all-gather
          reassembles the batch.

The GPU side of the same layout is pinned in tests/test_sharded_gpu.py (the
device blocks and merge equal these host restatements)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_05417_b200 import synth
from paper_2312_05417_b200.sharding import merge_packed, pack_block, split_by_owner

G = 2
N_DOCS, D, B, K, FINAL_K = 3000, 32, 5, 400, 10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    rp, codes = synth.make_table(N_DOCS, D, 1, 40, seed=11)
    q, src = synth.make_queries(rp, codes, D, B, seed=12)
    ids, cls, off = synth.make_candidates(N_DOCS, B, K, src=src, seed=13)
    return rp, codes, q, ids, cls, off


def local_topk(oracle_py, t, q, ids, cls, off, need, alpha, partial, k):
    """One shard's ranked lists: own needed candidates alpha*cls + MaxSim, own
    tail alpha*cls when partial (SPEC.md:276 (5)), rank (score desc, id asc)."""
    st, bow = oracle_py.maxsim_batch(t, q, ids, off)
    assert st == 0
    n_q = len(off) - 1
    out_i = np.zeros((n_q, k), np.uint32)
    out_s = np.zeros((n_q, k), np.float32)
    out_c = np.zeros(n_q, np.uint32)
    for b in range(n_q):
        a0, a1 = int(off[b]), int(off[b + 1])
        nd = int(need[b])
        s = (np.float32(alpha) * cls[a0:a1]).astype(np.float32)
        s[:nd] = (s[:nd] + bow[a0:a0 + nd]).astype(np.float32)
        cand = ids[a0:a1] if partial else ids[a0:a0 + nd]
        sc = s if partial else s[:nd]
        o = np.lexsort((cand, -sc))[:k]
        out_i[b, :o.size], out_s[b, :o.size], out_c[b] = cand[o], sc[o], o.size
    return out_i, out_s, out_c


def _worker(rank, port, R, partial, alpha, replica, result_q):
    import oracle_py
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    rp, codes, q, ids, cls, off = _case()
    t = oracle_py.OracleTable(rp, codes, D)
    q = np.ascontiguousarray(q, np.float32)
    if replica:
        bq = -(-B // G)
        b0, b1 = min(B, rank * bq), min(B, rank * bq + bq)
        sl_off = (off[b0:b1 + 1] - off[b0]).astype(np.uint64)
        sl_ids, sl_cls = ids[int(off[b0]):int(off[b1])], cls[int(off[b0]):int(off[b1])]
        need = np.minimum(np.diff(sl_off.astype(np.int64)), R)
        li, ls, lc = local_topk(oracle_py, t, q[b0:b1], sl_ids, sl_cls, sl_off, need, alpha, partial, FINAL_K)
        pi, ps, pc = np.zeros((bq, FINAL_K), np.uint32), np.zeros((bq, FINAL_K), np.float32), np.zeros(bq, np.uint32)
        pi[:b1 - b0], ps[:b1 - b0], pc[:b1 - b0] = li, ls, lc
        blk = pack_block(0, pi, ps, pc, FINAL_K)
    else:
        s_ids, s_cls, s_off, s_need = split_by_owner(ids, cls, off, R, G, rank)
        assert np.all(s_ids % G == rank)
        li, ls, lc = local_topk(oracle_py, t, q, s_ids, s_cls, s_off, s_need, alpha, partial, FINAL_K)
        blk = pack_block(0, li, ls, lc, FINAL_K)
    mine = torch.from_numpy(blk)
    allp = [torch.zeros_like(mine) for _ in range(G)]
    dist.all_gather(allp, mine)
    recv = torch.cat(allp).numpy()
    err, mi, ms, mc = merge_packed(recv, G, B, FINAL_K, replica=replica)
    result_q.put((rank, err, mi, ms, mc))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("R,partial,alpha,replica", [(K, False, 1.0, False), (64, True, 0.5, False),
                                                     (K, False, 1.0, True), (64, True, 0.5, True)])
def test_sharded_rerank_equals_unsharded(oracle, R, partial, alpha, replica):
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, R, partial, alpha, replica, result_q)) for r in range(G)]
    for p in procs:
        p.start()
    res = [result_q.get(timeout=300) for _ in range(G)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    rp, codes, q, ids, cls, off = _case()
    t = oracle.OracleTable(rp, codes, D)
    st, oi, os_, on = oracle.rerank_batch(t, np.ascontiguousarray(q, np.float32), ids, cls, off, R, FINAL_K, alpha,
                                          partial)
    assert st == 0
    for rank, err, mi, ms, mc in res:  # every rank holds the same global result
        assert err == 0
        for b in range(B):
            n = int(on[b])
            assert int(mc[b]) == n
            assert list(mi[b, :n]) == list(oi[b, :n]), f"rank {rank} query {b}"
            assert np.array_equal(ms[b, :n], os_[b, :n]), f"rank {rank} query {b}"


def test_pack_layout_round_trip():
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 2**32, size=(3, 4), dtype=np.uint64).astype(np.uint32)
    sc = rng.standard_normal((3, 4)).astype(np.float32)
    cnt = np.array([4, 0, 2], np.uint32)
    blk = pack_block(0x88, ids, sc, cnt, 4)
    assert blk.dtype == np.int32 and blk.size == 4 + 3 * 9
    err, i2, s2, c2 = merge_packed(np.concatenate([blk]), 1, 3, 4, replica=True)
    assert err == 0x88 and np.array_equal(c2, cnt)
    assert np.array_equal(i2[0], ids[0]) and np.array_equal(s2[0].view(np.uint32), sc[0].view(np.uint32))
    assert np.array_equal(i2[2, :2], ids[2, :2])
