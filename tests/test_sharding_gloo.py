"""Multi-GPU host logic on CPU with the gloo backend,
world_size 2: doc-id sharding (owner = id % G) of every query's candidate
list, per-shard re-rank of its share (the CPU oracle stands in for the GPU
here), ONE all-gather of the packed per-shard top-k, merge -> must equal the
unsharded re-rank exactly (ids and scores), for full and partial re-rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_05417_b200 import synth
from paper_2312_05417_b200.sharding import merge_ranked, split_by_owner

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


def _worker(rank, port, R, partial, alpha, result_q):
    import oracle_py
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    rp, codes, q, ids, cls, off = _case()
    t = oracle_py.OracleTable(rp, codes, D)
    qr = oracle_py.round_to(q)
    s_ids, s_cls, s_off, s_need = split_by_owner(ids, cls, off, R, G, rank)
    assert np.all(s_ids % G == rank)
    packed = np.zeros((B, 2 * FINAL_K + 1), np.float64)
    for b in range(B):
        a0, a1 = int(s_off[b]), int(s_off[b + 1])
        st, oi, os_, _ = oracle_py.rerank_query(t, qr[b], s_ids[a0:a1], s_cls[a0:a1], int(s_need[b]), FINAL_K,
                                                alpha, partial or int(s_need[b]) < FINAL_K)
        assert st == 0
        n = len(oi)
        packed[b, :n] = oi
        packed[b, FINAL_K:FINAL_K + n] = os_
        packed[b, -1] = n
    mine = torch.from_numpy(packed)
    allp = [torch.zeros_like(mine) for _ in range(G)]
    dist.all_gather(allp, mine)
    if rank == 0:
        merged = []
        for b in range(B):
            lists = [(p[b, :FINAL_K].numpy().astype(np.uint32), p[b, FINAL_K:2 * FINAL_K].numpy().astype(np.float32),
                      int(p[b, -1])) for p in allp]
            mi, ms = merge_ranked([l[0] for l in lists], [l[1] for l in lists], [l[2] for l in lists], FINAL_K)
            merged.append((mi, ms))
        result_q.put(merged)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("R,partial,alpha", [(K, False, 1.0), (64, True, 0.5)])
def test_sharded_rerank_equals_unsharded(oracle, R, partial, alpha):
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, R, partial, alpha, result_q)) for r in range(G)]
    for p in procs:
        p.start()
    merged = result_q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    rp, codes, q, ids, cls, off = _case()
    t = oracle.OracleTable(rp, codes, D)
    st, oi, os_, on = oracle.rerank_batch(t, oracle.round_to(q), ids, cls, off, R, FINAL_K, alpha, partial)
    assert st == 0
    for b in range(B):
        mi, ms = merged[b]
        n = int(on[b])
        assert len(mi) == n
        assert list(mi) == list(oi[b, :n]), f"query {b}"
        assert np.array_equal(ms, os_[b, :n]), f"query {b}"
