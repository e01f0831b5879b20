"""Multi-GPU re-rank through the C-ABI (espn_gpu_rerank_sharded and its
phases) on ONE B200: the SHARD and REPLICA placements run their G ranks'
local passes on the same device (espn_gpu_shard_pack per rank, the blocks
gathered by a device copy standing in for ncclAllGather, espn_gpu_shard_merge),
checked against the unsharded CPU oracle and against the host restatement of
the exchange layout (sharding.pack_block / merge_packed, also driven over
gloo in test_sharding_gloo.py).  The NCCL call itself runs with a one-rank
communicator (the boxes here have one GPU), eagerly and captured in a CUDA
graph, and through the single-process group entry point."""
import ctypes as C

import numpy as np
import pytest

from helpers import assert_topk_equivalent, oracle_full_scores

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import _lib as L  # noqa: E402
from paper_2312_05417_b200 import api, sharding, synth  # noqa: E402

N_DOCS, D, B, K, FINAL_K = 6000, 32, 6, 500, 10


def _cudart():
    return C.CDLL("libcudart.so.12")


def _case(seed=3):
    rp, codes = synth.make_table(N_DOCS, D, 1, 63, seed=seed)
    q, src = synth.make_queries(rp, codes, D, B, seed=seed + 1)
    ids, cls, off = synth.make_candidates(N_DOCS, B, K, src=src, seed=seed + 2)
    return rp, codes, q, ids, cls, off


def _dev(q, ids, cls):
    import torch
    return (torch.from_numpy(np.ascontiguousarray(q, np.float32)).cuda(),
            torch.from_numpy(ids.view(np.int32)).cuda(), torch.from_numpy(cls).cuda())


def _check_global(oracle, rp, codes, q, ids, cls, off, cfg, gi, gs, gc):
    ot = oracle.OracleTable(rp, codes, D)
    qf = np.ascontiguousarray(q, np.float32)
    st, obow = oracle.maxsim_batch(ot, qf, ids, off)
    assert st == 0
    st, oi, os_, on = oracle.rerank_batch(ot, qf, ids, cls, off, cfg.rerank_count, cfg.final_k, cfg.alpha,
                                          cfg.partial_rerank_enabled)
    assert st == 0
    for b in range(len(off) - 1):
        a0, a1 = int(off[b]), int(off[b + 1])
        need = min(a1 - a0, cfg.rerank_count)
        full = oracle_full_scores(obow[a0:a1], cls[a0:a1], cfg.alpha, need, cfg.partial_rerank_enabled)
        n = int(on[b])
        assert int(gc[b]) == n, f"query {b}"
        assert_topk_equivalent(gi[b, :n], gs[b, :n], oi[b, :n], os_[b, :n], ids[a0:a1], full, ctx=f"query {b}")


def _gather_blocks(blocks, P):
    """Stand-in for ncclAllGather on one device: the ranks' blocks, contiguous."""
    import torch
    recv = torch.empty(len(blocks) * P, dtype=torch.int32, device="cuda")
    rt = _cudart()
    torch.cuda.synchronize()
    for g, (ptr, words) in enumerate(blocks):
        assert words == P
        assert rt.cudaMemcpy(C.c_void_p(recv.data_ptr() + 4 * g * P), C.c_void_p(ptr), C.c_size_t(4 * P), 3) == 0
    return recv


@pytest.mark.parametrize("G,R,partial,alpha", [(2, K, False, 1.0), (3, 64, True, 0.5), (4, 200, False, 2.0)])
def test_shard_placement_pack_merge(oracle, cuda_ok, G, R, partial, alpha):
    import torch
    rp, codes, q, ids, cls, off = _case(seed=G)
    cfg = api.PipelineConfig(rerank_count=R, final_k=FINAL_K, alpha=alpha, partial_rerank_enabled=partial)
    dq, di, dc = _dev(q, ids, cls)
    stores, rrs, blocks = [], [], []
    for g in range(G):
        lrp, lcodes = sharding.shard_table(rp, codes, D, G, g)
        st = api.GpuStore(lrp, lcodes, D, shard_count=G, shard_index=g)
        rr = api.Reranker(st, B, int(off[-1]), 32)
        blocks.append(rr.shard_pack(dq, di, dc, off, cfg, G, g))
        stores.append(st)
        rrs.append(rr)
    P = sharding.pack_words(B, FINAL_K)
    recv = _gather_blocks(blocks, P)
    h = recv.cpu().numpy()
    # each rank's block: its own candidates' local top-k (the split the host restates)
    for g in range(G):
        err, bi, bs, bc = sharding.unpack_block(h[g * P:(g + 1) * P], B, FINAL_K)
        assert err == 0
        s_ids, s_cls, s_off, s_need = sharding.split_by_owner(ids, cls, off, R, G, g)
        for b in range(B):
            assert np.all(bi[b, :bc[b]] % G == g)
            assert set(bi[b, :bc[b]].tolist()) <= set(s_ids[int(s_off[b]):int(s_off[b + 1])].tolist())
    out = rrs[0].shard_merge(dq, di, dc, off, cfg, recv, G)
    gi, gs, gc = (x.cpu().numpy() for x in out)
    gi = gi.view(np.uint32)
    # the device merge == the host restatement of the merge over the same blocks
    herr, hi, hs, hc = sharding.merge_packed(h, G, B, FINAL_K)
    assert herr == 0 and np.array_equal(gc.view(np.uint32), hc)
    for b in range(B):
        n = int(hc[b])
        assert np.array_equal(gi[b, :n], hi[b, :n]) and np.array_equal(gs[b, :n], hs[b, :n])
    _check_global(oracle, rp, codes, q, ids, cls, off, cfg, gi, gs, gc)
    for rr, st in zip(rrs, stores):
        rr.close(); st.close()
    del torch


@pytest.mark.parametrize("G", [2, 4, 8])
def test_replica_placement_pack_merge(oracle, cuda_ok, G):
    rp, codes, q, ids, cls, off = _case(seed=10 + G)
    cfg = api.PipelineConfig(rerank_count=300, final_k=FINAL_K, partial_rerank_enabled=True)
    dq, di, dc = _dev(q, ids, cls)
    store = api.GpuStore(rp, codes, D)
    rrs = [api.Reranker(store, B, int(off[-1]), 32) for _ in range(G)]
    blocks = [rr.shard_pack(dq, di, dc, off, cfg, G, g) for g, rr in enumerate(rrs)]
    bq = -(-B // G)
    recv = _gather_blocks(blocks, sharding.pack_words(bq, FINAL_K))
    gi, gs, gc = (x.cpu().numpy() for x in rrs[0].shard_merge(dq, di, dc, off, cfg, recv, G))
    herr, hi, hs, hc = sharding.merge_packed(recv.cpu().numpy(), G, B, FINAL_K, replica=True)
    assert herr == 0 and np.array_equal(gc.view(np.uint32), hc) and np.array_equal(gi.view(np.uint32), hi)
    _check_global(oracle, rp, codes, q, ids, cls, off, cfg, gi.view(np.uint32), gs, gc)
    # REPLICA with one rank is exactly the plain call
    ref = rrs[0].rerank_arrays(q, ids, cls, off, cfg)
    blk = rrs[1].shard_pack(dq, di, dc, off, cfg, 1, 0)
    r1 = _gather_blocks([blk], sharding.pack_words(B, FINAL_K))
    one = [x.cpu().numpy() for x in rrs[1].shard_merge(dq, di, dc, off, cfg, r1, 1)]
    assert np.array_equal(one[0].view(np.uint32), ref[0]) and np.array_equal(one[1], ref[1])
    for rr in rrs:
        rr.close()
    store.close()


def test_shard_errors_surface_on_every_rank(cuda_ok):
    rp, codes, q, ids, cls, off = _case(seed=30)
    ids = ids.copy()
    ids[7] = 2 * N_DOCS + 1  # unknown doc, owned by rank 1 of 2
    cfg = api.PipelineConfig(rerank_count=K, final_k=FINAL_K)
    dq, di, dc = _dev(q, ids, cls)
    stores, rrs, blocks = [], [], []
    for g in range(2):
        lrp, lcodes = sharding.shard_table(rp, codes, D, 2, g)
        st = api.GpuStore(lrp, lcodes, D, shard_count=2, shard_index=g)
        rr = api.Reranker(st, B, int(off[-1]), 32)
        blocks.append(rr.shard_pack(dq, di, dc, off, cfg, 2, g))
        stores.append(st)
        rrs.append(rr)
    recv = _gather_blocks(blocks, sharding.pack_words(B, FINAL_K))
    errs = [sharding.unpack_block(recv.cpu().numpy()[g * sharding.pack_words(B, FINAL_K):], B, FINAL_K)[0]
            for g in range(2)]
    assert errs[0] == 0 and errs[1] != 0  # only the owner saw it ...
    for g in range(2):  # ... but both ranks' merges report it
        with pytest.raises(api.DataIntegrityError):
            rrs[g].shard_merge(dq, di, dc, off, cfg, recv, 2)
    # a sharded table needs a communicator of shard_count ranks
    uid = api.nccl_unique_id()
    comm = api.NcclComm(1, uid, 0, 0)
    with pytest.raises(api.InvalidConfigError):
        rrs[0].rerank_sharded(q, ids, cls, off, cfg, comm)
    comm.close()
    for rr, st in zip(rrs, stores):
        rr.close(); st.close()


def test_nccl_one_rank_eager_graph_and_group(oracle, cuda_ok):
    import torch
    rp, codes, q, ids, cls, off = _case(seed=40)
    cfg = api.PipelineConfig(rerank_count=400, final_k=FINAL_K)
    store = api.GpuStore(rp, codes, D)
    rr = api.Reranker(store, B, int(off[-1]), 32)
    ref = rr.rerank_arrays(q, ids, cls, off, cfg)
    comm = api.NcclComm(1, api.nccl_unique_id(), 0, 0)
    gi, gs, gc = rr.rerank_sharded(q, ids, cls, off, cfg, comm)  # host arrays in and out
    assert np.array_equal(gi, ref[0]) and np.array_equal(gs, ref[1]) and np.array_equal(gc, ref[2])
    # device arrays + device offsets, ASYNC: captured in a CUDA graph and replayed
    dq, di, dc = _dev(q, ids, cls)
    doff = torch.from_numpy(off.astype(np.int64)).cuda()
    out = (torch.zeros((B, FINAL_K), dtype=torch.int32, device="cuda"),
           torch.zeros((B, FINAL_K), dtype=torch.float32, device="cuda"),
           torch.zeros(B, dtype=torch.int32, device="cuda"))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rr.rerank_sharded(dq, di, dc, doff, cfg, comm, device_io=True, device_offsets=True, out=out,
                          stream=s.cuda_stream, sync=False)  # sizes the exchange buffers outside the capture
    s.synchronize()
    rr.sync(s.cuda_stream)
    for o in out:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rr.rerank_sharded(dq, di, dc, doff, cfg, comm, device_io=True, device_offsets=True, out=out,
                          stream=torch.cuda.current_stream().cuda_stream, sync=False)
    for _ in range(3):
        for o in out:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy().view(np.uint32), ref[0])
        assert np.array_equal(out[1].cpu().numpy(), ref[1])
    rr.sync(s.cuda_stream)
    comm.close()
    # single-process group entry point (ncclCommInitAll over the visible devices)
    comms = api.NcclComm.init_all([0])
    lib = L.lib()
    offs = np.ascontiguousarray(off, np.uint64)
    a = L.RerankArgs(n_queries=B, n_query_tokens=32, query_tokens=q.ctypes.data, cand_ids=ids.ctypes.data,
                     cand_cls=cls.ctypes.data, cand_offsets=offs.ctypes.data, rerank_count=400, final_k=FINAL_K,
                     alpha=1.0, flags=0, kernel=0)
    oi, osc, oc = np.zeros((B, FINAL_K), np.uint32), np.zeros((B, FINAL_K), np.float32), np.zeros(B, np.uint32)
    o = L.RerankOut(ids=oi.ctypes.data, scores=osc.ctypes.data, counts=oc.ctypes.data)
    tabs = (C.c_void_p * 1)(store.handle.value)
    wss = (C.c_void_p * 1)(rr.handle.value)
    cms = (C.c_void_p * 1)(comms[0].handle.value)
    sts = (C.c_void_p * 1)(None)
    rc = lib.espn_gpu_rerank_sharded_multi(1, C.addressof(tabs), C.addressof(wss), C.byref(a), C.addressof(o),
                                           C.addressof(cms), C.addressof(sts))
    assert rc == 0, L.last_error()
    assert np.array_equal(oi, ref[0]) and np.array_equal(osc, ref[1])
    comms[0].close()
    rr.close(); store.close()


@pytest.mark.parametrize("placement", ["shard", "replica"])
def test_sharded_local_pass_small_kernel_bitexact(oracle, cuda_ok, placement):
    """The ranks' local passes through the single-launch small-batch kernel
    (device offsets, per-query needed counts from the owner split, base
    offsets for REPLICA query slices): exact arithmetic, so the merged global
    lists equal the oracle's bit for bit."""
    G = 2
    rp, codes, q, ids, cls, off = _case(seed=40)
    cfg = api.PipelineConfig(rerank_count=200, final_k=FINAL_K, alpha=0.5, partial_rerank_enabled=True)
    dq, di, dc = _dev(q, ids, cls)
    stores, rrs, blocks = [], [], []
    for g in range(G):
        if placement == "shard":
            lrp, lcodes = sharding.shard_table(rp, codes, D, G, g)
            st = api.GpuStore(lrp, lcodes, D, shard_count=G, shard_index=g)
        else:
            st = api.GpuStore(rp, codes, D)
        rr = api.Reranker(st, B, int(off[-1]), 32, max_list=K)  # small kernel: lists <= 2048
        blocks.append(rr.shard_pack(dq, di, dc, off, cfg, G, g, kernel="small"))
        stores.append(st)
        rrs.append(rr)
    bq = B if placement == "shard" else -(-B // G)
    recv = _gather_blocks(blocks, sharding.pack_words(bq, FINAL_K))
    gi, gs, gc = (x.cpu().numpy() for x in rrs[0].shard_merge(dq, di, dc, off, cfg, recv, G))
    ot = oracle.OracleTable(rp, codes, D)
    st_, oi, os_, on = oracle.rerank_batch(ot, np.ascontiguousarray(q, np.float32), ids, cls, off,
                                           cfg.rerank_count, cfg.final_k, cfg.alpha, cfg.partial_rerank_enabled)
    assert st_ == 0
    assert np.array_equal(gc.astype(np.int64), np.asarray(on, np.int64))
    for b in range(B):
        n = int(on[b])
        assert np.array_equal(gi.view(np.uint32)[b, :n].astype(np.int64), np.asarray(oi[b, :n], np.int64)), b
        assert np.array_equal(gs[b, :n].view(np.uint32), np.asarray(os_[b, :n], np.float32).view(np.uint32)), b
    for rr, st in zip(rrs, stores):
        rr.close(); st.close()
