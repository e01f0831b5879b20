"""The persistent re-rank server (espn_gpu_server_start): one
long-lived tcgen05 MaxSim kernel fed by a device-side batch queue.  Served
batches must equal unserved ones bit for bit (same per-unit arithmetic, same
merge) and the oracle; the queue must survive many batches from several
workspaces (slot reuse), CUDA-graph replay, errors, idle exit + relaunch and
stop."""
import time

import numpy as np
import pytest

from helpers import assert_topk_equivalent, oracle_full_scores

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import api, synth  # noqa: E402


def _case(n_docs=20000, B=8, K=600, seed=1, dtype="f16"):
    rp, codes = synth.make_table(n_docs, 32, 1, 63, dtype=dtype, seed=seed)
    q, src = synth.make_queries(rp, codes, 32, B, dtype=dtype, seed=seed + 1)
    ids, cls, off = synth.make_candidates(n_docs, B, K, src=src, seed=seed + 2)
    return rp, codes, q, ids, cls, off


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_served_equals_unserved_and_oracle(oracle, cuda_ok, dtype):
    rp, codes, q, ids, cls, off = _case(dtype=dtype)
    cfg = api.PipelineConfig(rerank_count=500, final_k=10, alpha=0.5, partial_rerank_enabled=True)
    store = api.GpuStore(rp, codes, 32, dtype=dtype)
    rr = api.Reranker(store, len(off) - 1, int(off[-1]), 32)
    ref = [np.copy(x) for x in rr.rerank_arrays(q, ids, cls, off, cfg)[:3]]
    store.server_start()
    assert store.server_running
    for _ in range(4):  # eager, captured, replayed (the synchronous path's graph)
        got = rr.rerank_arrays(q, ids, cls, off, cfg)
        for g, r in zip(got[:3], ref):
            assert np.array_equal(g, r)
    c = rr.counters()
    store.server_stop()
    assert not store.server_running
    # and the oracle (the reference's fp32 query)
    odt = oracle.F16 if dtype == "f16" else oracle.BF16
    ot = oracle.OracleTable(rp, codes, 32, dtype=odt)
    st, obow = oracle.maxsim_batch(ot, q, ids, off)
    st2, oi, os_, on = oracle.rerank_batch(ot, q, ids, cls, off, 500, 10, 0.5, True)
    assert st == 0 and st2 == 0
    for b in range(len(off) - 1):
        a0, a1 = int(off[b]), int(off[b + 1])
        full = oracle_full_scores(obow[a0:a1], cls[a0:a1], 0.5, min(500, a1 - a0), True)
        n = int(on[b])
        assert int(ref[2][b]) == n
        assert_topk_equivalent(ref[0][b, :n], ref[1][b, :n], oi[b, :n], os_[b, :n], ids[a0:a1], full)
    assert c["batches"] >= 5
    rr.close(); store.close()


def test_many_batches_three_workspaces_graphs(cuda_ok):
    # more batches than queue slots, from three workspaces on three streams,
    # each batch a CUDA-graph replay of device-planned work
    import torch
    from paper_2312_05417_b200 import _lib as L
    import ctypes as C
    rp, codes, q, ids, cls, off = _case(n_docs=50000, B=16, K=1000, seed=7)
    store = api.GpuStore(rp, codes, 32)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    B, Cn = len(off) - 1, int(off[-1])
    dq, di, dc = (torch.from_numpy(q).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
                  torch.from_numpy(cls).cuda())
    doff = torch.from_numpy(off.astype(np.int64)).cuda()
    lanes = []
    lib = L.lib()
    for _ in range(3):
        rr = api.Reranker(store, B, Cn, 32, max_list=1000)
        out = torch.zeros(2 * B * 10 + B, dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()
        lanes.append((rr, out, s))
    ref = [x for x in api.Reranker(store, B, Cn, 32).rerank_arrays(q, ids, cls, off, cfg)[:3]]
    store.server_start()
    flags = L.ESPN_RERANK_DEVICE_IO | L.ESPN_RERANK_DEVICE_OFFSETS | L.ESPN_RERANK_ASYNC
    # (while the server runs, allocations and device-wide syncs in the process
    # wait for it to go idle: graphs are captured with the server paused and
    # nothing but the replays runs while it serves)

    def enqueue(rr, out, sp):
        a = L.RerankArgs(n_queries=B, n_query_tokens=32, query_tokens=dq.data_ptr(), cand_ids=di.data_ptr(),
                         cand_cls=dc.data_ptr(), cand_offsets=doff.data_ptr(), rerank_count=1000, final_k=10,
                         alpha=1.0, flags=flags, kernel=0)
        base = out.data_ptr()
        o = L.RerankOut(ids=base, scores=base + 4 * B * 10, counts=base + 8 * B * 10)
        assert lib.espn_gpu_rerank(store.handle, rr.handle, C.byref(a), C.byref(o), C.c_void_p(sp)) == 0, \
            L.last_error()

    graphs = []
    for rr, out, s in lanes:
        with torch.cuda.stream(s):
            enqueue(rr, out, s.cuda_stream)  # eager, served
        s.synchronize()
        rr.sync(s.cuda_stream)
    store.server_pause()
    for rr, out, s in lanes:
        out.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            enqueue(rr, out, torch.cuda.current_stream().cuda_stream)
        graphs.append(g)
    torch.cuda.synchronize()
    store.server_start()  # relaunch before the replays
    for i in range(60):
        rr, out, s = lanes[i % 3]
        with torch.cuda.stream(s):
            graphs[i % 3].replay()
    for rr, out, s in lanes:
        s.synchronize()
        rr.sync(s.cuda_stream)
    hs = [out.cpu().numpy() for _, out, _ in lanes]
    for h in hs:
        assert np.array_equal(h[:B * 10].view(np.uint32).reshape(B, 10), ref[0])
        assert np.array_equal(h[B * 10:2 * B * 10].view(np.float32).reshape(B, 10), ref[1])
    store.server_stop()
    for rr, _, _ in lanes:
        rr.close()
    store.close()


def test_idle_exit_relaunch_errors_and_stop(cuda_ok):
    rp, codes, q, ids, cls, off = _case(seed=21)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, len(off) - 1, int(off[-1]), 32)
    cfg = api.PipelineConfig(rerank_count=600, final_k=10)
    ref = [np.copy(x) for x in rr.rerank_arrays(q, ids, cls, off, cfg)[:3]]
    store.server_start(idle_us=5000)
    got = rr.rerank_arrays(q, ids, cls, off, cfg)
    assert np.array_equal(got[0], ref[0])
    time.sleep(0.2)  # idle: the server exits by itself
    assert not store.server_running
    got = rr.rerank_arrays(q, ids, cls, off, cfg)  # relaunched by the served call
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    # a duplicate id is still rejected, and the server keeps serving
    bad = ids.copy()
    bad[int(off[1]) + 3] = bad[int(off[1])]
    with pytest.raises(api.InvalidInputError):
        rr.rerank_arrays(q, bad, cls, off, cfg)
    got = rr.rerank_arrays(q, ids, cls, off, cfg)
    assert np.array_equal(got[0], ref[0])
    # batches the server cannot take fail cleanly instead of waiting for an SM
    with pytest.raises(api.InvalidStateError):
        rr.rerank_arrays(q, ids, cls, off, api.PipelineConfig(rerank_count=600, final_k=64))
    for kern in ("simt", "small"):  # CUDA-core kernels need SMs the server holds
        with pytest.raises(api.InvalidStateError):
            rr.rerank_arrays(q[:1], ids[:int(off[1])], cls[:int(off[1])], off[:2], cfg, kernel=kern)
    store.server_stop()
    got = rr.rerank_arrays(q, ids, cls, off, api.PipelineConfig(rerank_count=600, final_k=64))
    assert got[2][0] == 64
    rr.close(); store.close()
