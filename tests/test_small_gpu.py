"""GPU parity of the single-launch small-batch re-rank (ESPN_KERNEL_SMALL,
csrc/small.cuh): CUDA-core MaxSim on the fp32 query in the reference's order,
so bow scores, ranked ids, scores and counts are BIT-EXACT against the oracle
(scoring.hpp:7-21, pipeline.hpp:56-64).  Every call goes through the C-ABI."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import _lib as L  # noqa: E402
from paper_2312_05417_b200 import api, synth  # noqa: E402


def _dt(name):
    import oracle_py
    return oracle_py.F16 if name == "f16" else oracle_py.BF16


def _case(n_docs, d, t_max, B, K, nq=32, dtype="f16", seed=1, ragged=False):
    rp, codes = synth.make_table(n_docs, d, 1, t_max, dtype=dtype, seed=seed)
    q, src = synth.make_queries(rp, codes, d, B, nq=nq, dtype=dtype, seed=seed + 1)
    ids, cls, off = synth.make_candidates(n_docs, B, K, src=src, seed=seed + 2)
    if ragged:  # lengths K, 0, K//3, 1, ... cut from the same lists
        rng = np.random.default_rng(seed + 3)
        keep = [K if b == 0 else int(rng.choice([0, 1, K // 3, K])) for b in range(B)]
        ids_l, cls_l, offs = [], [], [0]
        for b in range(B):
            a0 = int(off[b])
            ids_l.append(ids[a0:a0 + keep[b]]); cls_l.append(cls[a0:a0 + keep[b]]); offs.append(offs[-1] + keep[b])
        ids = np.concatenate(ids_l).astype(np.uint32)
        cls = np.concatenate(cls_l).astype(np.float32)
        off = np.asarray(offs, np.uint64)
    return rp, codes, q, ids, cls, off, src


def _exact(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, got):
    gi, gs, gc, gbow = got
    ot = oracle.OracleTable(rp, codes, d, dtype=_dt(dtype))
    qr = np.ascontiguousarray(q, np.float32)  # the reference's fp32 query (types.hpp:33-44)
    st, obow = oracle.maxsim_batch(ot, qr, ids, off)
    assert st == 0
    st, oi, os_, on = oracle.rerank_batch(ot, qr, ids, cls, off, cfg.rerank_count, cfg.final_k, cfg.alpha,
                                          cfg.partial_rerank_enabled)
    assert st == 0
    B = len(off) - 1
    assert np.array_equal(gc.astype(np.int64), np.asarray(on, np.int64))
    for b in range(B):
        a0, a1 = int(off[b]), int(off[b + 1])
        need = min(a1 - a0, cfg.rerank_count)
        assert np.array_equal(gbow[a0:a0 + need].view(np.uint32), obow[a0:a0 + need].view(np.uint32)), b
        n = int(on[b])
        assert np.array_equal(gi[b, :n].astype(np.int64), np.asarray(oi[b, :n], np.int64)), b
        assert np.array_equal(gs[b, :n].view(np.uint32), np.asarray(os_[b, :n], np.float32).view(np.uint32)), b


def _run(rp, codes, d, dtype, q, ids, cls, off, cfg, kernel="small", max_b=None):
    store = api.GpuStore(rp, codes, d, dtype=dtype)
    B = len(off) - 1
    rr = api.Reranker(store, max_b or B, max(int(off[-1]), 1), q.shape[1])
    out = rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kernel, write_bow=True)
    launches = rr.counters()["kernel_launches"]
    rr.close()
    store.close()
    return out, launches


@pytest.mark.parametrize("B", [1, 2, 4])
def test_c1_shape_bitexact(oracle, cuda_ok, B):
    # configs[0]: <=32 tokens per doc, d=32 fp16, 32 query tokens, top-1000 -> top-10
    rp, codes, q, ids, cls, off, src = _case(20000, 32, 32, B, 1000, seed=3 + B)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    got, launches = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg)
    assert launches == 1  # the whole batch in one launch
    _exact(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, got)
    assert np.array_equal(got[0][:, 0], src.astype(np.uint32))


@pytest.mark.parametrize("d", [8, 16, 32, 48, 64, 96, 128])
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_dims_dtypes_bitexact(oracle, cuda_ok, d, dtype):
    rp, codes, q, ids, cls, off, _ = _case(3000, d, 40, 2, 300, nq=13, dtype=dtype, seed=d)
    cfg = api.PipelineConfig(rerank_count=300, final_k=32, alpha=0.7)
    got, _ = _run(rp, codes, d, dtype, q, ids, cls, off, cfg)
    _exact(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, got)


@pytest.mark.parametrize("partial", [False, True])
def test_partial_alpha_ragged_empty(oracle, cuda_ok, partial):
    rp, codes, q, ids, cls, off, _ = _case(5000, 32, 63, 7, 500, seed=41, ragged=True)
    R = 120 if partial else 500
    for k in (1, 10, 32):
        cfg = api.PipelineConfig(rerank_count=R, final_k=k, alpha=1.3, partial_rerank_enabled=partial)
        got, _ = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg)
        _exact(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, got)


def test_longest_lists_and_max_batch(oracle, cuda_ok):
    # 16 queries x 128 and 1 query x 2048 (the small path's bounds)
    for B, K in ((16, 128), (1, 2048), (3, 700)):
        rp, codes, q, ids, cls, off, _ = _case(8000, 32, 63, B, K, seed=B * 7 + K)
        cfg = api.PipelineConfig(rerank_count=K, final_k=10)
        got, launches = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg)
        assert launches == 1
        _exact(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, got)


def test_last_cta_merge_select_and_fallback(oracle, cuda_ok):
    # final_k = 32 over 2048-candidate lists: 4 queries get 74 CTAs each (the
    # last CTA's threshold select over 74 lists), 16 queries get 18 CTAs each
    # (fewer lists than k: all 576 keys survive, more than the select's 512
    # slots, so the two-level k-way merge runs instead)
    for B, K in ((4, 2048), (16, 2048)):
        rp, codes, q, ids, cls, off, _ = _case(40000, 32, 32, B, K, seed=B * 13 + 5)
        cfg = api.PipelineConfig(rerank_count=K, final_k=32)
        got, launches = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg)
        assert launches == 1
        _exact(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, got)


def test_matches_simt_and_tcgen05(oracle, cuda_ok):
    rp, codes, q, ids, cls, off, _ = _case(20000, 32, 32, 2, 1000, seed=77)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    small, _ = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg)
    simt, n_simt = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel="simt")
    assert n_simt == 3
    for a, b in zip(small[:3], simt[:3]):
        assert np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))
    tc, _ = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel="tcgen05")
    assert np.array_equal(tc[2], small[2])
    assert np.abs(tc[1] - small[1]).max() <= 1e-3 * max(1.0, float(np.abs(small[1]).max()))


def test_auto_choice(cuda_ok):
    rp, codes, q, ids, cls, off, _ = _case(4000, 32, 32, 1, 1000, seed=5)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    _, n = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel="auto")
    assert n == 3  # opt-in only: AUTO keeps the tcgen05 chain (one arithmetic for every batch size)
    _, n = _run(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel="small")
    assert n == 1
    cfg = api.PipelineConfig(rerank_count=1000, final_k=33)  # k beyond the fused lists
    rp, codes, q, ids, cls, off, _ = _case(4000, 32, 32, 1, 1000, seed=7)
    with pytest.raises(api.InvalidConfigError):
        _run(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel="small")


def test_errors_and_recovery(cuda_ok):
    rp, codes, q, ids, cls, off, _ = _case(1000, 32, 20, 2, 100, seed=61)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 2, 200, 32)
    cfg = api.PipelineConfig(rerank_count=100, final_k=10)
    good = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="small")
    for rep in range(3):  # eager, graph capture, graph replay: errors surface every time
        bad = ids.copy(); bad[5] = 1000
        with pytest.raises(api.DataIntegrityError):
            rr.rerank_arrays(q, bad, cls, off, cfg, kernel="small")
        dup = ids.copy(); dup[107] = dup[199]
        with pytest.raises(api.InvalidInputError):
            rr.rerank_arrays(q, dup, cls, off, cfg, kernel="small")
        ff = ids.copy(); ff[3] = 0xFFFFFFFF; ff[4] = 0xFFFFFFFF  # the hash's empty code, twice
        with pytest.raises((api.InvalidInputError, api.DataIntegrityError)):
            rr.rerank_arrays(q, ff, cls, off, cfg, kernel="small")
        nan = cls.copy(); nan[2] = np.nan
        with pytest.raises(api.InvalidInputError):
            rr.rerank_arrays(q, ids, nan, off, cfg, kernel="small")
        qn = q.copy(); qn[1, 3, 4] = np.inf
        with pytest.raises(api.InvalidInputError):
            rr.rerank_arrays(qn, ids, cls, off, cfg, kernel="small")
        again = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="small")
        for a, b in zip(good[:3], again[:3]):
            assert np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32)), rep
    rr.close(); store.close()


def test_graph_replay_tracks_list_lengths(oracle, cuda_ok):
    """Synchronous calls of one (B, C) shape replay a captured graph; the grid
    (CTAs per query) depends on the longest list, so a replay with a different
    length distribution must still be exact."""
    rp, codes = synth.make_table(6000, 32, 1, 32, seed=23)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 2, 1200, 32)
    cfg = api.PipelineConfig(rerank_count=1200, final_k=10)
    rng = np.random.default_rng(24)
    q, _ = synth.make_queries(rp, codes, 32, 2, seed=25)
    for offs in ([0, 600, 1200], [0, 600, 1200], [0, 600, 1200], [0, 1100, 1200], [0, 100, 1200], [0, 600, 1200]):
        ids = rng.permutation(6000)[:1200].astype(np.uint32)
        cls = rng.random(1200, dtype=np.float32)
        off = np.asarray(offs, np.uint64)
        got = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="small", write_bow=True)
        _exact(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, got)
    rr.close(); store.close()


def test_bad_device_offsets(cuda_ok):
    import torch
    rp, codes, q, ids, cls, off, _ = _case(2000, 32, 20, 2, 100, seed=71)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 2, 200, 32, max_list=100)
    dq = torch.from_numpy(q).cuda()
    did = torch.from_numpy(ids.view(np.int32)).cuda()
    dcl = torch.from_numpy(cls).cuda()
    out = torch.zeros(2 * 2 * 10 + 2, dtype=torch.int32, device="cuda")
    base = out.data_ptr()
    flags = L.ESPN_RERANK_DEVICE_IO | L.ESPN_RERANK_DEVICE_OFFSETS
    for offs, want in (([0, 100, 200], 0), ([0, 150, 100], L.ESPN_E_INVALID_INPUT), ([5, 100, 200], L.ESPN_E_INVALID_INPUT),
                       ([0, 100, 900], L.ESPN_E_INVALID_INPUT), ([0, 100, 200], 0)):
        doff = torch.tensor(offs, dtype=torch.int64, device="cuda")
        a = L.RerankArgs(n_queries=2, n_query_tokens=32, query_tokens=dq.data_ptr(), cand_ids=did.data_ptr(),
                         cand_cls=dcl.data_ptr(), cand_offsets=doff.data_ptr(), rerank_count=100, final_k=10,
                         alpha=1.0, flags=flags, kernel=L.ESPN_KERNEL_SMALL)
        o = L.RerankOut(ids=base, scores=base + 4 * 20, counts=base + 8 * 20)
        st = L.lib().espn_gpu_rerank(store.handle, rr.handle, C.byref(a), C.byref(o), None)
        assert st == want, (offs, st)
        if want == 0:
            assert list(out[40:].cpu().numpy()) == [10, 10]
    rr.close(); store.close()
