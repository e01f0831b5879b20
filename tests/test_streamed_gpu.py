"""Streamed tables (ESPN_TABLE_STREAMED + espn_gpu_table_load_rows) and the
streamed open_store: only the resident docs ever occupy HBM, the host tier is
tiled straight into pinned memory, the .espn file is read chunk by chunk.
The overflow tier really overflows: a table larger than the free HBM opens
and re-ranks like the oracle ("let the overflow tier overflow")."""
import numpy as np
import pytest

from helpers import assert_topk_equivalent, oracle_full_scores

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import api, synth  # noqa: E402


def _small(tmp_path, seed=3, n=4000):
    rp, codes = synth.make_table(n, 32, 1, 63, seed=seed)
    base = tmp_path / "s"
    rows = api.decode(codes, "f16")
    api.build_store(base, rp, rows, 32, d_cls=16, alignment=512)
    return rp, codes, base


@pytest.mark.parametrize("tiered", [False, True])
def test_streamed_open_store_equals_regular(tmp_path, cuda_ok, tiered):
    rp, codes, base = _small(tmp_path)
    n = rp.shape[0] - 1
    resident = (np.random.default_rng(1).random(n) < 0.3).astype(np.uint8) if tiered else None
    ref = api.GpuStore(rp, codes, 32, d_cls=16, alignment=512)
    st = api.GpuStore.open_store(base, resident=resident, chunk_bytes=1 << 16)  # many chunks
    assert st.n_docs == n and st.n_tokens == int(rp[-1])
    if tiered:
        assert st.tiered and st.resident_docs == int(resident.sum()) and st.host_bytes > 0
    q, src = synth.make_queries(rp, codes, 32, 4, seed=5)
    ids, cls, off = synth.make_candidates(n, 4, 700, src=src, seed=6)
    cfg = api.PipelineConfig(rerank_count=500, final_k=10, partial_rerank_enabled=True)
    a = api.Reranker(ref, 4, int(off[-1]), 32).rerank_arrays(q, ids, cls, off, cfg)
    b = api.Reranker(st, 4, int(off[-1]), 32).rerank_arrays(q, ids, cls, off, cfg)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    req = np.random.default_rng(2).integers(0, n, 300).astype(np.uint32)
    fa, fb = ref.fetch_batch(req), st.fetch_batch(req)
    for x, y in zip(fa.docs, fb.docs):
        assert np.array_equal(x.bow.values, y.bow.values)
    st.close(); ref.close()


def test_streamed_state_errors(cuda_ok):
    rp, codes = synth.make_table(1000, 32, 1, 20, seed=9)
    st = api.GpuStore(rp, None, 32, streamed=True)
    rr = api.Reranker(st, 1, 100, 32)
    q, _ = synth.make_queries(rp, codes, 32, 1, seed=1)
    ids = np.arange(100, dtype=np.uint32)
    cls = np.zeros(100, np.float32)
    with pytest.raises(api.InvalidStateError):  # not loaded yet
        rr.rerank_arrays(q, ids, cls, np.array([0, 100], np.uint64), api.PipelineConfig(rerank_count=100))
    half = int(rp[500])
    with pytest.raises(api.InvalidInputError):  # out of order
        from paper_2312_05417_b200 import _lib as L
        api._check(L.lib().espn_gpu_table_load_rows(st.handle, 500, 10, codes[half * 32:].ctypes.data))
    st.load_rows(0, codes[:half * 32])
    st.load_rows(500, codes[half * 32:])
    out = rr.rerank_arrays(q, ids, cls, np.array([0, 100], np.uint64), api.PipelineConfig(rerank_count=100))
    ref = api.GpuStore(rp, codes, 32)
    out2 = api.Reranker(ref, 1, 100, 32).rerank_arrays(q, ids, cls, np.array([0, 100], np.uint64),
                                                     api.PipelineConfig(rerank_count=100))
    assert np.array_equal(out[0], out2[0]) and np.array_equal(out[1], out2[1])
    rr.close(); st.close(); ref.close()


def test_table_larger_than_free_hbm(oracle, cuda_ok):
    """HBM is filled until 1.5 GB stay free; a 3 GB table (1.5 M docs, d=32)
    opens streamed with 20 % of its docs in HBM (0.6 GB) and the rest in the
    pinned-host tier, and re-ranks like the oracle."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    keep_free = int(1.5e9)
    blocker = torch.empty(max(free - keep_free, 0), dtype=torch.uint8, device="cuda")
    n, d = 1_500_000, 32
    rng = np.random.default_rng(77)
    t = rng.integers(1, 64, n)
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(t)
    table_bytes = int(rp[-1]) * d * 2
    assert table_bytes > torch.cuda.mem_get_info()[0], "the table must exceed the free HBM"
    resident = (rng.random(n) < 0.2).astype(np.uint8)
    B, K = 8, 1000
    cand = [np.sort(rng.choice(n, K, replace=False)).astype(np.uint32) for _ in range(B)]
    want = np.unique(np.concatenate(cand))
    store = api.GpuStore(rp, None, d, resident=resident, streamed=True)
    assert store.hbm_bytes < keep_free
    kept = {}
    chunk = 100_000
    for i in range(0, n, chunk):
        j = min(i + chunk, n)
        tok = int(rp[j] - rp[i])
        x = rng.standard_normal((tok, d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        c = x.astype(np.float16).view(np.uint16)
        c[(c & 0x7C00) == 0] &= 0x8000  # no subnormals
        store.load_rows(i, c.ravel())
        sel = want[(want >= i) & (want < j)]
        for g in sel:
            a, b = int(rp[g] - rp[i]), int(rp[g + 1] - rp[i])
            kept[int(g)] = c[a:b].copy()
    # queries: perturbed rows of a kept candidate; lists sorted by (cls desc, id asc)
    q = np.empty((B, 32, d), np.float32)
    ids_l, cls_l = [], []
    for b in range(B):
        rows = kept[int(cand[b][0])].view(np.float16).astype(np.float32)
        v = rows[rng.integers(0, rows.shape[0], 32)] + 0.1 * rng.standard_normal((32, d)).astype(np.float32)
        q[b] = v / np.linalg.norm(v, axis=1, keepdims=True)
        s = rng.random(K).astype(np.float32)
        o = np.lexsort((cand[b], -s))
        ids_l.append(cand[b][o]); cls_l.append(s[o])
    ids, cls = np.concatenate(ids_l), np.concatenate(cls_l)
    off = (np.arange(B + 1) * K).astype(np.uint64)
    cfg = api.PipelineConfig(rerank_count=K, final_k=10)
    rr = api.Reranker(store, B, B * K, 32, staging_bytes=64 << 20)
    gi, gs, gc, _ = rr.rerank_arrays(q, ids, cls, off, cfg)
    # oracle over the candidates' rows (compact table, ids remapped)
    uniq = np.array(sorted(kept), np.uint32)
    lrp = np.zeros(uniq.size + 1, np.uint64)
    lrp[1:] = np.cumsum([kept[int(u)].shape[0] for u in uniq])
    lcodes = np.concatenate([kept[int(u)].ravel() for u in uniq])
    ot = oracle.OracleTable(lrp, lcodes, d)
    rid = np.searchsorted(uniq, ids).astype(np.uint32)
    st, obow = oracle.maxsim_batch(ot, q, rid, off)
    st2, oi, os_, on = oracle.rerank_batch(ot, q, rid, cls, off, K, 10)
    assert st == 0 and st2 == 0
    for b in range(B):
        a0, a1 = int(off[b]), int(off[b + 1])
        full = oracle_full_scores(obow[a0:a1], cls[a0:a1], 1.0, K, False)
        n_b = int(on[b])
        assert int(gc[b]) == n_b
        assert_topk_equivalent(np.searchsorted(uniq, gi[b, :n_b]).astype(np.uint32), gs[b, :n_b], oi[b, :n_b],
                               os_[b, :n_b], rid[a0:a1], full, ctx=f"query {b}")
    rr.close(); store.close()
    del blocker
    torch.cuda.empty_cache()
