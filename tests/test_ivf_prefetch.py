"""IVF cursor (ivf.hpp:10-86) and the ANN-overlapped
prefetch hints (pipeline.hpp:56-97).

CPU: the SPEC's IVF examples and properties against brute-force oracles,
ESPNIVF1 persistence.  GPU: espn_gpu_prefetch_hints + PREFETCHED re-rank is
bit-identical to the unprefetched call, the device's hit counts equal the
host's set arithmetic exactly, and the hit-rate sweep rises to 1.0 at step 100.
"""
import numpy as np
import pytest

from paper_2312_05417_b200 import api, ivf, pipeline


def brute_topk(vecs, q, k):
    s = (vecs.astype(np.float64) @ q.astype(np.float64)).astype(np.float32)
    ids = np.arange(vecs.shape[0], dtype=np.uint32)
    o = np.lexsort((ids, -s))[:k]
    return ids[o]


@pytest.fixture(scope="module")
def corpus():
    cls = pipeline.make_cls_corpus(6000, 32, n_blobs=24, seed=3)
    return cls, ivf.train_ivf(cls, 48, 15, seed=1)


def test_train_examples():
    sq = np.array([[1, 1], [1, -1], [-1, 1], [-1, -1]], np.float32) * 5
    ix = ivf.train_ivf(sq, 4, 10, seed=0)
    assert sorted(np.diff(ix.list_off).tolist()) == [1, 1, 1, 1]
    x = np.random.default_rng(0).standard_normal((50, 8)).astype(np.float32)
    one = ivf.train_ivf(x, 1, 5, seed=0)
    assert one.size() == 50 and np.allclose(one.centroids[0], x.mean(0), atol=1e-5)
    with pytest.raises(api.InvalidInputError):
        ivf.train_ivf(x[:3], 4, 5)


def test_every_doc_in_exactly_one_nearest_list(corpus):
    cls, ix = corpus
    assert ix.size() == cls.shape[0]
    assert np.array_equal(np.sort(ix.ids), np.arange(cls.shape[0], dtype=np.uint32))
    d2 = ((cls[:, None, :] - ix.centroids[None]) ** 2).sum(-1)
    lists = np.repeat(np.arange(ix.nlist()), np.diff(ix.list_off).astype(np.int64))
    owner = np.empty(cls.shape[0], np.int64)
    owner[ix.ids] = lists
    best = d2.min(1)
    assert np.all(d2[np.arange(cls.shape[0]), owner] <= best + 1e-4)
    assert np.array_equal(ix.vectors, cls[ix.ids])


def test_blob_recovery():
    # vectors from 32 blobs, nlist=32 -> >= 90% co-listed with their blob majority
    rng = np.random.default_rng(4)
    centers = rng.standard_normal((32, 16)).astype(np.float32) * 4
    blob = rng.integers(0, 32, 1000)
    x = centers[blob] + 0.3 * rng.standard_normal((1000, 16)).astype(np.float32)
    ix = ivf.train_ivf(x, 32, 30, seed=2)
    lists = np.repeat(np.arange(32), np.diff(ix.list_off).astype(np.int64))
    owner = np.empty(1000, np.int64)
    owner[ix.ids] = lists
    agree = 0
    for bl in range(32):
        m = owner[blob == bl]
        if m.size:
            agree += np.bincount(m).max()
    assert agree / 1000 >= 0.9


def test_plan_and_exhaustive_equivalence(corpus):
    cls, ix = corpus
    rng = np.random.default_rng(5)
    for _ in range(5):
        q = cls[rng.integers(cls.shape[0])]
        cur = ivf.begin_search(ix, q, ix.nlist(), 200)
        cs = ix.centroids @ q
        assert np.array_equal(cur.plan, np.lexsort((np.arange(ix.nlist()), -cs)))
        assert cur.snapshot(10).entries == []
        cur.advance(0)
        cur.advance(ix.nlist())
        fin = cur.finish(200)
        ids = np.array([c.doc_id for c in fin.entries], np.uint32)
        assert np.array_equal(ids, brute_topk(cls, q, 200))  # exhaustive equivalence, ties by doc_id
        assert cur.snapshot(200).entries == fin.entries
        sc = [c.cls_score for c in fin.entries]
        assert all(a >= b for a, b in zip(sc, sc[1:]))


def test_acceptance2_exhaustive_top100():
    # nprobe = nlist on a 10k-doc seeded corpus -> top-100 equal the exhaustive oracle, 50 queries
    cls = pipeline.make_cls_corpus(10000, 128, n_blobs=32, seed=23)
    ix = ivf.train_ivf(cls, 64, 10, seed=24)
    qs = pipeline.query_cls_for(cls, np.random.default_rng(25).integers(0, 10000, 50), seed=26)
    for q in qs:
        cur = ivf.begin_search(ix, q, ix.nlist(), 100)
        cur.advance(ix.nlist())
        got = np.array([c.doc_id for c in cur.finish(100).entries], np.uint32)
        assert np.array_equal(got, brute_topk(cls, q, 100))


def test_acceptance6_hit_rate_trend_host():
    # SPEC.md:463 (scaled-down Fig. 5), host set arithmetic of the reference's hit rate
    # |snapshot(R) n top-R(final)| / R: 100k docs, 32 blobs, eta = 25% of nlist
    cls = pipeline.make_cls_corpus(100000, 128, n_blobs=32, spread=0.8, seed=27)
    ix = ivf.train_ivf(cls, 256, 8, seed=28)
    qs = pipeline.query_cls_for(cls, np.random.default_rng(29).integers(0, 100000, 40), seed=30)
    eta, R = 64, 1000
    hr = {}
    for st in (5, 30, 100):
        cfg = api.PipelineConfig(nprobe=eta, prefetch_step_pct=st, rerank_count=R)
        rates = []
        for q in qs:
            cur = ivf.begin_search(ix, q, eta, R)
            cur.advance(cfg.delta())
            snap = cur.snapshot_arrays(R)[0]
            cur.advance(eta - cfg.delta())
            need = cur.finish_arrays(R)[0]
            rates.append(np.isin(need, snap).mean())
        hr[st] = np.array(rates)
    assert np.all(hr[100] == 1.0)
    assert hr[30].mean() >= hr[5].mean()
    assert hr[30].mean() >= 0.8, hr[30].mean()


def test_two_step_advance_equals_one_step(corpus):
    cls, ix = corpus
    q = cls[11]
    a = ivf.begin_search(ix, q, 20, 100)
    a.advance(6)
    a.advance(14)
    b = ivf.begin_search(ix, q, 20, 100)
    b.advance(20)
    assert a.finish(100).entries == b.finish(100).entries
    with pytest.raises(api.InvalidInputError):
        b.advance(1)
    c = ivf.begin_search(ix, q, 20, 100)
    c.advance(3)
    with pytest.raises(api.InvalidStateError):
        c.finish(10)
    with pytest.raises(api.InvalidInputError):
        ivf.begin_search(ix, q, ix.nlist() + 1, 10)


def test_recall_nondecreasing_in_nprobe(corpus):
    cls, ix = corpus
    rng = np.random.default_rng(6)
    qs = pipeline.query_cls_for(cls, rng.integers(0, cls.shape[0], 40))
    prev = -1.0
    for frac in (0.02, 0.1, 0.25, 1.0):
        npb = max(1, int(ix.nlist() * frac))
        rec = []
        for q in qs:
            cur = ivf.begin_search(ix, q, npb, 100)
            cur.advance(npb)
            got = [c.doc_id for c in cur.finish(100).entries]
            rec.append(np.isin(brute_topk(cls, q, 100), got).mean())
        assert np.mean(rec) >= prev - 1e-12
        prev = np.mean(rec)
    assert prev > 0.98


def test_save_load_round_trip(tmp_path, corpus):
    _, ix = corpus
    ivf.save_ivf(ix, tmp_path / "i.ivf")
    jx = ivf.load_ivf(tmp_path / "i.ivf")
    for f in ("centroids", "list_off", "ids", "vectors"):
        assert np.array_equal(getattr(ix, f), getattr(jx, f))
    raw = (tmp_path / "i.ivf").read_bytes()
    (tmp_path / "bad.ivf").write_bytes(b"X" + raw[1:])
    with pytest.raises(api.FormatError):
        ivf.load_ivf(tmp_path / "bad.ivf")
    (tmp_path / "bad.ivf").write_bytes(raw[:-3])
    with pytest.raises(api.FormatError):
        ivf.load_ivf(tmp_path / "bad.ivf")
    with pytest.raises(api.IoError):
        ivf.load_ivf(tmp_path / "missing.ivf")


# ------------------------------------------------------------------ GPU: prefetch hints
def _tiered_setup(resident_frac, n_docs=20000, d=32, B=32, seed=21, staging=64 << 20):
    from paper_2312_05417_b200 import synth
    rp, codes = synth.make_table(n_docs, d, 1, 63, seed=seed)
    q, src = synth.make_queries(rp, codes, d, B, nq=32, seed=seed + 1)
    cls = pipeline.make_cls_corpus(n_docs, 128, n_blobs=64, seed=seed + 2)
    qc = pipeline.query_cls_for(cls, src, seed=seed + 3)
    ix = ivf.train_ivf(cls, 128, 10, seed=seed + 4)
    rng = np.random.default_rng(seed + 5)
    resident = (rng.random(n_docs) < resident_frac).astype(np.uint8)
    store = api.GpuStore(rp, codes, d, "f16", resident=resident)
    rr = api.Reranker(store, B, B * 1000, 32, staging_bytes=staging)
    global row_ptr_g
    row_ptr_g = rp
    return store, rr, q, qc, ix, resident


@pytest.mark.gpu
@pytest.mark.parametrize("resident_frac", [0.0, 0.3])
def test_prefetch_hints_bit_identical_and_counted(cuda_ok, resident_frac):
    store, rr, q, qc, ix, resident = _tiered_setup(resident_frac)
    base = dict(nprobe=64, rerank_count=200, final_k=10, candidate_k=1000, partial_rerank_enabled=True)
    off = pipeline.run_batch(q, qc, ix, rr, api.PipelineConfig(prefetch_enabled=False, **base))
    for step in (5.0, 30.0, 100.0):
        on = pipeline.run_batch(q, qc, ix, rr, api.PipelineConfig(prefetch_step_pct=step, **base), keep_lists=True)
        assert np.array_equal(on.ids, off.ids) and np.array_equal(on.counts, off.counts)
        assert np.array_equal(on.scores.view(np.uint32), off.scores.view(np.uint32))
        # device hits == host set arithmetic: needed host-tier rows hinted by ANY query of the batch
        union = np.unique(np.concatenate(on.hints))
        for b, f in enumerate(on.fetch):
            need = on.finals[b][0][:on.needed[b]]
            host_tier = need[resident[need] == 0]
            exp_hits = int(np.isin(host_tier, union).sum())
            assert f["needed"] == on.needed[b]
            assert f["resident"] == need.size - host_tier.size
            assert f["prefetched"] == exp_hits, (step, b)
            assert f["missed"] == host_tier.size - exp_hits
            # critical-path accounting: exactly the missed rows' bytes
            missed = host_tier[~np.isin(host_tier, union)]
            assert f["critical_bytes"] == int(sum(int(row_ptr_g[m + 1] - row_ptr_g[m]) for m in missed)) * 64
        if step == 100.0:
            assert np.all(on.hit_rate() == 1.0)
            assert all(f["missed"] == 0 and f["critical_bytes"] == 0 for f in on.fetch)
    rr.close()
    store.close()


@pytest.mark.gpu
def test_hit_rate_sweep_rises_to_one(cuda_ok):
    store, rr, q, qc, ix, _ = _tiered_setup(0.0)
    base = api.PipelineConfig(nprobe=64, rerank_count=200, final_k=10, candidate_k=1000,
                              partial_rerank_enabled=True)
    pts = pipeline.measure_hit_rate(q, qc, ix, rr, base, [5, 30, 100])
    hr = [p["mean_hit_rate"] for p in pts]
    assert hr[0] <= hr[1] <= hr[2] == 1.0, hr
    assert pts[2]["critical_bytes"] == 0
    # with every doc in the host tier the device's in-HBM rate is the batch-level hit rate
    assert all(p["device_in_hbm_rate"] >= p["mean_hit_rate"] - 1e-12 for p in pts)
    rr.close()
    store.close()


@pytest.mark.gpu
def test_hint_budget_overflow_falls_back_to_critical_path(cuda_ok):
    # a tiny staging buffer: hints stop at half of it, the rest are misses copied on the critical path
    store, rr, q, qc, ix, _ = _tiered_setup(0.0, B=8, staging=4 << 20)
    base = dict(nprobe=64, rerank_count=200, final_k=10, candidate_k=1000, partial_rerank_enabled=True)
    off = pipeline.run_batch(q[:8], qc[:8], ix, rr, api.PipelineConfig(prefetch_enabled=False, **base))
    on = pipeline.run_batch(q[:8], qc[:8], ix, rr, api.PipelineConfig(prefetch_step_pct=100.0, **base))
    assert np.array_equal(on.ids, off.ids)
    assert np.array_equal(on.scores.view(np.uint32), off.scores.view(np.uint32))
    assert sum(f["prefetch_bytes"] for f in on.fetch) <= (4 << 20) // 2
    assert sum(f["missed"] for f in on.fetch) > 0
    rr.close()
    store.close()


@pytest.mark.gpu
def test_prefetch_hints_state_errors_and_untiered_noop(cuda_ok):
    store, rr, q, qc, ix, _ = _tiered_setup(0.0, B=4)
    hints = np.arange(40, dtype=np.uint32)
    off = np.array([0, 10, 20, 30, 40], np.uint64)
    with pytest.raises(api.InvalidInputError):
        rr.prefetch_hints(hints, np.array([0, 10, 5, 30, 40], np.uint64))
    rr.prefetch_hints(hints, off)  # host ids
    rr.prefetch_hints(hints, off)
    with pytest.raises(api.InvalidStateError):  # both staging slots hold pending prefetches
        rr.prefetch_hints(hints, off)
    rr.close()
    store.close()
    # an all-HBM store: hints are a no-op and PREFETCHED re-ranks like a plain call
    from paper_2312_05417_b200 import synth
    rp, codes = synth.make_table(3000, 32, 1, 63, seed=5)
    qq, src = synth.make_queries(rp, codes, 32, 4, nq=32, seed=6)
    ids, cls, coff = synth.make_candidates(3000, 4, 300, src=src, seed=7)
    hbm = api.GpuStore(rp, codes, 32, "f16")
    r2 = api.Reranker(hbm, 4, 1200, 32)
    r2.prefetch_hints(ids, coff)
    cfg = api.PipelineConfig(rerank_count=300, final_k=10)
    a = [np.copy(x) for x in r2.rerank_arrays(qq, ids, cls, coff, cfg, prefetched=True)[:3]]
    b = [np.copy(x) for x in r2.rerank_arrays(qq, ids, cls, coff, cfg)[:3]]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    r2.close()
    hbm.close()


@pytest.mark.gpu
def test_prefetch_hints_sharded_ignore_foreign_ids(cuda_ok):
    """Two doc-id shards (owner = id % 2) of a host-tier table on one GPU: each
    gets the FULL hint lists, stages only its own docs, and the merged
    per-shard rankings equal the unsharded ranking."""
    from paper_2312_05417_b200 import synth
    from paper_2312_05417_b200.sharding import merge_ranked, split_by_owner
    G, n, d, B, K, R, k = 2, 6000, 32, 6, 500, 200, 10
    rp, codes = synth.make_table(n, d, 1, 63, seed=8)
    q, src = synth.make_queries(rp, codes, d, B, nq=32, seed=9)
    ids, cls, off = synth.make_candidates(n, B, K, src=src, seed=10)
    hints = np.concatenate([ids[int(off[b]):int(off[b]) + 150] for b in range(B)])  # a snapshot per query
    hoff = np.arange(B + 1, dtype=np.uint64) * 150
    cfg = api.PipelineConfig(rerank_count=R, final_k=k, partial_rerank_enabled=True)
    full = api.GpuStore(rp, codes, d, "f16")
    rf = api.Reranker(full, B, B * K, 32)
    ref_ids, ref_sc, ref_n, _ = [np.copy(x) if x is not None else None for x in rf.rerank_arrays(q, ids, cls, off, cfg)]
    rf.close()
    full.close()
    lens = np.diff(rp.astype(np.int64))
    per = []
    for s in range(G):
        loc = np.arange(s, n, G)
        lrp = np.zeros(loc.size + 1, np.uint64)
        lrp[1:] = np.cumsum(lens[loc])
        lcodes = np.concatenate([codes[int(rp[i]) * d:int(rp[i + 1]) * d] for i in loc])
        st = api.GpuStore(lrp, lcodes, d, "f16", shard_count=G, shard_index=s,
                          resident=np.zeros(loc.size, np.uint8))
        rr = api.Reranker(st, B, B * K, 32)
        s_ids, s_cls, s_off, s_need = split_by_owner(ids, cls, off, R, G, s)
        rr.prefetch_hints(hints, hoff)
        gi, gs, gc, _ = rr.rerank_arrays(q, s_ids, s_cls, s_off, cfg, needed_counts=s_need, prefetched=True,
                                         fetch_stats=True)
        hs = set(int(h) for h in hints if h % G == s)
        for b, f in enumerate(rr.last_fetch_stats):
            need = s_ids[int(s_off[b]):int(s_off[b]) + int(s_need[b])]
            assert f["needed"] == need.size
            assert f["prefetched"] == sum(int(x) in hs for x in need)
            assert f["missed"] == need.size - f["prefetched"]
        per.append((np.copy(gi), np.copy(gs), np.copy(gc)))
        rr.close()
        st.close()
    for b in range(B):
        mi, ms = merge_ranked([p[0][b] for p in per], [p[1][b] for p in per], [p[2][b] for p in per], k)
        assert np.array_equal(mi, ref_ids[b, :int(ref_n[b])])
        assert np.array_equal(ms.view(np.uint32), ref_sc[b, :int(ref_n[b])].view(np.uint32))


@pytest.mark.gpu
def test_reference_named_pipeline_entry_points(cuda_ok):
    """run_query / run_batch / measure_hit_rate with the reference's carrier
    types (pipeline.hpp:56-97): batch == per-query calls, prefetch on == off,
    QueryStats consistent, step 100 -> hit rate 1.0."""
    store, rr, q, qc, ix, _ = _tiered_setup(0.2, B=6)
    rr.close()
    queries = [api.QueryEmbedding(query_id=100 + b, cls=qc[b], rows=32, cols=32, tokens=q[b].ravel())
               for b in range(6)]
    base = dict(nprobe=64, rerank_count=200, final_k=10, candidate_k=1000, partial_rerank_enabled=True)
    on = pipeline.run_batch_queries(queries, ix, store, api.PipelineConfig(prefetch_step_pct=30.0, **base))
    off = pipeline.run_batch_queries(queries, ix, store, api.PipelineConfig(prefetch_enabled=False, **base))
    assert on.rankings == off.rankings
    # QueryStats field for field with the oracle's eo_rerank_query on the same
    # final candidates, prefetched = the same snapshot (pipeline.hpp:45-53);
    # the cursors are deterministic, so the snapshot / final lists are rebuilt here
    import oracle_py
    from paper_2312_05417_b200 import synth
    rp, codes = synth.make_table(20000, 32, 1, 63, seed=21)
    ot = oracle_py.OracleTable(rp, codes, 32)
    cfg_on = api.PipelineConfig(prefetch_step_pct=30.0, **base)
    for b, qe in enumerate(queries):
        rl, st = pipeline.run_query(qe, ix, store, cfg_on)
        assert rl == on.rankings[b]
        cur = ivf.SearchCursor(ix, qc[b], cfg_on.nprobe, cfg_on.effective_candidate_k())
        cur.advance(cfg_on.delta())
        snap = cur.snapshot_arrays(cfg_on.effective_prefetch_top_k())[0]
        cur.advance(cfg_on.nprobe - cfg_on.delta())
        fid, fcls = cur.finish_arrays(cfg_on.effective_candidate_k())
        for got in (st, on.stats[b]):
            ost_ = oracle_py.rerank_query(ot, q[b], fid, fcls, 200, 10, 1.0, True, True, snap)
            assert ost_[0] == 0
            o = ost_[3]
            assert got.query_id == qe.query_id
            for f in ("prefetched_count", "needed_count", "missed_count", "hit_rate", "prefetch_bytes",
                      "critical_fetch_bytes", "critical_blocks_read", "needed_payload_bytes"):
                assert getattr(got, f) == getattr(o, f), (b, f, getattr(got, f), getattr(o, f))
        st_off = off.stats[b]  # no prefetch: every needed doc is fetched on the critical path
        assert st_off.prefetched_count == 0 and st_off.missed_count == st_off.needed_count == 200
    pts = pipeline.measure_hit_rate_queries(queries, ix, store, api.PipelineConfig(**base), [5, 100])
    assert pts[-1].mean_hit_rate == 1.0 and pts[0].mean_hit_rate <= 1.0
    store.close()
