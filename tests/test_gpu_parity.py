"""GPU parity: libespn_gpu.so (tcgen05 and CUDA-core MaxSim, top-k, gather,
merge) against the CPU oracle on the same seeded inputs.  All calls go through
the C-ABI (ctypes).  Tolerances: tests/helpers.py."""
import numpy as np
import pytest

from helpers import RTOL, assert_topk_equivalent, oracle_full_scores, rel_err

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import api, synth  # noqa: E402


def _dt(name):
    import oracle_py
    return oracle_py.F16 if name == "f16" else oracle_py.BF16


def build_case(n_docs, d, t_min, t_max, B, K, nq=32, dtype="f16", seed=1):
    rp, codes = synth.make_table(n_docs, d, t_min, t_max, dtype=dtype, seed=seed)
    q, src = synth.make_queries(rp, codes, d, B, nq=nq, dtype=dtype, seed=seed + 1)
    ids, cls, off = synth.make_candidates(n_docs, B, K, src=src, seed=seed + 2)
    return rp, codes, q, ids, cls, off


def run_gpu(rp, codes, d, dtype, q, ids, cls, off, cfg, kernel, query_precision="auto"):
    store = api.GpuStore(rp, codes, d, dtype=dtype)
    rr = api.Reranker(store, len(off) - 1, max(int(off[-1]), 1), q.shape[1])
    out = rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kernel, write_bow=True, query_precision=query_precision)
    rr.close()
    store.close()
    return out


def check_against_oracle(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, kernel, bitexact_bow=False,
                         query_precision="auto", rtol=RTOL):
    ot = oracle.OracleTable(rp, codes, d, dtype=_dt(dtype))
    # the reference multiplies the fp32 query as given (types.hpp:33-44); only the
    # legacy "rounded" mode is compared against the oracle fed the dtype-rounded query
    qr = oracle.round_to(q, _dt(dtype)) if query_precision == "rounded" else np.ascontiguousarray(q, np.float32)
    gi, gs, gc, gbow = run_gpu(rp, codes, d, dtype, q, ids, cls, off, cfg, kernel, query_precision)
    st, obow = oracle.maxsim_batch(ot, qr, ids, off)
    assert st == 0
    st, oi, os_, on = oracle.rerank_batch(ot, qr, ids, cls, off, cfg.rerank_count, cfg.final_k, cfg.alpha,
                                          cfg.partial_rerank_enabled)
    assert st == 0
    B = len(off) - 1
    for b in range(B):
        a0, a1 = int(off[b]), int(off[b + 1])
        need = min(a1 - a0, cfg.rerank_count)
        g = gbow[a0:a0 + need]
        o = obow[a0:a0 + need]
        if bitexact_bow:
            assert np.array_equal(g.view(np.uint32), o.view(np.uint32)), f"query {b}: SIMT bow not bit-exact"
        elif need:
            e = rel_err(g, o)
            assert e.max() <= rtol, f"query {b}: max rel err {e.max()} at {int(e.argmax())}"
        full = oracle_full_scores(obow[a0:a1], cls[a0:a1], cfg.alpha, need, cfg.partial_rerank_enabled)
        assert int(gc[b]) == int(on[b])
        n = int(on[b])
        assert_topk_equivalent(gi[b, :n], gs[b, :n], oi[b, :n], os_[b, :n], ids[a0:a1], full, ctx=f"query {b}")
    return gbow, obow


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
def test_c1_shape_parity(oracle, cuda_ok, kernel):
    # configs[0]: 100k docs, <=32 tok/doc, d32 fp16, 32 query tok, top-1000 -> top-10 (B=1);
    # a 20k-doc table keeps the oracle fast; the shape law is the same.
    rp, codes, q, ids, cls, off = build_case(20000, 32, 1, 32, B=2, K=1000)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel,
                         bitexact_bow=(kernel == "simt"))


@pytest.mark.parametrize("d", [16, 32, 64, 128])
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_tcgen05_dims_dtypes(oracle, cuda_ok, d, dtype):
    t_max = 100 if d == 128 else 63
    rp, codes, q, ids, cls, off = build_case(3000, d, 1, t_max, B=3, K=257, dtype=dtype, seed=d)
    cfg = api.PipelineConfig(rerank_count=257, final_k=10)
    check_against_oracle(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, "tcgen05")


@pytest.mark.parametrize("d", [32, 64, 128])
def test_simt_bitexact(oracle, cuda_ok, d):
    rp, codes, q, ids, cls, off = build_case(2000, d, 1, 40, B=3, K=200, seed=3 + d)
    cfg = api.PipelineConfig(rerank_count=200, final_k=10)
    check_against_oracle(oracle, rp, codes, d, "f16", q, ids, cls, off, cfg, "simt", bitexact_bow=True)


def test_c2_shape_many_units(oracle, cuda_ok):
    # configs[1] shape law (t ~ U{1..63}, d32, K=R=1000, k=10) at batch 64 on a
    # 200k-doc table: hundreds of work units, stage/quarter straddling docs.
    rp, codes, q, ids, cls, off = build_case(200000, 32, 1, 63, B=64, K=1000, seed=5)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_fp32_query_parity_c2_shape(oracle, cuda_ok, dtype):
    # the reference's query is fp32 (types.hpp:33-44) and the
    # C-ABI takes fp32; the oracle here gets the UNROUNDED query.  Default:
    # bf16 tables carry it as hi + lo (two MMAs per K-step; a bf16-rounded
    # query alone is off by ~3e-3), f16 tables round it to f16 (<= ~5e-4);
    # "split" takes both to <= 1e-4.
    rp, codes, q, ids, cls, off = build_case(200000, 32, 1, 63, B=64, K=1000, dtype=dtype, seed=55)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    gbow, obow = check_against_oracle(oracle, rp, codes, 32, dtype, q, ids, cls, off, cfg, "tcgen05",
                                      rtol=1e-4 if dtype == "bf16" else 1e-3)
    gbow, obow = check_against_oracle(oracle, rp, codes, 32, dtype, q, ids, cls, off, cfg, "tcgen05",
                                      query_precision="split", rtol=1e-4)


@pytest.mark.parametrize("d,dtype", [(16, "bf16"), (64, "bf16"), (128, "bf16"), (128, "f16"), (32, "f16")])
def test_fp32_query_parity_dims(oracle, cuda_ok, d, dtype):
    # every dim against the unrounded-query oracle; forced split for f16 d=128
    t_max = 100 if d == 128 else 63
    rp, codes, q, ids, cls, off = build_case(4000, d, 1, t_max, B=5, K=400, dtype=dtype, seed=60 + d)
    cfg = api.PipelineConfig(rerank_count=400, final_k=10)
    check_against_oracle(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, "tcgen05")
    gbow, obow = check_against_oracle(oracle, rp, codes, d, dtype, q, ids, cls, off, cfg, "tcgen05",
                                      query_precision="split", rtol=1e-4)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_rounded_query_mode_matches_rounded_oracle(oracle, cuda_ok, dtype):
    # ESPN_RERANK_QUERY_ROUNDED: the legacy precision, equal to the oracle fed
    # the dtype-rounded query (SIMT bit-exact)
    rp, codes, q, ids, cls, off = build_case(3000, 32, 1, 63, B=3, K=300, dtype=dtype, seed=71)
    cfg = api.PipelineConfig(rerank_count=300, final_k=10)
    check_against_oracle(oracle, rp, codes, 32, dtype, q, ids, cls, off, cfg, "tcgen05", query_precision="rounded")
    check_against_oracle(oracle, rp, codes, 32, dtype, q, ids, cls, off, cfg, "simt", query_precision="rounded",
                         bitexact_bow=True)


def test_c3_shape_many_units(oracle, cuda_ok):
    # configs[2] shape law (t ~ U{40..100}, d=128 -> the replicated-A, N=256
    # MMA mode with two K-panels) at batch 32 on a 100k-doc table
    rp, codes, q, ids, cls, off = build_case(100000, 128, 40, 100, B=32, K=1000, seed=7)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    check_against_oracle(oracle, rp, codes, 128, "f16", q, ids, cls, off, cfg, "tcgen05")


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
def test_partial_rerank_and_alpha(oracle, cuda_ok, kernel):
    rp, codes, q, ids, cls, off = build_case(5000, 32, 1, 63, B=4, K=1000, seed=9)
    cfg = api.PipelineConfig(rerank_count=64, final_k=10, alpha=0.5, partial_rerank_enabled=True)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel)


def test_partial_with_r_equal_k_matches_full(cuda_ok):
    # R == candidate-list length => partial == full, bit-exact
    rp, codes, q, ids, cls, off = build_case(3000, 32, 1, 63, B=3, K=300, seed=21)
    full = run_gpu(rp, codes, 32, "f16", q, ids, cls, off, api.PipelineConfig(rerank_count=300, final_k=10), "auto")
    part = run_gpu(rp, codes, 32, "f16", q, ids, cls, off,
                   api.PipelineConfig(rerank_count=300, final_k=10, partial_rerank_enabled=True), "auto")
    assert np.array_equal(full[0], part[0]) and np.array_equal(full[1], part[1])


def test_short_lists_small_nq_long_docs(oracle, cuda_ok):
    # ragged: q=5 tokens, candidate lists shorter than final_k and than R,
    # docs up to 400 tokens (fewer docs per work unit)
    rp, codes = synth.make_table(1500, 32, 1, 400, seed=31)
    q, src = synth.make_queries(rp, codes, 32, 5, nq=5, seed=32)
    ids_l, cls_l, offs = [], [], [0]
    rng = np.random.default_rng(33)
    for b, n in enumerate([3, 0, 50, 700, 1]):
        c = rng.permutation(1500)[:n].astype(np.uint32)
        s = np.sort(rng.random(n).astype(np.float32))[::-1].copy()
        o = np.lexsort((c, -s))
        ids_l.append(c[o]); cls_l.append(s[o]); offs.append(offs[-1] + n)
    ids = np.concatenate(ids_l).astype(np.uint32)
    cls = np.concatenate(cls_l).astype(np.float32)
    off = np.asarray(offs, np.uint64)
    cfg = api.PipelineConfig(rerank_count=600, final_k=10)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "simt", bitexact_bow=True)


@pytest.mark.parametrize("d", [32, 128])
def test_max_length_docs(oracle, cuda_ok, d):
    # the longest doc the tcgen05 tiling takes (t = 4096 tokens, one doc per
    # work unit) mixed with short ones, plus a batch of one query (small units)
    rng = np.random.default_rng(51)
    t = rng.integers(1, 64, 600)
    tmax = 6144 if d == 32 else 2048  # UNITMAX x 64 slots (TcCfg, rounded query)
    t[[3, 77, 400]] = [tmax, tmax - 1, tmax // 2 + 1]
    rp = np.zeros(601, np.uint64)
    rp[1:] = np.cumsum(t)
    x = rng.standard_normal((int(rp[-1]), d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    codes = synth.flush_subnormals(api.encode(x.ravel(), "f16"), "f16")
    q, src = synth.make_queries(rp, codes, d, 3, nq=32, seed=52)
    ids, cls, off = synth.make_candidates(600, 3, 300, src=src, seed=53)
    for b in range(3):  # make sure the long docs are candidates
        seg = ids[int(off[b]):int(off[b + 1])]
        for j, doc in enumerate([3, 77, 400]):
            if doc not in seg:
                seg[-1 - j] = doc
    cfg = api.PipelineConfig(rerank_count=300, final_k=10)
    check_against_oracle(oracle, rp, codes, d, "f16", q, ids, cls, off, cfg, "tcgen05")
    q1, ids1, cls1 = q[:1], ids[:300], cls[:300]
    check_against_oracle(oracle, rp, codes, d, "f16", q1, ids1, cls1, off[:2], cfg, "tcgen05")
    # one token more than a unit holds: tcgen05 refuses with the limit, AUTO falls back to the CUDA cores
    t2 = t.copy()
    t2[5] = tmax + 1
    rp2 = np.zeros(601, np.uint64)
    rp2[1:] = np.cumsum(t2)
    codes2 = np.zeros(int(rp2[-1]) * d, np.uint16)
    codes2[:codes.size] = codes
    store = api.GpuStore(rp2, codes2, d)
    rr = api.Reranker(store, 3, int(off[-1]), 32)
    with pytest.raises(api.InvalidConfigError, match=str(tmax)):
        rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05")
    rr.rerank_arrays(q, ids, cls, off, cfg)  # auto -> CUDA cores
    if d == 32:  # the split-query layout has 64-doc units: 4096 slots
        with pytest.raises(api.InvalidConfigError, match="4096"):
            rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", query_precision="split")
    rr.close()
    store.close()


def test_single_token_docs_and_large_k(oracle, cuda_ok):
    rp, codes, q, ids, cls, off = build_case(4000, 32, 1, 1, B=2, K=3000, seed=41)
    cfg = api.PipelineConfig(rerank_count=3000, final_k=100)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")


def test_c5_candidate_count(oracle, cuda_ok):
    # configs[4]: 4000 candidates per query (top-k over > one sort chunk)
    rp, codes, q, ids, cls, off = build_case(50000, 32, 1, 63, B=2, K=4000, seed=51)
    cfg = api.PipelineConfig(rerank_count=4000, final_k=10)
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")


def test_errors(cuda_ok):
    rp, codes, q, ids, cls, off = build_case(1000, 32, 1, 20, B=2, K=100, seed=61)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 2, 200, 32)
    cfg = api.PipelineConfig(rerank_count=100, final_k=10)
    bad = ids.copy(); bad[5] = 1000  # store lacks a candidate -> DataIntegrityError
    with pytest.raises(api.DataIntegrityError):
        rr.rerank_arrays(q, bad, cls, off, cfg)
    dup = ids.copy(); dup[7] = dup[3]  # rank() rejects duplicates (scoring.hpp:16-18)
    with pytest.raises(api.InvalidInputError):
        rr.rerank_arrays(q, dup, cls, off, cfg)
    nan = cls.copy(); nan[2] = np.nan
    with pytest.raises(api.InvalidInputError):
        rr.rerank_arrays(q, ids, nan, off, cfg)
    with pytest.raises(api.InvalidInputError):  # R < final_k without partial
        rr.rerank_arrays(q, ids, cls, off, api.PipelineConfig(rerank_count=5, final_k=10))
    qn = q.copy(); qn[1, 3, 4] = np.inf
    with pytest.raises(api.InvalidInputError):
        rr.rerank_arrays(qn, ids, cls, off, cfg)
    # still usable after errors
    gi, gs, gc, _ = rr.rerank_arrays(q, ids, cls, off, cfg)
    assert list(gc) == [10, 10]
    rr.close(); store.close()


def test_gather_bitexact(oracle, cuda_ok):
    rp, codes = synth.make_table(5000, 32, 1, 63, seed=71)
    store = api.GpuStore(rp, codes, 32)
    ot = oracle.OracleTable(rp, codes, 32)
    rng = np.random.default_rng(72)
    req = rng.integers(0, 5000, size=1000).astype(np.uint32)
    req[10] = req[11]  # duplicates allowed (store.hpp:92)
    res = store.fetch_batch(req)
    st, orp, orows = oracle.gather(ot, req)
    assert st == 0
    assert len(res.docs) == len(req)
    got = np.concatenate([api.encode(doc.bow.values, "f16") for doc in res.docs])
    assert np.array_equal(got, orows)
    assert [doc.bow.rows for doc in res.docs] == list(np.diff(orp).astype(int))
    assert [doc.bow.doc_id for doc in res.docs] == list(req.astype(int))
    with pytest.raises(api.InvalidInputError):
        store.fetch_batch([1, 5000])
    assert store.fetch_batch([]).docs == []
    store.close()


def test_merge_topk(cuda_ok):
    import torch
    from paper_2312_05417_b200 import _lib as L
    rng = np.random.default_rng(81)
    G, B, k = 4, 8, 10
    ids = np.zeros((G, B, k), np.uint32); sc = np.zeros((G, B, k), np.float32); cnt = np.zeros((G, B), np.uint32)
    allc = [[] for _ in range(B)]
    for g in range(G):
        for b in range(B):
            n = int(rng.integers(0, k + 1))
            i = rng.choice(100000, size=n, replace=False).astype(np.uint32) * G + g  # disjoint shards
            s = rng.standard_normal(n).astype(np.float32)
            s[:n // 2] = 0.25  # exact ties broken by id asc
            o = np.lexsort((i, -s))
            ids[g, b, :n] = i[o]; sc[g, b, :n] = s[o]; cnt[g, b] = n
            allc[b] += list(zip(s[o], i[o]))
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(dev)
    oi = torch.zeros((B, k), dtype=torch.int32, device=dev)
    os_ = torch.zeros((B, k), dtype=torch.float32, device=dev)
    oc = torch.zeros(B, dtype=torch.int32, device=dev)
    ti, ts, tc = t(ids), t(sc), t(cnt)
    # separate arrays: list stride B*k for ids/scores, B for counts -> use a packed
    # buffer [ids | scores | counts] per list like the bench's all-gather does
    P = 2 * B * k + B
    packed = np.zeros((G, P), np.uint32)
    packed[:, :B * k] = ids.reshape(G, -1)
    packed[:, B * k:2 * B * k] = sc.reshape(G, -1).view(np.uint32)
    packed[:, 2 * B * k:] = cnt
    tp = t(packed)
    base = tp.data_ptr()
    rc = L.lib().espn_gpu_merge_topk(base, base + 4 * B * k, base + 8 * B * k, G, P, B, k, oi.data_ptr(),
                                     os_.data_ptr(), oc.data_ptr(), None)
    assert rc == 0
    torch.cuda.synchronize()
    oi, os_, oc = oi.cpu().numpy().view(np.uint32), os_.cpu().numpy(), oc.cpu().numpy()
    for b in range(B):
        exp = sorted(allc[b], key=lambda x: (-x[0], x[1]))[:k]
        assert oc[b] == len(exp)
        assert list(oi[b, :oc[b]]) == [int(e[1]) for e in exp]
        assert np.array_equal(os_[b, :oc[b]], np.asarray([e[0] for e in exp], np.float32))


def test_api_mirror_rerank_candidates(oracle, cuda_ok):
    rp, codes, q, ids, cls, off = build_case(3000, 32, 1, 63, B=1, K=200, seed=91)
    store = api.GpuStore(rp, codes, 32)
    qe = api.QueryEmbedding(query_id=3, cls=np.zeros(128, np.float32), rows=32, cols=32, tokens=q[0].ravel())
    cl = api.CandidateList([api.Candidate(int(i), float(c)) for i, c in zip(ids, cls)])
    ranked, stats = api.rerank_candidates(qe, cl, store, api.PipelineConfig(rerank_count=200, final_k=10))
    ot = oracle.OracleTable(rp, codes, 32)
    st, oi, os_, ostats = oracle.rerank_query(ot, np.ascontiguousarray(q[0], np.float32), ids, cls, 200, 10)
    assert st == 0
    assert [e.doc_id for e in ranked.entries] == list(oi)
    assert stats.needed_count == 200 and stats.query_id == 3
    for f in ("prefetched_count", "needed_count", "missed_count", "hit_rate", "prefetch_bytes",
              "critical_fetch_bytes", "critical_blocks_read", "needed_payload_bytes"):
        assert getattr(stats, f) == getattr(ostats, f), f"QueryStats.{f}: {getattr(stats, f)} vs {getattr(ostats, f)}"
    store.close()


def test_synth_table_on_device(cuda_ok):
    import torch
    from paper_2312_05417_b200 import _lib as L
    n, d, G, g = 10000, 32, 3, 1
    rp = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    assert L.lib().espn_gpu_synth_table(n, d, 0, 1, 63, 42, G, g, rp.data_ptr(), None, None) == 0
    t = torch.diff(rp).cpu().numpy()
    assert t.min() >= 1 and t.max() <= 63 and abs(t.mean() - 32) < 1.5
    gids = np.arange(n) * G + g  # shard g of 3: keyed by global id
    assert np.array_equal(t, synth.device_lengths(gids, 1, 63, 42))
    rows = torch.zeros(int(rp[-1]) * d, dtype=torch.int16, device="cuda")
    assert L.lib().espn_gpu_synth_table(n, d, 0, 1, 63, 42, G, g, rp.data_ptr(), rows.data_ptr(), None) == 0
    host = synth.device_rows(int(gids[7]), int(t[7]), d, 42)
    a = int(rp[7])
    # the generator writes the HBM tile layout; untile doc 7 on the host
    doc7 = rows[a * d:(a + int(t[7])) * d].cpu().numpy().view(np.uint16)
    doc7 = synth.untile_rows(np.array([0, int(t[7])]), doc7, d)
    dev7 = doc7.view(np.float16).astype(np.float32).reshape(-1, d)
    assert np.abs(dev7 - host).max() < 2e-3
    v = rows.cpu().numpy().view(np.float16).astype(np.float32).reshape(-1, d)
    nrm = np.linalg.norm(v, axis=1)
    assert np.all(np.isfinite(v)) and np.abs(nrm - 1).max() < 5e-3
    assert not np.any((rows.cpu().numpy().view(np.uint16) & 0x7C00) == 0) or True
    codes = rows.cpu().numpy().view(np.uint16)
    sub = ((codes & 0x7C00) == 0) & ((codes & 0x3FF) != 0)
    assert not sub.any(), "synthetic table must not contain fp16 subnormals"


# ---- tiered store + prefetcher (SURVEY.md §8 a9, configs[3]) -----------------
def _tiered_case(seed=101):
    rp, codes, q, ids, cls, off = build_case(6000, 32, 1, 63, B=8, K=600, seed=seed)
    rng = np.random.default_rng(seed)
    resident = (rng.random(6000) < 0.2).astype(np.uint8)  # 1/5 in HBM, 4/5 in pinned host
    return rp, codes, q, ids, cls, off, resident


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
def test_tiered_store_matches_resident_and_oracle(oracle, cuda_ok, kernel):
    rp, codes, q, ids, cls, off, resident = _tiered_case()
    cfg = api.PipelineConfig(rerank_count=64, final_k=10, alpha=0.5, partial_rerank_enabled=True)
    full = run_gpu(rp, codes, 32, "f16", q, ids, cls, off, cfg, kernel)
    store = api.GpuStore(rp, codes, 32, resident=resident)
    assert store.tiered and store.resident_docs == int(resident.sum()) and store.host_bytes > 0
    rr = api.Reranker(store, len(off) - 1, int(off[-1]), 32)
    got = rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kernel, write_bow=True, fetch_stats=True)
    # identical arithmetic on identical rows: bit-identical scores and order
    for g, f in zip(got[:3], full[:3]):
        assert np.array_equal(g, f)
    need = np.minimum(np.diff(off), 64)
    for b, fs in enumerate(rr.last_fetch_stats):  # no prefetch: host-tier rows are critical-path misses
        assert fs["needed"] == need[b] and fs["prefetched"] == 0
        a0 = int(off[b])
        res = int(resident[ids[a0:a0 + need[b]]].sum())
        assert fs["resident"] == res and fs["missed"] == need[b] - res
        t = (rp[ids[a0:a0 + need[b]] + 1] - rp[ids[a0:a0 + need[b]]])
        assert fs["critical_bytes"] == int((t * (1 - resident[ids[a0:a0 + need[b]]])).sum()) * 64
    rr.close(); store.close()


def test_prefetch_on_off_identical_and_hit_rate(cuda_ok):
    # prefetching only moves I/O off the critical path
    import torch
    rp, codes, q, ids, cls, off, resident = _tiered_case(seed=202)
    cfg = api.PipelineConfig(rerank_count=64, final_k=10, partial_rerank_enabled=True)
    store = api.GpuStore(rp, codes, 32, resident=resident)
    B, C = len(off) - 1, int(off[-1])
    rr = api.Reranker(store, B, C, 32)
    dev = torch.device("cuda")
    dq, di, dc = (torch.from_numpy(q).to(dev), torch.from_numpy(ids.view(np.int32)).to(dev),
                  torch.from_numpy(cls).to(dev))
    side = torch.cuda.Stream()
    off_ref = rr.rerank_arrays(dq, di, dc, off, cfg, device_io=True, fetch_stats=True)
    ref = [x.cpu().numpy() for x in off_ref[:3]]
    ref_stats = rr.last_fetch_stats
    rr.prefetch(dq, di, dc, off, cfg, stream=side.cuda_stream)
    got = rr.rerank_arrays(dq, di, dc, off, cfg, device_io=True, prefetched=True, fetch_stats=True)
    for g, r in zip(got[:3], ref):
        assert np.array_equal(g.cpu().numpy(), r)
    for fs, rs in zip(rr.last_fetch_stats, ref_stats):
        assert fs["missed"] == 0 and fs["critical_bytes"] == 0
        assert fs["prefetched"] == rs["missed"] and fs["prefetch_bytes"] == rs["critical_bytes"]
        assert fs["resident"] + fs["prefetched"] == fs["needed"]  # hit rate 1.0
    # the api mirror's QueryStats carry the same accounting
    qs = [api.QueryEmbedding(query_id=b, cls=np.zeros(128, np.float32), rows=32, cols=32, tokens=q[b].ravel())
          for b in range(B)]
    cl = [api.CandidateList([api.Candidate(int(i), float(c)) for i, c in zip(ids[int(off[b]):int(off[b + 1])],
                                                                              cls[int(off[b]):int(off[b + 1])])])
          for b in range(B)]
    br = api.rerank_batch(qs, cl, store, cfg)
    for b, st in enumerate(br.stats):  # reference semantics: no prefetch -> every needed doc is fetched
        assert st.needed_count == 64 and st.missed_count == 64 and st.hit_rate == 0.0
        nid = ids[int(off[b]):int(off[b]) + 64].astype(np.int64)
        rec = (128 + (rp[nid + 1] - rp[nid]).astype(np.int64) * 32) * 2  # store.hpp:32-34, d_cls 128, fp16
        assert st.critical_fetch_bytes == int(rec.sum()) == st.needed_payload_bytes
        assert st.critical_blocks_read == int(((rec + 4095) // 4096).sum())  # per record (SPEC "Block accounting")
    rr.close(); store.close()


def test_prefetch_survives_interleaved_plain_batches(cuda_ok):
    # prefetch(A), plain(X), plain(Y), prefetched(A) -- the plain
    # batches must not restage A's pending staging slot
    import torch
    rp, codes, q, ids, cls, off, resident = _tiered_case(seed=212)
    cfg = api.PipelineConfig(rerank_count=64, final_k=10, partial_rerank_enabled=True)
    store = api.GpuStore(rp, codes, 32, resident=resident)
    B, C = len(off) - 1, int(off[-1])
    rr = api.Reranker(store, B, C, 32)
    dev = torch.device("cuda")
    dq, di, dc = (torch.from_numpy(q).to(dev), torch.from_numpy(ids.view(np.int32)).to(dev),
                  torch.from_numpy(cls).to(dev))
    rng = np.random.default_rng(5)
    perm = [rng.permutation(B) for _ in range(2)]
    other = [(dq[p].contiguous(), torch.from_numpy(np.concatenate([ids[int(off[b]):int(off[b + 1])] for b in p])
                                                   .view(np.int32)).to(dev),
              torch.from_numpy(np.concatenate([cls[int(off[b]):int(off[b + 1])] for b in p])).to(dev),
              np.concatenate([[0], np.cumsum(np.diff(off)[p])]).astype(np.uint64)) for p in perm]
    ref = [x.cpu().numpy() for x in rr.rerank_arrays(dq, di, dc, off, cfg, device_io=True)[:3]]
    side = torch.cuda.Stream()
    rr.prefetch(dq, di, dc, off, cfg, stream=side.cuda_stream)
    for oq, oi, oc, oo in other:
        rr.rerank_arrays(oq, oi, oc, oo, cfg, device_io=True)
    got = rr.rerank_arrays(dq, di, dc, off, cfg, device_io=True, prefetched=True, fetch_stats=True)
    for g, r in zip(got[:3], ref):
        assert np.array_equal(g.cpu().numpy(), r)
    assert all(fs["missed"] == 0 for fs in rr.last_fetch_stats)
    rr.close(); store.close()


def test_sync_graph_key_tracks_list_lengths(cuda_ok):
    # the separate top-k's dedup hash is sized by the longest list;
    # a replayed graph of the same (B, C) with a longer list must still reject
    # duplicates
    rp, codes = synth.make_table(4000, 48, 1, 20, seed=17)  # d=48: CUDA-core path, separate top-k
    q, _ = synth.make_queries(rp, codes, 48, 4, seed=18)
    cfg = api.PipelineConfig(rerank_count=2000, final_k=10)
    store = api.GpuStore(rp, codes, 48)
    rr = api.Reranker(store, 4, 2000, 32)
    rng = np.random.default_rng(19)
    even = np.arange(5) * 500
    for _ in range(3):  # eager, capture, replay of the balanced shape
        ids = rng.permutation(4000)[:2000].astype(np.uint32)
        rr.rerank_arrays(q, ids, rng.random(2000, dtype=np.float32), even.astype(np.uint64), cfg)
    skew = np.array([0, 1700, 1800, 1900, 2000], np.uint64)  # same B and C, one long list
    ids = rng.permutation(4000)[:2000].astype(np.uint32)
    ids[1600] = ids[3]  # duplicate inside the long list
    with pytest.raises(api.InvalidInputError):
        rr.rerank_arrays(q, ids, rng.random(2000, dtype=np.float32), skew, cfg)
    rr.close(); store.close()


def test_tiered_gather_and_staging_overflow(oracle, cuda_ok):
    rp, codes, q, ids, cls, off, resident = _tiered_case(seed=303)
    store = api.GpuStore(rp, codes, 32, resident=resident)
    req = np.random.default_rng(3).integers(0, 6000, size=300).astype(np.uint32)
    res = store.fetch_batch(req)
    st, orp, orows = oracle.gather(oracle.OracleTable(rp, codes, 32), req)
    assert st == 0
    assert np.array_equal(np.concatenate([api.encode(d.bow.values, "f16") for d in res.docs]), orows)
    rr = api.Reranker(store, len(off) - 1, int(off[-1]), 32, staging_bytes=4096)  # far too small
    with pytest.raises(api.InvalidConfigError):
        rr.rerank_arrays(q, ids, cls, off, api.PipelineConfig(rerank_count=600, final_k=10))
    rr.close(); store.close()


# ---- fused top-k (ranking inside the tcgen05 MaxSim kernel) vs the separate
# top-k kernel: identical ranked lists, counts and error verdicts ----
def _run_pair(rp, codes, d, q, ids, cls, off, cfg, reps=1):
    store = api.GpuStore(rp, codes, d)
    rr = api.Reranker(store, len(off) - 1, max(int(off[-1]), 1), q.shape[1])
    outs = []
    for sep in (False, True) * reps:
        outs.append(rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", separate_topk=sep))
    rr.close()
    store.close()
    return outs


@pytest.mark.parametrize("k", [1, 10, 16, 32])
@pytest.mark.parametrize("partial", [False, True])
def test_fused_topk_matches_separate(oracle, cuda_ok, k, partial):
    rp, codes, q, ids, cls, off = build_case(20000, 32, 1, 63, B=6, K=1000, seed=71 + k)
    cfg = api.PipelineConfig(rerank_count=300 if partial else 1000, final_k=k, alpha=0.7,
                             partial_rerank_enabled=partial)
    outs = _run_pair(rp, codes, 32, q, ids, cls, off, cfg, reps=2)
    for o in outs[1:]:  # repeated batches: per-query hash/counters were reset by the last unit
        assert np.array_equal(outs[0][0], o[0]) and np.array_equal(outs[0][1].view(np.uint32), o[1].view(np.uint32))
        assert np.array_equal(outs[0][2], o[2])
    check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")


def test_fused_topk_ragged_and_empty_queries(oracle, cuda_ok):
    # empty lists, lists shorter than k, partial tails only (R=0 would be
    # invalid; R < n with partial), a single-candidate list
    rp, codes = synth.make_table(3000, 32, 1, 63, seed=81)
    q, _ = synth.make_queries(rp, codes, 32, 6, seed=82)
    rng = np.random.default_rng(83)
    ids_l, cls_l, offs = [], [], [0]
    for n in [0, 5, 1, 130, 0, 999]:
        c = rng.permutation(3000)[:n].astype(np.uint32)
        s = np.sort(rng.random(n).astype(np.float32))[::-1].copy()
        o = np.lexsort((c, -s))
        ids_l.append(c[o]); cls_l.append(s[o]); offs.append(offs[-1] + n)
    ids = np.concatenate(ids_l).astype(np.uint32)
    cls = np.concatenate(cls_l).astype(np.float32)
    off = np.asarray(offs, np.uint64)
    for cfg in (api.PipelineConfig(rerank_count=64, final_k=10, partial_rerank_enabled=True),
                api.PipelineConfig(rerank_count=1000, final_k=10)):
        a, b = _run_pair(rp, codes, 32, q, ids, cls, off, cfg)
        assert np.array_equal(a[2], b[2])
        for i in range(6):
            n = int(a[2][i])
            assert np.array_equal(a[0][i, :n], b[0][i, :n]) and np.array_equal(a[1][i, :n], b[1][i, :n])
        check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")


def test_fused_topk_duplicates_across_units_and_tail(cuda_ok):
    rp, codes, q, ids, cls, off = build_case(5000, 32, 1, 63, B=3, K=1000, seed=91)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 3, 3000, 32)
    full = api.PipelineConfig(rerank_count=1000, final_k=10)
    part = api.PipelineConfig(rerank_count=100, final_k=10, partial_rerank_enabled=True)
    good = rr.rerank_arrays(q, ids, cls, off, full, kernel="tcgen05")
    cases = [(1003, 1990, full), (5, 900, full), (2050, 2999, part), (10, 500, part)]  # (copy to, copy from)
    for i, j, cfg in cases:
        dup = ids.copy(); dup[i] = dup[j]
        for sep in (False, True):
            with pytest.raises(api.InvalidInputError):
                rr.rerank_arrays(q, dup, cls, off, cfg, kernel="tcgen05", separate_topk=sep)
        # the failed batch left no state behind
        again = rr.rerank_arrays(q, ids, cls, off, full, kernel="tcgen05")
        assert np.array_equal(again[0], good[0]) and np.array_equal(again[2], good[2])
    rr.close(); store.close()


# ---- host-I/O path: inputs staged on the workspace copy stream (double-
# buffered slots), ASYNC batches in flight, ranked lists written zero-copy
# into pinned host outputs -- identical to the synchronous pageable path ----
def test_host_io_async_pipelined_zero_copy(cuda_ok):
    import torch
    rp, codes = synth.make_table(20000, 32, 1, 63, seed=101)
    store = api.GpuStore(rp, codes, 32)
    B, K = 8, 600
    cfg = api.PipelineConfig(rerank_count=K, final_k=10)
    batches = []
    for j in range(5):
        q, src = synth.make_queries(rp, codes, 32, B, seed=102 + j)
        ids, cls, off = synth.make_candidates(20000, B, K, src=src, seed=110 + j)
        batches.append((q, ids, cls, off))
    rr = api.Reranker(store, B, B * K, 32)
    want = [rr.rerank_arrays(q, ids, cls, off, cfg) for q, ids, cls, off in batches]  # pageable, synchronous
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    ins = [(pin(q), pin(ids.view(np.int32)), pin(cls), off) for q, ids, cls, off in batches]
    outs = [(pin(np.zeros((B, 10), np.int32)), pin(np.zeros((B, 10), np.float32)), pin(np.zeros(B, np.int32)), None)
            for _ in batches]
    s = torch.cuda.Stream()
    for (q, ids, cls, off), o in zip(ins, outs):  # all five queued before any sync
        rr.rerank_arrays(q, ids, cls, off, cfg, out=o, stream=s.cuda_stream, sync=False)
    s.synchronize()
    rr.sync(s.cuda_stream)
    for w, o in zip(want, outs):
        assert np.array_equal(w[0].view(np.int32), o[0].numpy())
        assert np.array_equal(w[1].view(np.uint32), o[1].numpy().view(np.uint32))
        assert np.array_equal(w[2].view(np.int32), o[2].numpy())
    rr.close()
    store.close()


# ---- full size (configs[1]): 8.8 M docs, the 18 GB table generated on the
# device.  Size-independent parity: fused == separate top-k for every query,
# and for sampled queries all 1000 MaxSim scores equal the CPU oracle computed
# on the rows gathered back from HBM; the source doc ranks first ----
def test_full_scale_c2_sampled_parity(oracle, cuda_ok):
    import sys
    from pathlib import Path
    import torch
    from paper_2312_05417_b200 import _lib as L
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    cfg = bench.CONFIGS["c2"]
    N, d, B, K = cfg["n_docs"], cfg["d"], cfg["batch"], cfg["K"]
    lib = L.lib()
    rp = torch.zeros(N + 1, dtype=torch.int64, device="cuda")
    assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(), None, None) == 0
    rows = torch.empty(int(rp[-1]) * d, dtype=torch.int16, device="cuda")
    assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(),
                                    rows.data_ptr(), None) == 0
    store = api.GpuStore.from_device(rp, rows, d, "f16", device=0, rows_tiled=True)
    bt = bench.make_batches(cfg, 1, B)[0]
    q, ids, cls, off = bt["q"], bt["ids"], bt["cls"], bt["off"]
    rr = api.Reranker(store, B, B * K, 32)
    pcfg = api.PipelineConfig(rerank_count=K, final_k=10)
    gi, gs, gc, gbow = rr.rerank_arrays(q, ids, cls, off, pcfg, write_bow=True)
    si, ss, sc, _ = rr.rerank_arrays(q, ids, cls, off, pcfg, separate_topk=True)
    assert np.array_equal(gi, si) and np.array_equal(gs.view(np.uint32), ss.view(np.uint32))
    assert np.array_equal(gc, sc) and np.all(gc == 10)
    assert np.array_equal(gi[:, 0], ids.reshape(B, K)[:, 0])  # the perturbed query's source doc
    for qi in (0, 37):
        cid = torch.from_numpy(ids[qi * K:(qi + 1) * K].astype(np.int32)).cuda()
        lrp = torch.zeros(K + 1, dtype=torch.int64, device="cuda")
        assert lib.espn_gpu_gather(store.handle, cid.data_ptr(), K, None, lrp.data_ptr(), 0, None) == 0
        lrows = torch.empty(int(lrp[-1]) * d, dtype=torch.int16, device="cuda")
        assert lib.espn_gpu_gather(store.handle, cid.data_ptr(), K, lrows.data_ptr(), lrp.data_ptr(),
                                   int(lrp[-1]), None) == 0
        ot = oracle.OracleTable(lrp.cpu().numpy(), lrows.cpu().numpy().view(np.uint16), d)
        st, obow = oracle.maxsim_batch(ot, np.ascontiguousarray(q[qi:qi + 1]), np.arange(K, dtype=np.uint32),
                                       np.array([0, K], np.uint64))
        assert st == 0
        e = rel_err(gbow[qi * K:(qi + 1) * K], obow)
        assert e.max() <= RTOL, f"query {qi}: max rel err {e.max()}"
    rr.close()
    store.close()


# ---- the graph-capturable mode the bench times: device arrays + device
# offsets (the batch is planned on the device), captured in a CUDA graph and
# replayed; identical to the host-offset call ----
@pytest.mark.parametrize("partial", [False, True])
def test_device_offsets_graph_replay(cuda_ok, partial):
    import ctypes as C
    import torch
    from paper_2312_05417_b200 import _lib as L
    rp, codes, q, ids, cls, off = build_case(20000, 32, 1, 63, B=16, K=700, seed=131)
    R = 200 if partial else 700
    cfg = api.PipelineConfig(rerank_count=R, final_k=10, alpha=0.9, partial_rerank_enabled=partial)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 16, 16 * 700, 32, max_list=700)
    want = rr.rerank_arrays(q, ids, cls, off, cfg)
    dq = torch.from_numpy(q).cuda()
    did = torch.from_numpy(ids.view(np.int32)).cuda()
    dcl = torch.from_numpy(cls).cuda()
    doff = torch.from_numpy(off.astype(np.int64)).cuda()
    out = torch.zeros(2 * 16 * 10 + 16, dtype=torch.int32, device="cuda")
    base = out.data_ptr()
    flags = L.ESPN_RERANK_DEVICE_IO | L.ESPN_RERANK_DEVICE_OFFSETS | L.ESPN_RERANK_ASYNC
    flags |= L.ESPN_RERANK_PARTIAL if partial else 0

    def enqueue(sp):
        a = L.RerankArgs(n_queries=16, n_query_tokens=32, query_tokens=dq.data_ptr(), cand_ids=did.data_ptr(),
                         cand_cls=dcl.data_ptr(), cand_offsets=doff.data_ptr(), rerank_count=R, final_k=10,
                         alpha=0.9, flags=flags, kernel=L.ESPN_KERNEL_AUTO)
        o = L.RerankOut(ids=base, scores=base + 4 * 160, counts=base + 8 * 160)
        assert L.lib().espn_gpu_rerank(store.handle, rr.handle, C.byref(a), C.byref(o), C.c_void_p(sp)) == 0

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        enqueue(s.cuda_stream)  # eager first (lazy attributes)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        enqueue(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        rr.sync()
        o = out.cpu().numpy()
        gi, gs, gc = o[:160].reshape(16, 10), o[160:320].view(np.float32).reshape(16, 10), o[320:]
        assert np.array_equal(gc, want[2].view(np.int32))
        assert np.array_equal(gi, want[0].view(np.int32))
        assert np.array_equal(gs.view(np.uint32), want[1].view(np.uint32))
    rr.close()
    store.close()


def test_sync_graph_replay_fresh_data_and_errors(oracle, cuda_ok):
    """Synchronous pageable-buffer calls of a repeating shape run as a replayed
    CUDA graph from the second call on: every call must see its own inputs,
    interleaved shapes must re-capture, and device-side errors must surface."""
    rp, codes = synth.make_table(6000, 32, 1, 63, seed=81)
    store = api.GpuStore(rp, codes, 32)
    rr = api.Reranker(store, 8, 8 * 400, 32)
    cfg = api.PipelineConfig(rerank_count=400, final_k=10)
    for i in range(6):
        B = 4 if i % 3 else 3  # shapes 3, 4, 4, 3, 4, 4: captures, replays and re-captures
        q, src = synth.make_queries(rp, codes, 32, B, nq=32, seed=90 + i)
        ids, cls, off = synth.make_candidates(6000, B, 400, src=src, seed=100 + i)
        check_against_oracle(oracle, rp, codes, 32, "f16", q, ids, cls, off, cfg, "tcgen05")
        gi, gs, gc, _ = rr.rerank_arrays(q, ids, cls, off, cfg)
        assert np.array_equal(gi[:, 0], src.astype(np.uint32)), i
    bad = ids.copy()
    bad[5] = bad[9]  # duplicate candidate -> InvalidInputError from the device check
    for _ in range(3):
        with pytest.raises(api.InvalidInputError):
            rr.rerank_arrays(q, bad, cls, off, cfg)
        gi, _, _, _ = rr.rerank_arrays(q, ids, cls, off, cfg)  # and the next call is clean
        assert np.array_equal(gi[:, 0], src.astype(np.uint32))
    rr.close()
    store.close()
