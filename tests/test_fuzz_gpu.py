"""GPU fuzz: seeded random shapes and knobs (batch size, ragged list lengths,
R, k, partial re-rank, alpha, dim, dtype, doc lengths, query tokens) through
the public re-rank call, each checked against the CPU oracle with the same
tolerances as tests/test_gpu_parity.py.  One workspace per table serves every
case three times in a row, so shape changes, the synchronous-call graph
(eager first call, capture on the second, replay on the third) and the
small-batch work units are all exercised."""
import os

import numpy as np
import pytest

from helpers import assert_topk_equivalent, oracle_full_scores
from paper_2312_05417_b200 import api, synth

pytestmark = pytest.mark.gpu


def _lists(rng, n_docs, B, kmax, src):
    ids_l, cls_l, offs = [], [], [0]
    for b in range(B):
        n = int(rng.integers(0, kmax + 1)) if rng.random() < 0.25 else kmax
        c = rng.permutation(n_docs)[:n].astype(np.uint32)
        if n and src[b] not in c:
            c[0] = src[b]
        s = rng.random(n).astype(np.float32)
        o = np.lexsort((c, -s))
        ids_l.append(c[o]); cls_l.append(s[o]); offs.append(offs[-1] + n)
    return (np.concatenate(ids_l).astype(np.uint32), np.concatenate(cls_l).astype(np.float32),
            np.asarray(offs, np.uint64))


@pytest.mark.parametrize("d,dtype,served", [(32, "f16", False), (16, "bf16", False), (64, "f16", False),
                                            (128, "bf16", False), (32, "f16", True), (64, "bf16", True)])
def test_random_shapes_against_oracle(oracle, cuda_ok, d, dtype, served):
    # served: the same cases through the persistent re-rank server (fused
    # top-k only: k <= 32, the server's query precision)
    import oracle_py
    odt = oracle_py.F16 if dtype == "f16" else oracle_py.BF16
    rng = np.random.default_rng(1000 + d)
    n_docs = 3000
    rp, codes = synth.make_table(n_docs, d, 1, int(rng.choice([8, 40, 120])), dtype=dtype, seed=d)
    store = api.GpuStore(rp, codes, d, dtype=dtype)
    rr = api.Reranker(store, 17, 17 * 900, 32)
    ot = oracle.OracleTable(rp, codes, d, dtype=odt)
    if served:
        store.server_start()
    for case in range(int(os.environ.get("ESPN_FUZZ_CASES", "8"))):
        B = int(rng.choice([1, 2, 5, 17]))
        kmax = int(rng.choice([1, 30, 300, 900]))
        nq = int(rng.choice([1, 7, 32]))
        q, src = synth.make_queries(rp, codes, d, B, nq=nq, dtype=dtype, seed=case + 10 * d)
        ids, cls, off = _lists(rng, n_docs, B, kmax, src)
        k = int(rng.choice([1, 10, 32] if served else [1, 10, 32, 100]))
        partial = bool(rng.random() < 0.5)
        R = int(rng.integers(1, kmax + 2)) if partial else int(rng.choice([k, max(k, kmax // 2), kmax + 5]))
        alpha = float(rng.choice([1.0, 0.5, 2.0]))
        cfg = api.PipelineConfig(rerank_count=R, final_k=k, alpha=alpha, partial_rerank_enabled=partial)
        qp = "auto" if served else str(rng.choice(["auto", "auto", "split", "rounded"]))
        # the reference's fp32 query, unrounded (the legacy "rounded" mode: the dtype-rounded one)
        qr = oracle.round_to(q, odt) if qp == "rounded" else np.ascontiguousarray(q, np.float32)
        if not partial and R < k:  # R < final_k needs partial re-ranking: both sides reject
            st, *_ = oracle.rerank_batch(ot, qr, ids, cls, off, R, k, alpha, partial)
            assert st != 0
            with pytest.raises(api.InvalidInputError):
                rr.rerank_arrays(q, ids, cls, off, cfg, query_precision=qp)
            continue
        st, obow = oracle.maxsim_batch(ot, qr, ids, off)
        assert st == 0
        st, oi, os_, on = oracle.rerank_batch(ot, qr, ids, cls, off, R, k, alpha, partial)
        assert st == 0
        for rep in range(3):  # eager, captured, replayed
            gi, gs, gc, _ = [np.copy(x) if x is not None else None for x in rr.rerank_arrays(q, ids, cls, off, cfg, query_precision=qp)]
            for b in range(B):
                a0, a1 = int(off[b]), int(off[b + 1])
                need = min(a1 - a0, R)
                full = oracle_full_scores(obow[a0:a1], cls[a0:a1], alpha, need, partial)
                assert int(gc[b]) == int(on[b]), (case, rep, b)
                n = int(on[b])
                assert_topk_equivalent(gi[b, :n], gs[b, :n], oi[b, :n], os_[b, :n], ids[a0:a1], full,
                                       ctx=f"d={d} {qp} case {case} rep {rep} query {b}")
    if served:
        store.server_stop()
    rr.close()
    store.close()


@pytest.mark.parametrize("d,dtype", [(32, "f16"), (16, "bf16"), (48, "f16"), (128, "f16")])
def test_small_kernel_random_shapes_bitexact(oracle, cuda_ok, d, dtype):
    """The single-launch small-batch kernel (ESPN_KERNEL_SMALL) over random
    shapes within its bounds (B <= 16, scored lists <= 2048, k <= 32):
    ranked ids, scores, counts and bow BIT-EXACT against the oracle on the
    fp32 query, through eager, captured and replayed synchronous calls."""
    import oracle_py
    odt = oracle_py.F16 if dtype == "f16" else oracle_py.BF16
    rng = np.random.default_rng(2000 + d)
    n_docs = 3000
    rp, codes = synth.make_table(n_docs, d, 1, int(rng.choice([8, 40, 63])), dtype=dtype, seed=d + 1)
    store = api.GpuStore(rp, codes, d, dtype=dtype)
    rr = api.Reranker(store, 16, 16 * 2048, 32)
    ot = oracle.OracleTable(rp, codes, d, dtype=odt)
    for case in range(int(os.environ.get("ESPN_FUZZ_CASES", "8"))):
        B = int(rng.choice([1, 2, 3, 8, 16]))
        kmax = int(rng.choice([1, 30, 300, 2048 // B]))
        nq = int(rng.choice([1, 7, 32]))
        q, src = synth.make_queries(rp, codes, d, B, nq=nq, dtype=dtype, seed=case + 20 * d)
        ids, cls, off = _lists(rng, n_docs, B, kmax, src)
        k = int(rng.choice([1, 10, 32]))
        partial = bool(rng.random() < 0.5)
        R = int(rng.integers(1, kmax + 2)) if partial else int(rng.choice([k, max(k, kmax // 2), kmax + 5]))
        alpha = float(rng.choice([1.0, 0.5, 2.0]))
        if not partial and R < k:
            continue
        cfg = api.PipelineConfig(rerank_count=R, final_k=k, alpha=alpha, partial_rerank_enabled=partial)
        qr = np.ascontiguousarray(q, np.float32)
        st, obow = oracle.maxsim_batch(ot, qr, ids, off)
        assert st == 0
        st, oi, os_, on = oracle.rerank_batch(ot, qr, ids, cls, off, R, k, alpha, partial)
        assert st == 0
        for rep in range(3):  # eager, captured, replayed
            gi, gs, gc, gb = [np.copy(x) for x in rr.rerank_arrays(q, ids, cls, off, cfg, kernel="small",
                                                                    write_bow=True)]
            assert np.array_equal(gc.astype(np.int64), np.asarray(on, np.int64)), (case, rep)
            for b in range(B):
                a0, a1 = int(off[b]), int(off[b + 1])
                need = min(a1 - a0, R)
                n = int(on[b])
                assert np.array_equal(gb[a0:a0 + need].view(np.uint32), obow[a0:a0 + need].view(np.uint32))
                assert np.array_equal(gi[b, :n].astype(np.int64), np.asarray(oi[b, :n], np.int64)), (case, rep, b)
                assert np.array_equal(gs[b, :n].view(np.uint32), np.asarray(os_[b, :n], np.float32).view(np.uint32))
    rr.close()
    store.close()
