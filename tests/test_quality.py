"""Quality harness (metrics.hpp:10-20).

CPU: the SPEC's metric examples, qrels parsing and errors, metric bounds and
monotonicity in k, and the C++ espn::gpu metrics against the Python mirror.
GPU: the device re-ranker's MRR@10 / Recall@10 over an R sweep equal the
oracle's on the same inputs, and MRR is nondecreasing in R.
"""
import subprocess

import numpy as np
import pytest

from paper_2312_05417_b200 import api, build, quality

ROOT = build.ROOT


def rl(*ids):
    return api.RankedList([api.ScoredDoc(d, float(100 - i)) for i, d in enumerate(ids)])


def test_spec_mrr_examples():
    # SPEC.md:76-79
    assert api.mrr_at_k({1: rl(7, 8)}, {1: {7}}, 10) == 1.0
    assert api.mrr_at_k({1: rl(8, 7)}, {1: {7}}, 10) == 0.5
    res = {1: rl(5, 6, 7), 2: rl(1, 2, 3, 9), 3: rl(1, 2, 3)}
    q = {1: {5}, 2: {9}, 3: {42}}
    assert api.mrr_at_k(res, q, 3) == pytest.approx(1 / 3)


def test_spec_recall_examples():
    # SPEC.md:84-87
    assert api.recall_at_k({1: rl(1, 2, 3)}, {1: {1, 3}}, 3) == 1.0
    assert api.recall_at_k({1: rl(1, 2, 3)}, {1: {4, 5}}, 3) == 0.0
    assert api.recall_at_k({1: rl(1, 2, 3)}, {1: {2, 9}}, 3) == 0.5


def test_missing_results_count_zero_and_k_checked():
    assert api.mrr_at_k({}, {1: {1}, 2: {2}}, 10) == 0.0
    assert api.mrr_at_k({1: rl(1)}, {1: {1}, 2: {2}}, 10) == 0.5
    assert api.mrr_at_k({1: rl(1)}, {}, 10) == 0.0
    with pytest.raises(api.InvalidInputError):
        api.mrr_at_k({1: rl(1)}, {1: {1}}, 0)
    with pytest.raises(api.InvalidInputError):
        api.recall_at_k({1: rl(1)}, {1: {1}}, 0)


def test_load_qrels(tmp_path):
    p = tmp_path / "q.txt"
    p.write_text("1 0 10 1\n\n1 0 11 0\n  \n2 0 20 2\n1 0 12 3\n3 0 30 0\n")
    assert api.load_qrels(p) == {1: {10, 12}, 2: {20}}
    for bad in ["1 0 10\n", "1 0 x 1\n", "1 0 10 1 extra\n", "-1 0 10 1\n"]:
        p.write_text(bad)
        with pytest.raises(api.FormatError):
            api.load_qrels(p)
    with pytest.raises(api.IoError):
        api.load_qrels(tmp_path / "missing.txt")


def test_bounds_and_monotone_in_k():
    rng = np.random.default_rng(3)
    for _ in range(20):
        res = {q: list(rng.permutation(50)[:20]) for q in range(30)}
        qrels = {q: set(rng.integers(0, 50, rng.integers(1, 5)).tolist()) for q in range(35)}
        prev = (0.0, 0.0)
        for k in range(1, 25):
            m, r = api.mrr_at_k(res, qrels, k), api.recall_at_k(res, qrels, k)
            assert 0.0 <= m <= 1.0 and 0.0 <= r <= 1.0
            assert m >= prev[0] and r >= prev[1]
            prev = (m, r)


def _metrics_exe(tmp_path):
    lib = build.build_host()
    exe = tmp_path / "metrics_test"
    cmd = [build.CXX, "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-o", str(exe),
           str(ROOT / "tests" / "cpp" / "metrics_test.cpp"), "-L", str(lib.parent), "-lespn_host", "-lespn_gpu",
           "-lespn_store", f"-Wl,-rpath,{lib.parent}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_metrics_match_python(tmp_path):
    exe = _metrics_exe(tmp_path)
    rng = np.random.default_rng(9)
    res = {q: [int(x) for x in rng.permutation(200)[:rng.integers(0, 30)]] for q in range(60)}
    qrels = {q: set(int(x) for x in rng.integers(0, 200, rng.integers(1, 6))) for q in range(0, 70, 1)}
    qp, rp = tmp_path / "qrels", tmp_path / "res"
    lines = [f"{q} 0 {d} {int(rng.integers(1, 3))}" for q, ds in qrels.items() for d in sorted(ds)]
    lines += [f"{q} 0 {1000 + q} 0" for q in range(5)]  # non-relevant judgements
    qp.write_text("\n".join(lines) + "\n")
    rp.write_text("".join(f"{q} {' '.join(map(str, ds))}\n" for q, ds in res.items()))
    ks = [1, 3, 10, 100]
    out = subprocess.run([str(exe), str(qp), str(rp), *map(str, ks)], capture_output=True, text=True,
                         check=True).stdout.split("\n")
    q2 = api.load_qrels(qp)
    assert q2 == qrels
    for k, line in zip(ks, out):
        m, r = (float(x) for x in line.split())
        assert m == pytest.approx(api.mrr_at_k(res, q2, k), rel=1e-15, abs=0)
        assert r == pytest.approx(api.recall_at_k(res, q2, k), rel=1e-15, abs=0)
    qp.write_text("1 0 zz 1\n")
    assert subprocess.run([str(exe), str(qp), str(rp), "10"], capture_output=True, text=True).stdout.strip() \
        == "error FormatError"
    assert subprocess.run([str(exe), str(tmp_path / "nope"), str(rp), "10"], capture_output=True,
                          text=True).stdout.strip() == "error IoError"
    qp.write_text("1 0 1 1\n")
    assert subprocess.run([str(exe), str(qp), str(rp), "0"], capture_output=True, text=True).stdout.strip() \
        == "error InvalidInputError"


def test_eval_set_shape():
    rp, codes, q, ids, cls, off, qrels = quality.make_eval_set(2000, 32, 16, 300, seed=3)
    assert q.shape == (16, 32, 32) and len(off) == 17 and len(qrels) == 16
    for b in range(16):
        seg_ids, seg_cls = ids[int(off[b]):int(off[b + 1])], cls[int(off[b]):int(off[b + 1])]
        assert len(np.unique(seg_ids)) == seg_ids.size
        assert np.all(np.diff(seg_cls) <= 0)


@pytest.mark.gpu
def test_rerank_sweep_matches_oracle_and_is_monotone(oracle, cuda_ok):
    rp, codes, q, ids, cls, off, qrels = quality.make_eval_set(20000, 32, 64, 1000, seed=11)
    store = api.GpuStore(rp, codes, 32, "f16")
    Rs = [16, 64, 256, 1000]
    r = quality.rerank_sweep(store, q, ids, cls, off, qrels, Rs, k=10)
    store.close()
    import oracle_py
    ot = oracle.OracleTable(rp, codes, 32, dtype=oracle_py.F16)
    qr = np.ascontiguousarray(q, np.float32)  # the reference's fp32 query
    for R in Rs:
        st, oi, _, on = oracle.rerank_batch(ot, qr, ids, cls, off, R, 10, 1.0, True)
        assert st == 0
        res = quality.results_from_arrays(oi, on)
        assert r["R"][R]["mrr"] == pytest.approx(api.mrr_at_k(res, qrels, 10), abs=1e-12), R
        assert r["R"][R]["recall"] == pytest.approx(api.recall_at_k(res, qrels, 10), abs=1e-12), R
    mrr = [r["R"][R]["mrr"] for R in Rs]
    assert all(a <= b for a, b in zip(mrr, mrr[1:])), mrr
    assert mrr[-1] > r["first_stage"]["mrr"]
    # SPEC.md:464 (scaled-down Fig. 6): MRR@10(R=64) / MRR@10(R=1000) expected >= 0.95
    assert r["mrr_ratio_vs_Rmax"][64] >= 0.95, r["mrr_ratio_vs_Rmax"]
