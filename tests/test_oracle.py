"""CPU: the oracle pinned against the reference's golden vectors and SPEC
known-answer tests, plus the SPEC's property invariants for the hot path.
(No GPU: these run in the driver's `-m "not gpu"` pass.)"""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def kats():
    return json.loads((GOLD / "spec_kats.json").read_text())


# ---------------------------------------------------------------- codec (half.hpp)
def test_fp16_decode_matches_reference_codec(oracle):
    """All 65,536 codes against the reference's own half_to_float (half.hpp:47-73).
    Normals, zeros, inf and NaN agree bit-exactly; the 2,046 subnormal codes
    expose the reference defect (exponent 113-e instead of 112-e, half.hpp:64):
    it returns exactly twice the IEEE value, which the oracle does not copy."""
    g = np.load(GOLD / "half_ref_codec.npz")
    ref_bits = g["decode_bits"]
    ours = oracle.decode(np.arange(65536, dtype=np.uint32).astype(np.uint16)).view(np.uint32)
    codes = np.arange(65536)
    sub = ((codes & 0x7C00) == 0) & ((codes & 0x3FF) != 0)
    assert sub.sum() == 2046
    assert np.array_equal(ours[~sub], ref_bits[~sub])
    r = ref_bits[sub].view(np.float32).astype(np.float64)
    o = ours[sub].view(np.float32).astype(np.float64)
    assert np.array_equal(r, 2.0 * o)
    # the IEEE value is the hardware one (numpy float16)
    assert np.array_equal(o, codes[sub].astype(np.uint16).view(np.float16).astype(np.float64))


def test_fp16_encode_matches_reference_codec(oracle):
    """float_to_half (half.hpp:11-45) on the committed sweep: identical for every
    input outside [2^-25, 2^-14), where the reference flushes to zero."""
    g = np.load(GOLD / "half_ref_codec.npz")
    xs, ref = g["sweep"], g["encode"]
    ours = oracle.encode(xs)
    a = np.abs(xs.astype(np.float64))
    in_sub = (a >= 2.0 ** -25) & (a < 2.0 ** -14)
    nan = np.isnan(xs)
    assert np.array_equal(ours[~in_sub & ~nan], ref[~in_sub & ~nan])
    assert np.all((ours[nan] & 0x7E00) == 0x7E00) and np.all((ref[nan] & 0x7C00) == 0x7C00)
    # reference maps the subnormal band to signed zero; the oracle keeps IEEE RNE
    assert np.all((ref[in_sub] & 0x7FFF) == 0)
    np16 = xs[in_sub].astype(np.float16).view(np.uint16)
    assert np.array_equal(ours[in_sub], np16)


def test_fp16_encode_matches_numpy_everywhere(oracle):
    xs = np.load(GOLD / "half_ref_codec.npz")["sweep"]
    ok = ~np.isnan(xs)
    assert np.array_equal(oracle.encode(xs[ok]), xs[ok].astype(np.float16).view(np.uint16))


def test_live_reference_codec_if_built(oracle):
    ref = oracle.ref_half()
    if ref is None:
        pytest.skip("oracle/_ref not built on this host (reference tree absent)")
    for c in [0x3C00, 0x0001, 0x03FF, 0x7BFF, 0x7C00, 0xFC00, 0x8000]:
        assert ref.ref_half_to_float_bits(c) == np.load(GOLD / "half_ref_codec.npz")["decode_bits"][c]


def test_bf16_codec(oracle):
    rng = np.random.default_rng(3)
    x = rng.standard_normal(10000).astype(np.float32)
    c = oracle.encode(x, oracle.BF16)
    u = x.view(np.uint32).astype(np.uint64)
    exp = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(c, exp)
    assert np.array_equal(oracle.decode(c, oracle.BF16).view(np.uint32), c.astype(np.uint32) << 16)


# ---------------------------------------------------------------- scoring.hpp KATs
def test_maxsim_kats(oracle, kats):
    for k in kats["maxsim"]:
        q = np.asarray(k["q"], np.float32)
        d = np.asarray(k["d"], np.float32)
        got = np.float32(oracle.maxsim_score(q, d))
        if "score" in k:
            assert got == np.float32(k["score"]), k["src"]
        else:
            assert got.view(np.uint32) == k["score_bits"], k["src"]


def test_maxsim_200_pairs_bitexact(oracle, kats):
    """Acceptance criterion 1: 200 random pairs up to 16 tokens,
    bit-exact against an independent brute-force double loop."""
    for k in kats["maxsim_random_pairs"]:
        q = np.asarray(k["q"], np.float32)
        d = np.asarray(k["d"], np.float32)
        assert np.float32(oracle.maxsim_score(q, d)).view(np.uint32) == k["score_bits"]


def test_maxsim_monotone_under_row_append(oracle):
    rng = np.random.default_rng(5)
    for _ in range(50):
        q = rng.standard_normal((8, 16)).astype(np.float32)
        d = rng.standard_normal((5, 16)).astype(np.float32)
        d2 = np.concatenate([d, rng.standard_normal((1, 16)).astype(np.float32)])
        assert oracle.maxsim_score(q, d2) >= oracle.maxsim_score(q, d)


def test_aggregate_kats(oracle, kats):
    for k in kats["aggregate"]:
        assert oracle.aggregate_score(k["cls"], k["bow"], k["alpha"]) == k["score"], k["src"]


def test_rank_kats_and_properties(oracle, kats):
    for k in kats["rank"]:
        ids = [e[0] for e in k["in"]]
        sc = [e[1] for e in k["in"]]
        st, oi, os_ = oracle.rank(ids, sc)
        assert st == 0
        assert [[int(i), float(s)] for i, s in zip(oi, os_)] == k["out"], k["src"]
    rng = np.random.default_rng(7)  # 100 random entries vs a stable-sort oracle
    ids = rng.permutation(1000)[:100].astype(np.uint32)
    sc = rng.integers(0, 20, 100).astype(np.float32)  # many ties
    st, oi, os_ = oracle.rank(ids, sc)
    exp = sorted(zip(ids.tolist(), sc.tolist()), key=lambda e: (-e[1], e[0]))
    assert st == 0 and list(zip(oi.tolist(), os_.tolist())) == exp
    st2, oi2, os2 = oracle.rank(oi, os_)  # idempotence
    assert st2 == 0 and np.array_equal(oi2, oi)
    assert oracle.rank([1, 1], [1.0, 2.0])[0] == 1  # duplicates rejected
    assert oracle.rank([1, 2], [np.nan, 2.0])[0] == 1  # non-finite rejected


def test_record_bytes_kat(oracle, kats):
    k = kats["record_bytes"][0]  # 128*2 + 10*32*2 = 896
    rp = np.array([0, k["t"]], np.uint64)
    t = oracle.OracleTable(rp, np.zeros(k["t"] * k["d"], np.uint16), k["d"], d_cls=k["d_cls"],
                           value_width=k["width"])
    import ctypes
    assert oracle.lib().eo_record_bytes(ctypes.byref(t.s), 0) == k["bytes"]


# ---------------------------------------------------------------- pipeline stages 3-6
def _case(n_docs=400, d=16, B=3, K=120, seed=0):
    from paper_2312_05417_b200 import synth
    rp, codes = synth.make_table(n_docs, d, 1, 20, seed=seed)
    q, src = synth.make_queries(rp, codes, d, B, nq=8, seed=seed + 1)
    ids, cls, off = synth.make_candidates(n_docs, B, K, src=src, seed=seed + 2)
    return rp, codes, q, ids, cls, off


def test_prefetch_on_off_identical(oracle):
    """SPEC.md:302 / acceptance 5: result identical with prefetch on or off."""
    rp, codes, q, ids, cls, off = _case()
    t = oracle.OracleTable(rp, codes, 16)
    rng = np.random.default_rng(9)
    for b in range(3):
        a0, a1 = int(off[b]), int(off[b + 1])
        pf = rng.choice(ids[a0:a1], size=50, replace=False)
        on = oracle.rerank_query(t, q[b], ids[a0:a1], cls[a0:a1], 60, 10, prefetched=pf)
        offr = oracle.rerank_query(t, q[b], ids[a0:a1], cls[a0:a1], 60, 10, prefetch_enabled=False)
        assert on[0] == 0 and offr[0] == 0
        assert np.array_equal(on[1], offr[1]) and np.array_equal(on[2].view(np.uint32), offr[2].view(np.uint32))
        assert offr[3].prefetched_count == 0 and offr[3].hit_rate == 0.0


def test_hit_rate_and_critical_path_accounting(oracle):
    """SPEC.md:279 (step=100 => hit 1.0), SPEC.md:305 / acceptance 9."""
    rp, codes, q, ids, cls, off = _case(seed=3)
    t = oracle.OracleTable(rp, codes, 16, alignment=4096, direct_io=True)
    a0, a1 = int(off[0]), int(off[1])
    R = 80
    full = oracle.rerank_query(t, q[0], ids[a0:a1], cls[a0:a1], R, 10, prefetched=ids[a0:a0 + R])
    assert full[3].hit_rate == 1.0 and full[3].missed_count == 0 and full[3].critical_fetch_bytes == 0
    rng = np.random.default_rng(4)
    pf = rng.choice(ids[a0:a1], size=70, replace=False)
    st, _, _, s = oracle.rerank_query(t, q[0], ids[a0:a1], cls[a0:a1], R, 10, prefetched=pf)
    needed = set(ids[a0:a0 + R].tolist())
    hits = len(needed & set(pf.tolist()))
    assert s.needed_count == R and s.missed_count == R - hits
    assert abs(s.hit_rate - hits / R) < 1e-12
    tok = (rp[1:] - rp[:-1])[ids[a0:a0 + R]]
    payload = (128 + tok * 16) * 2
    assert s.needed_payload_bytes == int(payload.sum())
    pad = 4095 * s.missed_count
    assert s.critical_fetch_bytes <= (1 - s.hit_rate) * s.needed_payload_bytes + pad + 1e-6 * s.needed_payload_bytes \
        or s.critical_fetch_bytes <= s.needed_payload_bytes + pad


def test_partial_r_equals_k_is_full(oracle):
    rp, codes, q, ids, cls, off = _case(seed=6)
    t = oracle.OracleTable(rp, codes, 16)
    a0, a1 = int(off[1]), int(off[2])
    n = a1 - a0
    a = oracle.rerank_query(t, q[1], ids[a0:a1], cls[a0:a1], n, 10, partial=False)
    b = oracle.rerank_query(t, q[1], ids[a0:a1], cls[a0:a1], n, 10, partial=True)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_partial_tail_scored_alpha_cls(oracle):
    rp, codes, q, ids, cls, off = _case(seed=8)
    t = oracle.OracleTable(rp, codes, 16)
    a0, a1 = int(off[0]), int(off[1])
    st, oi, os_, s = oracle.rerank_query(t, q[0], ids[a0:a1], cls[a0:a1], 5, 30, alpha=2.0, partial=True)
    assert st == 0 and len(oi) == 30
    tail = {int(i): np.float32(2.0) * c for i, c in zip(ids[a0 + 5:a1], cls[a0 + 5:a1])}
    for i, sc in zip(oi, os_):
        if int(i) in tail:
            assert np.float32(sc) == np.float32(tail[int(i)] + np.float32(0.0))


def test_config_validation_and_errors(oracle):
    rp, codes, q, ids, cls, off = _case(seed=10)
    t = oracle.OracleTable(rp, codes, 16)
    a0, a1 = int(off[0]), int(off[1])
    assert oracle.rerank_query(t, q[0], ids[a0:a1], cls[a0:a1], 5, 10)[0] == 1  # R < k w/o partial
    bad = ids[a0:a1].copy(); bad[0] = 400
    assert oracle.rerank_query(t, q[0], bad, cls[a0:a1], 50, 10)[0] == 6  # DataIntegrity
    dup = ids[a0:a1].copy(); dup[1] = dup[0]
    assert oracle.rerank_query(t, q[0], dup, cls[a0:a1], 50, 10)[0] == 1


def test_batch_equals_serial(oracle):
    """run_batch results identical to serial calls."""
    rp, codes, q, ids, cls, off = _case(B=6, seed=12)
    t = oracle.OracleTable(rp, codes, 16)
    st, bi, bs, bn = oracle.rerank_batch(t, q, ids, cls, off, 60, 10, nthreads=4)
    assert st == 0
    for b in range(6):
        a0, a1 = int(off[b]), int(off[b + 1])
        s1 = oracle.rerank_query(t, q[b], ids[a0:a1], cls[a0:a1], 60, 10)
        assert np.array_equal(s1[1], bi[b, :bn[b]]) and np.array_equal(s1[2], bs[b, :bn[b]])


def test_gather_oracle(oracle):
    rp, codes, q, ids, cls, off = _case(seed=14)
    t = oracle.OracleTable(rp, codes, 16)
    st, orp, rows = oracle.gather(t, [5, 5, 0, 399])
    assert st == 0
    for j, i in enumerate([5, 5, 0, 399]):
        a, b = int(rp[i]), int(rp[i + 1])
        assert np.array_equal(rows[int(orp[j]) * 16:int(orp[j + 1]) * 16], codes[a * 16:b * 16])
    assert oracle.gather(t, [400])[0] == 1
