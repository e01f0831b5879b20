"""Bandwidth model: the SPEC's examples
and properties for Eq. 2-4 and the index-size estimate, plus the tiered-step
predictor bench.py uses for configs[3]."""
import json
from fractions import Fraction

import numpy as np
import pytest

from paper_2312_05417_b200 import api
from paper_2312_05417_b200 import bandwidth as bw


def test_prefetch_budget_examples():
    t = bw.AnnTimeTable.linear(0.01e-3, 3000)  # 0.01 ms per probe
    assert bw.prefetch_budget(t, 2000, 2000) == 0.0
    assert bw.prefetch_budget(t, 2000, 200) == pytest.approx(18e-3)
    with pytest.raises(api.InvalidInputError):
        bw.prefetch_budget(t, 200, 2000)
    with pytest.raises(api.InvalidInputError):
        bw.prefetch_budget(t, 4000, 200)  # outside the measured table


def test_ann_table_interpolates_and_validates():
    t = bw.AnnTimeTable([(100, 1.0), (0, 0.0), (300, 5.0)])
    assert t(50) == 0.5 and t(200) == 3.0 and t(300) == 5.0
    with pytest.raises(api.InvalidInputError):
        bw.AnnTimeTable([(0, 1.0), (10, 0.5)])
    with pytest.raises(api.InvalidInputError):
        bw.AnnTimeTable([])


def test_prefetch_step_examples():
    assert bw.prefetch_step(77, 77) == 100.0
    assert bw.prefetch_step(300, 3000) == pytest.approx(10.0)
    assert bw.prefetch_step(48, 160) == pytest.approx(30.0)
    for d, e in [(0, 10), (11, 10)]:
        with pytest.raises(api.InvalidInputError):
            bw.prefetch_step(d, e)


def test_batch_threshold_examples_and_linearity():
    ssd = bw.TierProfile("ssd", 2e9, 4096)
    assert bw.batch_threshold(ssd, 0.0, 1000 * 4096) == 0.0
    assert bw.batch_threshold(ssd, 0.028, 1000 * 4096) == pytest.approx(2e9 * 0.028 / 4.096e6)
    assert 13.6 < bw.batch_threshold(ssd, 0.028, 1000 * 4096) < 13.7
    base = bw.batch_threshold(bw.TierProfile("a", 1000, 1), 3, 7)
    assert Fraction(bw.batch_threshold(bw.TierProfile("a", 2000, 1), 3, 7)).limit_denominator() == \
        2 * Fraction(base).limit_denominator()
    assert bw.batch_threshold(bw.TierProfile("a", 1000, 1), 6, 7) == pytest.approx(2 * base)
    assert bw.batch_threshold(bw.TierProfile("a", 1000, 1), 3, 14) == pytest.approx(base / 2)
    with pytest.raises(api.InvalidInputError):
        bw.batch_threshold(ssd, 0.028, 0)
    with pytest.raises(api.InvalidInputError):
        bw.TierProfile("x", 0, 4096)


def test_index_size_estimate():
    cg, rr, tot = bw.index_size_estimate(1, 68, 32, 2, 256)
    assert (cg, rr, tot) == (256, 68 * 32 * 2, 256 + 68 * 32 * 2)
    # MS MARCO v1 shape.  The formula gives 597.9M tokens x 64 B
    # = 38.3 GB; the SPEC's "16.8 GB-scale" (PAPER Table 3) is not reachable by
    # this arithmetic, so only the formula and its scaling are asserted.
    _, rr, _ = bw.index_size_estimate(8.8e6, 597.9e6 / 8.8e6, 32, 2, 256)
    assert rr == pytest.approx(597.9e6 * 32 * 2)
    _, rr2, _ = bw.index_size_estimate(138.4e6, 597.9e6 / 8.8e6, 32, 2, 256)
    assert rr2 == pytest.approx(rr * 138.4 / 8.8)


def test_bytes_per_query_from_manifest(tmp_path):
    rng = np.random.default_rng(1)
    t = rng.integers(1, 64, 40)
    rp = np.zeros(41, np.uint64)
    rp[1:] = np.cumsum(t)
    m = api.build_store(tmp_path / "s", rp, rng.standard_normal((int(rp[-1]), 32)).astype(np.float32), 32)
    want = 64 * np.mean(-(-((128 + t * 32) * 2) // 4096) * 4096)
    assert bw.bytes_per_query_from_manifest(m, 64) == pytest.approx(want)
    assert bw.bytes_per_query_from_manifest(m, 64, block=1) == pytest.approx(64 * np.mean((128 + t * 32) * 2))


def test_predict_tiered_step():
    pcie = bw.TierProfile("pcie", 50e9, 1)
    on = bw.predict_tiered_step(100e-6, 6.8e6, pcie, prefetch=True)
    off = bw.predict_tiered_step(100e-6, 6.8e6, pcie, prefetch=False)
    assert on["step_s"] == pytest.approx(136e-6) and on["bound"] == "transfer"
    assert off["step_s"] == pytest.approx(236e-6)
    assert bw.predict_tiered_step(200e-6, 6.8e6, pcie, True)["bound"] == "compute"


def test_load_profile(tmp_path):
    p = tmp_path / "p.json"
    p.write_text(json.dumps({"bandwidth_bytes_per_sec": 2e9, "block_size": 4096,
                             "ann_time_table": [[0, 0.0], [2000, 0.03]]}))
    tier, table = bw.load_profile(p)
    assert tier.bandwidth_bytes_per_sec == 2e9 and table(1000) == pytest.approx(0.015)
    p.write_text("{}")
    with pytest.raises(api.InvalidInputError):
        bw.load_profile(p)
