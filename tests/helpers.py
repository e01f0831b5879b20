"""Shared helpers for the parity tests (tolerances are the north_star's)."""
from __future__ import annotations

import numpy as np

# MaxSim scores within 1e-3 relative for fp16/bf16 inputs (BASELINE.json
# north_star); |ref| is floored at 1.0 so near-zero scores use 1e-3 absolute.
RTOL = 1e-3
# "Ties" for the top-k order exemption: |a-b| <= 1e-3*max(|a|,|b|)
TIE_RTOL = 1e-3


def rel_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)


def oracle_full_scores(bow, cls, alpha, n_needed, partial):
    """aggregate_score over a query's candidates (scoring.hpp:12-14)."""
    s = np.float32(alpha) * cls.astype(np.float32)
    s = s.astype(np.float32)
    out = s.copy()
    out[:n_needed] = (s[:n_needed] + bow[:n_needed].astype(np.float32)).astype(np.float32)
    if not partial:
        out = out[:n_needed]
    return out


def assert_topk_equivalent(ids_g, sc_g, ids_o, sc_o, cand_ids, cand_scores_oracle, ctx=""):
    """Order identical except at stated ties: at every rank position the GPU's
    doc must carry (by the oracle's own scoring) the oracle's score at that
    position up to TIE_RTOL, and the GPU score must be within RTOL."""
    assert len(ids_g) == len(ids_o), f"{ctx}: count {len(ids_g)} != {len(ids_o)}"
    pos = {int(i): j for j, i in enumerate(cand_ids)}
    for r, (ig, io) in enumerate(zip(ids_g, ids_o)):
        so = float(sc_o[r])
        assert abs(float(sc_g[r]) - so) <= RTOL * max(abs(so), 1.0), f"{ctx}: rank {r} score {sc_g[r]} vs {so}"
        if int(ig) != int(io):
            assert int(ig) in pos, f"{ctx}: rank {r}: GPU returned non-candidate {ig}"
            s_of_g = float(cand_scores_oracle[pos[int(ig)]])
            assert abs(s_of_g - so) <= TIE_RTOL * max(abs(s_of_g), abs(so), 1e-6), (
                f"{ctx}: rank {r}: id {ig} (oracle score {s_of_g}) vs oracle id {io} ({so}) is not a tie")
    assert len(set(int(i) for i in ids_g)) == len(ids_g), f"{ctx}: duplicate ids in GPU top-k"
