"""Bandwidth model (PAPER §4.2 Eq. 2-4, §1).

The paper's capacity-planning calculators, re-parameterised for the B200
tiers: the "SSD" of Eq. 4 becomes whichever tier the missed rows come from
(HBM, pinned host over PCIe, NVMe), fed with MEASURED bandwidths, and the
prefetch budget of Eq. 2 becomes the device time the prefetch hides behind.
bench.py --config c4 uses predict_tiered_step() to predict the tiered step
time from the measured PCIe bandwidth and the measured scoring time, and
reports prediction vs measurement.

Pure host arithmetic (no device): calculators, not part of the re-rank path.
"""
from __future__ import annotations

import bisect
import json
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

from .api import InvalidInputError


@dataclass
class TierProfile:
    """SsdProfile for any tier: bytes/s of random reads at
    `block_size` granularity."""
    name: str = "ssd"
    bandwidth_bytes_per_sec: float = 2e9
    block_size: int = 4096

    def __post_init__(self):
        if not (self.bandwidth_bytes_per_sec > 0 and self.block_size > 0):
            raise InvalidInputError("tier bandwidth and block size must be positive (SPEC.md:330)")


@dataclass
class AnnTimeTable:
    """ANNSearchTime(nprobe) as measured points, linearly interpolated
    (SPEC.md:333-335, 381)."""
    points: List[Tuple[int, float]] = field(default_factory=list)

    def __post_init__(self):
        self.points = sorted((int(n), float(t)) for n, t in self.points)
        if not self.points:
            raise InvalidInputError("ann_time table is empty")
        ts = [t for _, t in self.points]
        if any(b < a for a, b in zip(ts, ts[1:])):
            raise InvalidInputError("ann_time must be nondecreasing in nprobe (SPEC.md:334)")

    @classmethod
    def linear(cls, seconds_per_probe: float, max_nprobe: int) -> "AnnTimeTable":
        return cls([(0, 0.0), (max_nprobe, seconds_per_probe * max_nprobe)])

    def __call__(self, nprobe: float) -> float:
        xs = [n for n, _ in self.points]
        if not (xs[0] <= nprobe <= xs[-1]):
            raise InvalidInputError(f"ann_time undefined at nprobe={nprobe} (table covers [{xs[0]}, {xs[-1]}])")
        i = bisect.bisect_left(xs, nprobe)
        if xs[i] == nprobe:
            return self.points[i][1]
        (x0, y0), (x1, y1) = self.points[i - 1], self.points[i]
        return y0 + (y1 - y0) * (nprobe - x0) / (x1 - x0)


def prefetch_budget(ann_time: AnnTimeTable, eta: int, delta: int) -> float:
    """Eq. 2: ANNSearchTime(eta) - ANNSearchTime(delta) seconds."""
    if delta > eta:
        raise InvalidInputError("delta must be <= eta (SPEC.md:343)")
    return ann_time(eta) - ann_time(delta)


def prefetch_step(delta: int, eta: int) -> float:
    """Eq. 3: delta / eta * 100 percent."""
    if not (1 <= delta <= eta):
        raise InvalidInputError("need 1 <= delta <= eta (SPEC.md:351)")
    return delta / eta * 100.0


def batch_threshold(profile: TierProfile, budget_s: float, bytes_per_query: float) -> float:
    """Eq. 4: BW * budget / bytes_per_query, fractional:
    the largest batch whose misses the tier can deliver within the budget."""
    if bytes_per_query <= 0:
        raise InvalidInputError("bytes_per_query must be positive (SPEC.md:361)")
    if budget_s < 0:
        raise InvalidInputError("budget must be nonnegative")
    return profile.bandwidth_bytes_per_sec * budget_s / bytes_per_query


def index_size_estimate(n_docs: float, t_avg: float, d: int, b: int, cls_bytes_per_doc: float):
    """O(NI + Ntdb) (PAPER §1): (candidate-gen bytes N*I,
    re-rank bytes N*t*d*b, total)."""
    cg = n_docs * cls_bytes_per_doc
    rr = n_docs * t_avg * d * b
    return cg, rr, cg + rr


def bytes_per_query(record_bytes: Sequence[int], R: int, alignment: int = 1) -> float:
    """Default Eq. 4 input: R x mean(record bytes rounded up to
    the tier's alignment / block)."""
    if not len(record_bytes):
        raise InvalidInputError("no records")
    if alignment < 1:
        raise InvalidInputError("alignment must be >= 1")
    rounded = [-(-int(x) // alignment) * alignment for x in record_bytes]
    return R * sum(rounded) / len(rounded)


def bytes_per_query_from_manifest(manifest, R: int, block: int = 0) -> float:
    """bytes_per_query from a .espn manifest (api.load_manifest), blocks of
    `block` bytes (default the store's alignment)."""
    return bytes_per_query(manifest.records["byte_length"].tolist(), R, block or manifest.alignment)


def predict_tiered_step(compute_s: float, miss_bytes: float, tier: TierProfile, prefetch: bool) -> dict:
    """Step time of one batch whose missed rows (`miss_bytes` in total) come
    from `tier`: with the prefetcher the transfer of batch n+1 overlaps batch
    n's scoring (step = max), without it the transfer sits on the critical
    path (step = sum).  Eq. 4's threshold at this batch = budget/transfer."""
    xfer = miss_bytes / tier.bandwidth_bytes_per_sec
    step = max(compute_s, xfer) if prefetch else compute_s + xfer
    return {"step_s": step, "transfer_s": xfer, "compute_s": compute_s,
            "bound": ("transfer" if xfer > compute_s else "compute") if prefetch else "serial",
            "hidden_fraction": min(1.0, compute_s / xfer) if xfer > 0 else 1.0}


def load_profile(path) -> Tuple[TierProfile, AnnTimeTable]:
    """JSON profile {bandwidth_bytes_per_sec, block_size, ann_time_table:
    [[nprobe, seconds], ...]}."""
    try:
        with open(path) as f:
            j = json.load(f)
        tier = TierProfile(j.get("name", "ssd"), float(j["bandwidth_bytes_per_sec"]), int(j["block_size"]))
        table = AnnTimeTable([tuple(p) for p in j["ann_time_table"]])
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidInputError(f"bad bandwidth profile {path}: {e}") from None
    return tier, table
