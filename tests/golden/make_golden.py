"""Generates the committed golden fixtures under tests/golden/.

Run in the build container (needs /root/reference for the codec leg):

    make -C oracle ref && python tests/golden/make_golden.py

half_ref_codec.npz -- the reference's own fp16 codec (proj/include/espn/half.hpp:
  11-76, compiled unmodified into oracle/_ref/libref_half.so):
  * decode of all 65,536 codes (as fp32 bit patterns)
  * encode of a fixed float sweep (boundaries, subnormal range, overflow,
    inf/nan, 20,000 seeded randoms)
spec_kats.json -- SPEC.md's known-answer examples for the hot path plus the
  seeded "4x8 query vs 7x8 doc" MaxSim case evaluated with an
  independent pure-Python double loop in fp32 (numpy float32 scalars).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))

import oracle_py  # noqa: E402


def float_sweep() -> np.ndarray:
    special = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, 65536.0, 1e30, -1e30,
                        6.103515625e-05, 6.0975552e-05, 5.9604645e-08, 2.9802322e-08, 2.98023259e-08,
                        3e-8, 1e-7, 1e-5, 3.0517578e-05, 0.1, 0.333333, np.inf, -np.inf, np.nan,
                        1.0009765625, 1.00048828125, 1.000732421875, 2049.0, 2051.0], np.float32)
    rng = np.random.default_rng(2024)
    mags = np.exp(rng.uniform(np.log(1e-9), np.log(7e4), 20000)).astype(np.float32)
    signs = np.where(rng.random(20000) < 0.5, -1.0, 1.0).astype(np.float32)
    return np.concatenate([special, mags * signs]).astype(np.float32)


def make_codec():
    ref = oracle_py.ref_half()
    if ref is None:
        raise SystemExit("oracle/_ref/libref_half.so missing: run `make -C oracle ref` here first")
    codes = np.arange(65536, dtype=np.uint32)
    dec = np.array([ref.ref_half_to_float_bits(int(c)) for c in codes], np.uint32)
    xs = float_sweep()
    enc = np.array([ref.ref_float_bits_to_half(int(b)) for b in xs.view(np.uint32)], np.uint16)
    np.savez_compressed(HERE / "half_ref_codec.npz", decode_bits=dec, sweep=xs, encode=enc)


def brute_maxsim(q: np.ndarray, d: np.ndarray) -> np.float32:
    """Independent double-loop oracle: fp32 scalars, dot over k
    ascending, max over doc tokens, sum over query tokens ascending."""
    s = np.float32(0.0)
    for i in range(q.shape[0]):
        best = None
        for j in range(d.shape[0]):
            acc = np.float32(0.0)
            for k in range(q.shape[1]):
                acc = np.float32(acc + np.float32(q[i, k] * d[j, k]))
            if best is None or acc > best:
                best = acc
        s = np.float32(s + best)
    return s


def make_kats():
    rng = np.random.default_rng(42)
    q = rng.standard_normal((4, 8)).astype(np.float32)
    d = rng.standard_normal((7, 8)).astype(np.float32)
    pairs = []
    rng2 = np.random.default_rng(1)
    for _ in range(200):  # acceptance criterion 1: 200 random pairs up to 16 tokens
        nq, t, dim = int(rng2.integers(1, 17)), int(rng2.integers(1, 17)), int(rng2.integers(1, 17))
        a = rng2.standard_normal((nq, dim)).astype(np.float32)
        b = rng2.standard_normal((t, dim)).astype(np.float32)
        pairs.append({"q": a.tolist(), "d": b.tolist(), "score_bits": int(brute_maxsim(a, b).view(np.uint32))})
    kats = {
        "maxsim": [
            {"q": [[1, 0]], "d": [[1, 0]], "score": 1.0, "src": "SPEC.md:50"},
            {"q": [[1, 0], [0, 1]], "d": [[0, 1], [1, 0]], "score": 2.0, "src": "SPEC.md:51"},
            {"q": q.tolist(), "d": d.tolist(), "score_bits": int(brute_maxsim(q, d).view(np.uint32)),
             "src": "SPEC.md:52 (seed 42, numpy default_rng)"},
        ],
        "maxsim_random_pairs": pairs,
        "aggregate": [
            {"cls": 2.0, "bow": 3.0, "alpha": 0.0, "score": 3.0, "src": "SPEC.md:59"},
            {"cls": 2.0, "bow": 0.0, "alpha": 1.0, "score": 2.0, "src": "SPEC.md:60"},
            {"cls": 1.5, "bow": 4.0, "alpha": 0.5, "score": 4.75, "src": "SPEC.md:61"},
        ],
        "rank": [
            {"in": [[3, 1.0], [1, 2.0]], "out": [[1, 2.0], [3, 1.0]], "src": "SPEC.md:68"},
            {"in": [[2, 1.0], [1, 1.0]], "out": [[1, 1.0], [2, 1.0]], "src": "SPEC.md:69"},
        ],
        "record_bytes": [{"d_cls": 128, "d": 32, "t": 10, "width": 2, "bytes": 896, "src": "SPEC.md:216"}],
    }
    (HERE / "spec_kats.json").write_text(json.dumps(kats))


if __name__ == "__main__":
    make_codec()
    make_kats()
    print("wrote", HERE / "half_ref_codec.npz", HERE / "spec_kats.json")
