"""Seeded synthetic MS-MARCO-shaped inputs.

Host-side (numpy) generator for tests and the CPU baseline; the bench builds
multi-GB tables on the device with espn_gpu_synth_table instead (same shape
law, counter-based RNG).

  * doc token rows: i.i.d. N(0,1), L2-normalised per row, rounded to the
    table dtype with subnormals flushed;
  * t ~ U{t_min..t_max} per doc;
  * queries: perturbed copies (sigma) of a sampled source doc's rows,
    resampled to q tokens, normalised;
  * candidates: the source doc plus K-1 distinct uniform ids, cls scores in
    (0, 1) sorted (cls desc, id asc) as ivf.hpp:45-46 requires.
"""
from __future__ import annotations

import numpy as np

from .api import decode, encode


def flush_subnormals(codes: np.ndarray, dtype: str) -> np.ndarray:
    codes = codes.copy()
    if dtype in ("f16", "fp16"):
        sub = (codes & 0x7C00) == 0
    else:
        sub = (codes & 0x7F80) == 0
    codes[sub] &= 0x8000
    return codes


def make_table(n_docs: int, d: int, t_min: int, t_max: int, dtype: str = "f16", seed: int = 42):
    rng = np.random.default_rng(seed)
    t = rng.integers(t_min, t_max + 1, size=n_docs, dtype=np.int64)
    row_ptr = np.zeros(n_docs + 1, np.uint64)
    row_ptr[1:] = np.cumsum(t)
    n_tok = int(row_ptr[-1])
    x = rng.standard_normal((n_tok, d), dtype=np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    codes = flush_subnormals(encode(x.ravel(), dtype), dtype)
    return row_ptr, codes


def make_queries(row_ptr, codes, d: int, n_queries: int, nq: int = 32, dtype: str = "f16",
                 sigma: float = 0.1, seed: int = 7):
    """Returns (q fp32 [B, nq, d], source doc ids [B])."""
    rng = np.random.default_rng(seed)
    n_docs = row_ptr.shape[0] - 1
    src = rng.integers(0, n_docs, size=n_queries)
    q = np.empty((n_queries, nq, d), np.float32)
    for b, s in enumerate(src):
        a, e = int(row_ptr[s]), int(row_ptr[s + 1])
        rows = decode(codes[a * d:e * d], dtype).reshape(e - a, d)
        pick = rng.integers(0, e - a, size=nq)
        v = rows[pick] + sigma * rng.standard_normal((nq, d), dtype=np.float32)
        q[b] = v / np.linalg.norm(v, axis=1, keepdims=True)
    return q, src


# ---- host mirror of espn_gpu_synth_table (kernels_misc.cuh synth_*) -----------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def device_lengths(gids, t_min: int, t_max: int, seed: int) -> np.ndarray:
    """Token counts the device generator gives global docs `gids` (exact)."""
    g = np.asarray(gids, np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) ^ (g * np.uint64(0xD1B54A32D192ED03)))
    return (np.uint64(t_min) + h % np.uint64(t_max - t_min + 1)).astype(np.int64)


def device_rows(gid: int, t: int, d: int, seed: int, dtype: str = "f16") -> np.ndarray:
    """Token rows (fp32 after dtype rounding) of global doc `gid` as the device
    generator writes them, up to float rounding of log/sincos (<= 1 ulp)."""
    rseed = splitmix64(np.asarray([np.uint64(seed) ^ np.uint64(0x5EED)]))[0]
    with np.errstate(over="ignore"):
        base = splitmix64(np.asarray([rseed ^ (np.uint64(gid) * np.uint64(0x9E3779B97F4A7C15))]))[0]
        j = np.arange(t, dtype=np.uint64)[:, None]
        k = np.arange(0, d, 2, dtype=np.uint64)[None, :]
        h = splitmix64(base + (j << np.uint64(16)) + k)
    u1 = (((h >> np.uint64(40)).astype(np.float64) + 1.0) * (1.0 / 16777217.0)).astype(np.float32)
    u2 = ((h & np.uint64(0xFFFFFF)).astype(np.float64) * (1.0 / 16777216.0)).astype(np.float32)
    rad = np.sqrt(-2.0 * np.log(u1.astype(np.float64)))
    ang = np.pi * (2.0 * u2.astype(np.float64))
    v = np.empty((t, d), np.float32)
    v[:, 0::2] = rad * np.cos(ang)
    v[:, 1::2] = rad * np.sin(ang)
    v /= np.sqrt((v.astype(np.float64) ** 2).sum(axis=1, keepdims=True)).astype(np.float32)
    codes = flush_subnormals(encode(v.ravel(), dtype), dtype)
    return decode(codes, dtype).reshape(t, d)


def make_candidates(n_docs: int, n_queries: int, k: int, src=None, seed: int = 11):
    """CSR candidate lists: (ids u32, cls f32, offsets u64)."""
    rng = np.random.default_rng(seed)
    k = min(k, n_docs)
    ids = np.empty((n_queries, k), np.uint32)
    cls = np.empty((n_queries, k), np.float32)
    for b in range(n_queries):
        if n_docs <= 4 * k:
            c = rng.permutation(n_docs)[:k]
        else:
            c = np.unique(rng.integers(0, n_docs, size=int(k * 1.2) + 16))
            c = rng.permutation(c)[:k]
            while c.size < k:
                extra = np.setdiff1d(np.unique(rng.integers(0, n_docs, size=k)), c)
                c = np.concatenate([c, extra])[:k]
        if src is not None and src[b] not in c:
            c[0] = src[b]
        s = rng.random(k, dtype=np.float32)
        if src is not None:
            s[c == src[b]] = 1.0
        order = np.lexsort((c, -s))  # cls desc, id asc
        ids[b] = c[order]
        cls[b] = s[order]
    off = np.arange(n_queries + 1, dtype=np.uint64) * k
    return ids.ravel(), cls.ravel(), off


# ---- host mirror of the HBM tile layout (common.cuh RowLayout) ----------------
def tile_chunk_offsets(t: int, d: int) -> np.ndarray:
    """[t, 2d/16] byte offsets, inside a doc of t rows, of each 16-byte chunk of
    each plain row in the HBM tile layout (identity for non-tensor-core dims)."""
    rowb = 2 * d
    ch = rowb // 16
    j = np.arange(t, dtype=np.int64)[:, None]
    c = np.arange(ch, dtype=np.int64)[None, :]
    if d not in (16, 32, 64, 128):
        return j * rowb + c * 16
    pw = min(rowb, 128)
    cpp = pw // 16
    p, cc = c // cpp, c % cpp
    sw = ((j * pw) >> 7) & (cpp - 1)
    return (p * t + j) * pw + ((cc ^ sw) << 4)


def untile_rows(row_ptr, tiled_codes, d: int) -> np.ndarray:
    """HBM tile layout -> plain row-major codes (test helper)."""
    b = np.asarray(tiled_codes, np.uint16).view(np.uint8)
    out = np.empty_like(b)
    rp = np.asarray(row_ptr, np.int64)
    rowb = 2 * d
    for i in range(rp.shape[0] - 1):
        a, t = int(rp[i]) * rowb, int(rp[i + 1] - rp[i])
        off = tile_chunk_offsets(t, d).ravel()
        chunks = np.stack([b[a + o:a + o + 16] for o in off]) if t else np.zeros((0, 16), np.uint8)
        out[a:a + t * rowb] = chunks.ravel()
    return out.view(np.uint16)
