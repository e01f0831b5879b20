"""IVF candidate generator with a staged cursor (ivf.hpp:10-86)
-- the source of the prefetch hints of SURVEY.md §8 f1.

This is the UPSTREAM producer of the re-rank path, restated on the host
(numpy/BLAS) as the paper runs it (ANN on the CPU while the prefetcher moves
embeddings to the GPU, PAPER §4.2).  Its role here is to emit, per query, the
snapshot after delta clusters (the prefetch hints fed to
espn_gpu_prefetch_hints) and the final candidate list (fed to
espn_gpu_rerank).  Inner products use BLAS, so cls scores may differ from the
reference's ascending-order dot_f32 in the last bits (they are float64 sums
rounded once to fp32); the re-rank path takes the cls scores it is given, so
this does not affect parity of the path.

  * train_ivf: k-means++ seeding + Lloyd iterations (L2) on a seeded sample
    of at most `sample_per_list` x nlist vectors, then every vector goes to
    its nearest centroid's list (deterministic for a seed);
  * begin_search: plan = the nprobe centroids by descending inner product
    (ties by centroid index);
  * SearchCursor.advance / snapshot / finish: bounded top-K by (score desc,
    doc_id asc), as ivf.hpp:52-81;
  * save_ivf / load_ivf: "ESPNIVF1" single file, little-endian (ivf.hpp:35-38).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import List

import numpy as np

from .api import Candidate, CandidateList, FormatError, InvalidInputError, InvalidStateError, IoError


@dataclass
class IvfIndex:
    """ivf.hpp:10-28, lists stored as one CSR (list_off, ids, vectors)."""
    d_cls: int
    centroids: np.ndarray   # nlist x d_cls f32
    list_off: np.ndarray    # nlist + 1 u64
    ids: np.ndarray         # N u32, grouped by list
    vectors: np.ndarray     # N x d_cls f32, same order

    def nlist(self) -> int:
        return int(self.centroids.shape[0])

    def size(self) -> int:
        return int(self.ids.shape[0])

    def list_ids(self, c: int) -> np.ndarray:
        return self.ids[int(self.list_off[c]):int(self.list_off[c + 1])]


def _sq_dists(x: np.ndarray, c: np.ndarray) -> np.ndarray:
    return (x * x).sum(1)[:, None] - 2.0 * (x @ c.T) + (c * c).sum(1)[None, :]


def _nearest(x: np.ndarray, c: np.ndarray, chunk: int = 65536) -> np.ndarray:
    out = np.empty(x.shape[0], np.int64)
    cn = (c * c).sum(1)[None, :]
    for i in range(0, x.shape[0], chunk):
        xb = x[i:i + chunk]
        out[i:i + chunk] = np.argmin(cn - 2.0 * (xb @ c.T), axis=1)  # |x|^2 is constant per row
    return out


def train_ivf(vectors: np.ndarray, nlist: int, max_iters: int = 20, seed: int = 0,
              sample_per_list: int = 64, seed_per_list: int = 16) -> IvfIndex:
    """train_ivf (ivf.hpp:30-33)."""
    x = np.ascontiguousarray(vectors, dtype=np.float32)
    if x.ndim != 2 or nlist < 1 or x.shape[0] < nlist:
        raise InvalidInputError("train_ivf needs at least nlist vectors (SPEC.md:155)")
    if max_iters < 1:
        raise InvalidInputError("max_iters must be >= 1")
    if not np.all(np.isfinite(x)):
        raise InvalidInputError("non-finite CLS vector")
    n, d = x.shape
    rng = np.random.default_rng(seed)
    s = x if n <= sample_per_list * nlist else x[np.sort(rng.choice(n, sample_per_list * nlist, replace=False))]
    # k-means++ seeding on a sub-sample of <= seed_per_list x nlist vectors
    # (distances as |s|^2 - 2 s.c + |c|^2, one BLAS GEMV per centroid)
    ss = s if s.shape[0] <= seed_per_list * nlist else s[np.sort(rng.choice(s.shape[0], seed_per_list * nlist,
                                                                             replace=False))]
    sn = (ss * ss).sum(1)
    c = np.empty((nlist, d), np.float32)
    c[0] = ss[rng.integers(ss.shape[0])]
    dmin = np.maximum(sn - 2.0 * (ss @ c[0]) + float(c[0] @ c[0]), 0.0)
    for i in range(1, nlist):
        tot = float(dmin.sum(dtype=np.float64))
        if tot > 0:
            j = int(np.searchsorted(np.cumsum(dmin, dtype=np.float64), rng.random() * tot, side="right"))
            j = min(j, ss.shape[0] - 1)
        else:
            j = int(rng.integers(ss.shape[0]))
        c[i] = ss[j]
        np.minimum(dmin, np.maximum(sn - 2.0 * (ss @ c[i]) + float(c[i] @ c[i]), 0.0), out=dmin)
    # Lloyd
    assign = _nearest(s, c)
    for _ in range(max_iters):
        sums = np.zeros((nlist, d), np.float64)
        np.add.at(sums, assign, s)
        cnt = np.bincount(assign, minlength=nlist)
        nz = cnt > 0
        c[nz] = (sums[nz] / cnt[nz, None]).astype(np.float32)
        new = _nearest(s, c)
        if np.array_equal(new, assign):
            break
        assign = new
    a = _nearest(x, c)
    order = np.argsort(a, kind="stable")
    off = np.zeros(nlist + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(a, minlength=nlist))
    return IvfIndex(d, c, off, order.astype(np.uint32), x[order])


def _ip(vecs: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Inner products accumulated in float64 and rounded once to fp32: the
    same value whatever BLAS blocking or segment split computes it, so the
    cursor's candidates are reproducible and match an exhaustive oracle
    computed the same way (SPEC acceptance #2)."""
    return (vecs.astype(np.float64) @ q.astype(np.float64)).astype(np.float32)


def _top(ids: np.ndarray, scores: np.ndarray, k: int):
    o = np.lexsort((ids, -scores))[:k]  # score desc, doc_id asc (ivf.hpp:45-46)
    return ids[o], scores[o]


class SearchCursor:
    """ivf.hpp:52-81: fixed visitation plan, bounded top-K."""

    def __init__(self, index: IvfIndex, query_cls, nprobe: int, k: int):
        if not (1 <= nprobe <= index.nlist()):
            raise InvalidInputError(f"nprobe {nprobe} outside [1, nlist={index.nlist()}] (SPEC.md:164)")
        if k < 1:
            raise InvalidInputError("k must be >= 1")
        self.index = index
        self.query = np.ascontiguousarray(query_cls, dtype=np.float32).reshape(-1)
        if self.query.shape[0] != index.d_cls:
            raise InvalidInputError("query CLS dimension mismatch")
        cs = index.centroids @ self.query
        self.plan = np.lexsort((np.arange(cs.shape[0]), -cs))[:nprobe]
        self.visited = 0
        self.capacity = int(k)
        self._ids = np.zeros(0, np.uint32)
        self._scores = np.zeros(0, np.float32)

    def nprobe(self) -> int:
        return int(self.plan.shape[0])

    def clusters_visited(self) -> int:
        return self.visited

    def advance(self, n_clusters: int) -> None:
        if n_clusters < 0 or self.visited + n_clusters > self.nprobe():
            raise InvalidInputError("advance past nprobe (SPEC.md:172)")
        if n_clusters == 0:
            return
        ix = self.index
        segs = [(int(ix.list_off[c]), int(ix.list_off[c + 1])) for c in self.plan[self.visited:self.visited + n_clusters]]
        self.visited += n_clusters
        ids = np.concatenate([self._ids] + [ix.ids[a:b] for a, b in segs])
        sc = np.concatenate([self._scores] + [_ip(ix.vectors[a:b], self.query) for a, b in segs]).astype(np.float32)
        self._ids, self._scores = _top(ids, sc, self.capacity)

    def snapshot(self, top_k: int) -> CandidateList:
        if top_k < 1:
            raise InvalidInputError("top_k must be >= 1")
        return _to_list(self._ids[:top_k], self._scores[:top_k], self.visited)

    def finish(self, k: int) -> CandidateList:
        if self.visited != self.nprobe():
            raise InvalidStateError("finish before the cursor is fully advanced (SPEC.md:186)")
        return _to_list(self._ids[:k], self._scores[:k], self.visited)

    # array forms (no per-candidate Python objects) for the batch driver
    def snapshot_arrays(self, top_k: int):
        return self._ids[:top_k], self._scores[:top_k]

    def finish_arrays(self, k: int):
        if self.visited != self.nprobe():
            raise InvalidStateError("finish before the cursor is fully advanced (SPEC.md:186)")
        return self._ids[:k], self._scores[:k]


def _to_list(ids, scores, visited) -> CandidateList:
    return CandidateList([Candidate(int(i), float(s)) for i, s in zip(ids, scores)], clusters_visited=visited)


def begin_search(index: IvfIndex, query_cls, nprobe: int, k: int) -> SearchCursor:
    """ivf.hpp:83-86."""
    return SearchCursor(index, query_cls, nprobe, k)


_IVF_HDR = struct.Struct("<8sIIQ")  # magic, version, d_cls, nlist


def save_ivf(index: IvfIndex, path) -> None:
    """ESPNIVF1: header, centroid block, per list (u64 length, u32 ids, f32 vectors)."""
    try:
        with open(path, "wb") as f:
            f.write(_IVF_HDR.pack(b"ESPNIVF1", 1, index.d_cls, index.nlist()))
            f.write(np.ascontiguousarray(index.centroids, "<f4").tobytes())
            for c in range(index.nlist()):
                a, b = int(index.list_off[c]), int(index.list_off[c + 1])
                f.write(struct.pack("<Q", b - a))
                f.write(np.ascontiguousarray(index.ids[a:b], "<u4").tobytes())
                f.write(np.ascontiguousarray(index.vectors[a:b], "<f4").tobytes())
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from None


def load_ivf(path) -> IvfIndex:
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from None
    if len(raw) < _IVF_HDR.size:
        raise FormatError("truncated IVF header")
    magic, ver, d, nlist = _IVF_HDR.unpack_from(raw)
    if magic != b"ESPNIVF1" or ver != 1 or d == 0 or nlist == 0:
        raise FormatError("not an ESPNIVF1 file")
    p = _IVF_HDR.size
    need = nlist * d * 4
    if len(raw) < p + need:
        raise FormatError("truncated centroid block")
    cent = np.frombuffer(raw, "<f4", nlist * d, p).reshape(nlist, d).copy()
    p += need
    ids: List[np.ndarray] = []
    vecs: List[np.ndarray] = []
    off = np.zeros(nlist + 1, np.uint64)
    for c in range(nlist):
        if len(raw) < p + 8:
            raise FormatError("truncated list header")
        (n,) = struct.unpack_from("<Q", raw, p)
        p += 8
        if len(raw) < p + n * 4 * (1 + d):
            raise FormatError("truncated list block")
        ids.append(np.frombuffer(raw, "<u4", n, p).copy())
        p += n * 4
        vecs.append(np.frombuffer(raw, "<f4", n * d, p).reshape(n, d).copy())
        p += n * d * 4
        off[c + 1] = off[c] + n
    if p != len(raw):
        raise FormatError("trailing bytes after the last list")
    return IvfIndex(int(d), cent, off, np.concatenate(ids).astype(np.uint32),
                    np.concatenate(vecs).astype(np.float32).reshape(-1, d))
