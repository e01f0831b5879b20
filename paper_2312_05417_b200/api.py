"""Reference-shaped host API over the C-ABI (include/espn_gpu.h).

Mirrors the re-rank slice of the reference's C++ interface -- names, fields,
argument meaning and error classes -- so code written against
proj/include/espn/{types,error,scoring,store,pipeline}.hpp maps 1:1:

  reference (proj/include/espn/)                 here
  ---------------------------------------------  -----------------------------------
  error.hpp:8-42   Error + 6 subclasses           Error, InvalidInputError, ...
  types.hpp:14-55  EmbeddingMatrix, QueryEmbedding, ScoredDoc, RankedList
  ivf.hpp:40-50    Candidate, CandidateList       Candidate, CandidateList
  pipeline.hpp:11-29 PipelineConfig               PipelineConfig (same fields/defaults)
  pipeline.hpp:36-54 QueryStats                   QueryStats (same fields)
  pipeline.hpp:66-79 BatchStats, BatchResult      BatchStats, BatchResult
  store.hpp:80-112 StoreHandle / open_store       GpuStore (HBM tier of the table)
  store.hpp:94     fetch_batch                    GpuStore.fetch_batch (K1 gather)
  pipeline.hpp:61  run_query stages 3-6           rerank_candidates (the new seam)
  pipeline.hpp:83  run_batch                      rerank_batch

All compute runs in libespn_gpu.so; this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L


# ---- error.hpp:8-42 ---------------------------------------------------------
class Error(RuntimeError):
    """Base class for every error the engine reports (error.hpp:9-12)."""


class InvalidInputError(Error):
    pass


class InvalidStateError(Error):
    pass


class InvalidConfigError(Error):
    pass


class FormatError(Error):
    pass


class IoError(Error):
    pass


class DataIntegrityError(Error):
    pass


_STATUS = {
    L.ESPN_E_INVALID_INPUT: InvalidInputError,
    L.ESPN_E_INVALID_STATE: InvalidStateError,
    L.ESPN_E_INVALID_CONFIG: InvalidConfigError,
    L.ESPN_E_FORMAT: FormatError,
    L.ESPN_E_IO: IoError,
    L.ESPN_E_DATA_INTEGRITY: DataIntegrityError,
    L.ESPN_E_CUDA: Error,
}


def _check(rc: int) -> None:
    if rc != L.ESPN_OK:
        raise _STATUS.get(rc, Error)(L.last_error())


def _check_store(rc: int) -> None:
    if rc != L.ESPN_OK:
        raise _STATUS.get(rc, Error)(L.store_last_error())


# ---- the on-disk store (store.hpp:37-54, include/espn_store.h) ---------------------
@dataclass
class StoreManifest:
    """store.hpp:20-35 (records as a numpy structured array)."""
    version: int
    d: int
    d_cls: int
    value_width: int
    alignment: int
    records: np.ndarray  # dtype [("byte_offset", u8), ("byte_length", u4), ("token_count", u4)]

    def count(self) -> int:
        return int(self.records.shape[0])

    def record_bytes(self, token_count):
        return (self.d_cls + np.asarray(token_count, dtype=np.uint64) * self.d) * self.value_width


_RECORD_DT = np.dtype([("byte_offset", "<u8"), ("byte_length", "<u4"), ("token_count", "<u4")])


def build_store(base, row_ptr, rows, d: int, d_cls: int = 128, value_width: int = 2, alignment: int = 4096,
                cls=None) -> StoreManifest:
    """build_store (store.hpp:48-51): <base>.espn + <base>.manifest + .manifest.json
    from a CSR of fp32 token rows (and optional n_docs x d_cls CLS vectors)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    rows = np.ascontiguousarray(rows, dtype=np.float32)
    n = int(row_ptr.shape[0]) - 1
    if n < 0 or (n and int(row_ptr[0]) != 0) or np.any(np.diff(row_ptr.astype(np.int64)) < 0):
        raise InvalidInputError("row_ptr must start at 0 and be non-decreasing")
    if rows.size < int(row_ptr[-1]) * int(d):
        raise InvalidInputError("rows hold fewer than row_ptr[n] * d values")
    cls_a = None if cls is None else np.ascontiguousarray(cls, dtype=np.float32)
    if cls_a is not None and cls_a.size < n * int(d_cls):
        raise InvalidInputError("cls holds fewer than n_docs * d_cls values")
    _check_store(L.store_lib().espn_store_build(str(base).encode(), n, int(d), int(d_cls), int(value_width),
                                                int(alignment), row_ptr.ctypes.data, rows.ctypes.data,
                                                cls_a.ctypes.data if cls_a is not None else None))
    return load_manifest(base)


def load_manifest(base) -> StoreManifest:
    """load_manifest (store.hpp:54)."""
    h = L.StoreHeader()
    lib = L.store_lib()
    _check_store(lib.espn_store_load_manifest(str(base).encode(), C.byref(h), None))
    recs = np.zeros(int(h.count), _RECORD_DT)
    _check_store(lib.espn_store_load_manifest(str(base).encode(), C.byref(h), recs.ctypes.data if h.count else None))
    return StoreManifest(int(h.version), int(h.d), int(h.d_cls), int(h.value_width), int(h.alignment), recs)


def read_store_table(base, dtype: str = "f16", with_cls: bool = False):
    """Every document's rows as the GPU table's CSR of 2-byte `dtype` codes
    (+ fp32 CLS vectors): (row_ptr, codes, cls or None)."""
    m = load_manifest(base)
    tok = m.records["token_count"].astype(np.uint64)
    row_ptr = np.zeros(m.count() + 1, np.uint64)
    codes = np.empty(max(int(tok.sum()) * m.d, 1), np.uint16)
    cls = np.empty((m.count(), m.d_cls), np.float32) if with_cls else None
    _check_store(L.store_lib().espn_store_read_table(str(base).encode(), _DTYPES[dtype], row_ptr.ctypes.data,
                                                     codes.ctypes.data, cls.ctypes.data if cls is not None else None))
    return row_ptr, codes[: int(row_ptr[-1]) * m.d], cls


class StoreReader:
    """The reference's file-backed StoreHandle (store.hpp:56-112) over
    libespn_store: ReadMode direct (O_DIRECT) / buffered / mmap with
    queue_depth reads in flight -- the host side of the disk tier."""

    _MODES = {"direct": 0, "buffered": 1, "mmap": 2}

    def __init__(self, base, mode: str = "direct", queue_depth: int = 16):
        self._lib = L.store_lib()
        self._h = C.c_void_p()
        self.header = L.StoreHeader()
        _check_store(self._lib.espn_store_open(str(base).encode(), self._MODES[mode], int(queue_depth),
                                               C.byref(self._h), C.byref(self.header)))
        self.d_cls, self.value_width = int(self.header.d_cls), int(self.header.value_width)

    def fetch(self, ids, out=None):
        """Records of ids in request order -> (payload bytes, offsets[n+1],
        {bytes_read, blocks_read, wall_time}) (store.hpp:61-65, 91-94).
        `out`: optional preallocated uint8 buffer (numpy, or a pinned torch
        tensor) large enough for the payloads."""
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        n = ids.shape[0]
        off = np.zeros(n + 1, np.uint64)
        br, bl, wt = C.c_uint64(), C.c_uint64(), C.c_double()
        _check_store(self._lib.espn_store_fetch(self._h, ids.ctypes.data, n, None, off.ctypes.data, 0,
                                                C.byref(br), C.byref(bl), C.byref(wt)))
        need = int(off[-1])
        if out is None:
            out = np.empty(max(need, 1), np.uint8)
        cap = int(out.nbytes) if isinstance(out, np.ndarray) else int(out.numel())
        if cap < need:
            raise InvalidInputError("fetch buffer too small")
        ptr = out.ctypes.data if isinstance(out, np.ndarray) else int(out.data_ptr())
        _check_store(self._lib.espn_store_fetch(self._h, ids.ctypes.data, n, ptr, off.ctypes.data, cap,
                                                C.byref(br), C.byref(bl), C.byref(wt)))
        return out, off, {"bytes_read": br.value, "blocks_read": bl.value, "wall_time": wt.value}

    def row_offsets(self, off):
        """Byte offsets of each fetched record's BOW rows inside the payload
        buffer (the CLS vector comes first: d_cls x value_width bytes)."""
        return np.asarray(off[:-1], np.uint64) + np.uint64(self.d_cls * self.value_width)

    def close(self) -> None:
        if self._h:
            self._lib.espn_store_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- types.hpp / ivf.hpp / pipeline.hpp carriers --------------------------------
@dataclass
class EmbeddingMatrix:
    """types.hpp:16-25: t x d row-major fp32 token embeddings of one doc."""
    doc_id: int = 0
    rows: int = 0
    cols: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))


@dataclass
class QueryEmbedding:
    """types.hpp:34-44: one CLS vector plus a q x d token matrix (fp32)."""
    query_id: int = 0
    cls: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    rows: int = 0
    cols: int = 0
    tokens: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))


@dataclass
class ScoredDoc:
    doc_id: int = 0
    score: float = 0.0


@dataclass
class RankedList:
    """types.hpp:53-55: sorted by (score desc, doc_id asc), no duplicate ids."""
    entries: List[ScoredDoc] = field(default_factory=list)


@dataclass
class Candidate:
    doc_id: int = 0
    cls_score: float = 0.0


@dataclass
class CandidateList:
    """ivf.hpp:47-50: sorted by (cls_score desc, doc_id asc), deduplicated."""
    entries: List[Candidate] = field(default_factory=list)
    clusters_visited: int = 0


@dataclass
class PipelineConfig:
    """pipeline.hpp:11-29 (same fields and defaults)."""
    nprobe: int = 0
    prefetch_step_pct: float = 10.0
    rerank_count: int = 0
    final_k: int = 10
    prefetch_top_k: int = 0
    candidate_k: int = 0
    alpha: float = 1.0
    prefetch_enabled: bool = True
    partial_rerank_enabled: bool = False

    def effective_prefetch_top_k(self) -> int:
        return self.prefetch_top_k or self.rerank_count

    def effective_candidate_k(self) -> int:
        return self.candidate_k or max(self.rerank_count, self.final_k)

    def delta(self) -> int:
        """round(nprobe * step / 100), at least 1 (pipeline.hpp:8-10)."""
        return max(1, int(math.floor(self.nprobe * self.prefetch_step_pct / 100.0 + 0.5)))


@dataclass
class QueryStats:
    """pipeline.hpp:36-54 (same fields)."""
    query_id: int = 0
    ann_time: float = 0.0
    prefetch_time: float = 0.0
    early_rerank_time: float = 0.0
    critical_fetch_time: float = 0.0
    rerank_time: float = 0.0
    total_time: float = 0.0
    prefetched_count: int = 0
    needed_count: int = 0
    missed_count: int = 0
    hit_rate: float = 0.0
    prefetch_bytes: int = 0
    critical_fetch_bytes: int = 0
    critical_blocks_read: int = 0
    needed_payload_bytes: int = 0


@dataclass
class BatchStats:
    n_queries: int = 0
    mean_latency: float = 0.0
    p50_latency: float = 0.0
    p99_latency: float = 0.0
    wall_time: float = 0.0
    total_critical_fetch_bytes: int = 0


@dataclass
class BatchResult:
    rankings: List[RankedList] = field(default_factory=list)
    stats: List[QueryStats] = field(default_factory=list)
    batch: BatchStats = field(default_factory=BatchStats)


@dataclass
class FetchedDoc:
    bow: EmbeddingMatrix


@dataclass
class FetchResult:
    """store.hpp:66-71: docs in request order plus transfer counters."""
    docs: List[FetchedDoc] = field(default_factory=list)
    bytes_read: int = 0
    blocks_read: int = 0
    wall_time: float = 0.0


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


_DTYPES = {"f16": L.ESPN_DTYPE_F16, "fp16": L.ESPN_DTYPE_F16, "bf16": L.ESPN_DTYPE_BF16}
_QPREC = {"auto": 0, "split": L.ESPN_RERANK_QUERY_SPLIT, "rounded": L.ESPN_RERANK_QUERY_ROUNDED}
_KERNELS = {"auto": L.ESPN_KERNEL_AUTO, "tcgen05": L.ESPN_KERNEL_TCGEN05, "simt": L.ESPN_KERNEL_SIMT,
            "small": L.ESPN_KERNEL_SMALL}


class GpuStore:
    """The HBM tier of the embedding table -- the re-rank path's StoreHandle
    (store.hpp:80-107).  Rows are CSR: doc i's token rows are
    rows[row_ptr[i]:row_ptr[i+1]], 2-byte codes of `dtype`.  d_cls /
    value_width / alignment describe the reference's on-disk record and feed
    only the QueryStats byte counters (store.hpp:32-34, 61-65)."""

    def __init__(self, row_ptr, rows, d: int, dtype: str = "f16", d_cls: int = 128,
                 value_width: int = 2, alignment: int = 4096, device: int = 0,
                 borrowed_device: bool = False, shard_count: int = 1, shard_index: int = 0,
                 rows_tiled: bool = False, resident=None, streamed: bool = False, disk_tier: bool = False):
        self.d = int(d)
        self.dtype = dtype
        self.d_cls = int(d_cls)
        self.value_width = int(value_width)
        self.alignment = int(alignment)
        self.device = int(device)
        self._keep = (row_ptr, rows)
        if borrowed_device:
            n_docs = int(row_ptr.numel()) - 1
            self._row_ptr_host = None
            rp_p, rows_p, flags = _ptr(row_ptr), _ptr(rows), L.ESPN_TABLE_DEVICE_BORROWED
            if rows_tiled:
                flags |= L.ESPN_TABLE_ROWS_TILED
        elif streamed:  # ESPN_TABLE_STREAMED: allocated from row_ptr, filled by load_rows
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
            n_docs = int(row_ptr.shape[0]) - 1
            self._row_ptr_host = row_ptr
            self._keep = (row_ptr,)
            rp_p, rows_p, flags = _ptr(row_ptr), None, L.ESPN_TABLE_STREAMED
            if disk_tier:  # non-resident docs stay in the store file (espn_gpu_prefetch_rows)
                flags |= L.ESPN_TABLE_DISK_TIER
        else:
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
            rows = np.ascontiguousarray(rows, dtype=np.uint16)
            n_docs = int(row_ptr.shape[0]) - 1
            self._row_ptr_host = row_ptr
            self._keep = (row_ptr, rows)
            rp_p, rows_p, flags = _ptr(row_ptr), _ptr(rows), 0
        self._resident = None
        if resident is not None:  # tiered store: HBM for resident docs, pinned host for the rest
            self._resident = np.ascontiguousarray(np.asarray(resident, dtype=np.uint8))
            if self._resident.shape[0] != n_docs:
                raise InvalidInputError("resident mask must have one entry per doc")
        desc = L.TableDesc(n_docs=n_docs, d=self.d, dtype=_DTYPES[dtype], d_cls=self.d_cls,
                           value_width=self.value_width, alignment=self.alignment, flags=flags,
                           row_ptr=rp_p, rows=rows_p, device=self.device, shard_count=int(shard_count),
                           shard_index=int(shard_index),
                           resident=self._resident.ctypes.data if self._resident is not None else None)
        self.shard_count = max(int(shard_count), 1)
        self.shard_index = int(shard_index) if self.shard_count > 1 else 0
        h = C.c_void_p()
        _check(L.lib().espn_gpu_table_open(C.byref(desc), C.byref(h)))
        self._h = h
        if not borrowed_device:
            self._keep = None  # uploaded; host copies no longer needed by the library
        info = L.TableInfo()
        _check(L.lib().espn_gpu_table_info(self._h, C.byref(info)))
        self.n_docs = int(info.n_docs)
        self.n_tokens = int(info.n_tokens)
        self.hbm_bytes = int(info.hbm_bytes)
        self.host_bytes = int(info.host_bytes)
        self.resident_docs = int(info.resident_docs)
        self.tiered = self._resident is not None
        self.max_tokens = int(info.max_tokens)
        self.min_tokens = int(info.min_tokens)
        self._workspaces = {}

    @classmethod
    def open_store(cls, base, dtype: str = "f16", mode: str = "buffered", chunk_bytes: int = 64 << 20,
                   **kw) -> "GpuStore":
        """open_store (store.hpp:111-112) for the GPU table, STREAMED from the
        .espn file (include/espn_store.h): the table is allocated from the
        manifest (only resident docs in HBM when `resident` is given, the rest
        in the pinned-host tier) and filled chunk by chunk (chunk_bytes of
        rows at a time), so the store is never read whole into memory.
        d_cls / value_width / alignment come from the manifest."""
        m = load_manifest(base)
        tok = m.records["token_count"].astype(np.uint64)
        row_ptr = np.zeros(m.count() + 1, np.uint64)
        row_ptr[1:] = np.cumsum(tok)
        store = cls(row_ptr, None, m.d, dtype, d_cls=m.d_cls, value_width=m.value_width, alignment=m.alignment,
                    streamed=True, **kw)
        slib = L.store_lib()
        reader = C.c_void_p()
        h = L.StoreHeader()
        _check_store(slib.espn_store_open(str(base).encode(), {"direct": L.ESPN_READ_DIRECT, "buffered":
                                          L.ESPN_READ_BUFFERED, "mmap": L.ESPN_READ_MMAP}[mode], 16,
                                          C.byref(reader), C.byref(h)))
        try:
            i, n = 0, m.count()
            row_bytes = m.d * 2
            while i < n:
                j = int(np.searchsorted(row_ptr, row_ptr[i] + max(chunk_bytes // row_bytes, 1), side="right")) - 1
                j = min(max(j, i + 1), n)
                rp_l = np.zeros(j - i + 1, np.uint64)
                codes = np.empty(max(int(row_ptr[j] - row_ptr[i]) * m.d, 1), np.uint16)
                _check_store(slib.espn_store_read_rows(reader, i, j - i, _DTYPES[dtype], rp_l.ctypes.data,
                                                       codes.ctypes.data))
                store.load_rows(i, codes)
                i = j
        finally:
            slib.espn_store_close(reader)
        return store

    def load_rows(self, doc_begin: int, codes) -> None:
        """espn_gpu_table_load_rows: the next docs' plain 2-byte codes (streamed tables)."""
        codes = np.ascontiguousarray(codes, dtype=np.uint16)
        rp = self._row_ptr_host
        n = int(np.searchsorted(rp, rp[doc_begin] + codes.size // self.d, side="right")) - 1 - doc_begin
        _check(L.lib().espn_gpu_table_load_rows(self._h, int(doc_begin), int(n), codes.ctypes.data))

    @classmethod
    def from_device(cls, row_ptr, rows, d: int, dtype: str = "f16", **kw) -> "GpuStore":
        """Adopt CUDA tensors (torch) already resident in HBM (borrowed).  Pass
        rows_tiled=True for rows already in the HBM tile layout (synth output);
        plain rows get a library-owned tiled copy."""
        return cls(row_ptr, rows, d, dtype, borrowed_device=True, **kw)

    @property
    def handle(self):
        return self._h

    def record_bytes(self, token_count):
        """store.hpp:32-34."""
        return (self.d_cls + np.asarray(token_count, dtype=np.uint64) * self.d) * self.value_width

    def token_counts(self, doc_ids) -> Optional[np.ndarray]:
        if self._row_ptr_host is None:
            return None
        ids = np.asarray(doc_ids, dtype=np.int64)
        return (self._row_ptr_host[ids + 1] - self._row_ptr_host[ids]).astype(np.uint64)

    def fetch_batch(self, doc_ids: Sequence[int]) -> FetchResult:
        """store.hpp:91-94 through K1: request order, duplicates allowed,
        unknown ids raise InvalidInputError.  Decodes to fp32 like the
        reference's value_width=2 path."""
        import torch
        ids = np.ascontiguousarray(np.asarray(doc_ids, dtype=np.uint32))
        n = int(ids.shape[0])
        t0 = time.perf_counter()
        dev = torch.device("cuda", self.device)
        d_ids = torch.from_numpy(ids.astype(np.int32)).to(dev)
        d_rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        _check(L.lib().espn_gpu_gather(self._h, _ptr(d_ids) if n else None, n, None, _ptr(d_rp), 0, None))
        rp = d_rp.cpu().numpy().astype(np.uint64)
        total = int(rp[-1]) if n else 0
        d_rows = torch.empty(max(total * self.d, 1), dtype=torch.int16, device=dev)
        if n:
            _check(L.lib().espn_gpu_gather(self._h, _ptr(d_ids), n, _ptr(d_rows), _ptr(d_rp), total, None))
        codes = d_rows[: total * self.d].cpu().numpy().view(np.uint16)
        vals = decode(codes, self.dtype)
        res = FetchResult()
        for i in range(n):
            a, b = int(rp[i]), int(rp[i + 1])
            res.docs.append(FetchedDoc(EmbeddingMatrix(int(ids[i]), b - a, self.d,
                                                       vals[a * self.d:b * self.d].copy())))
        tok = np.diff(rp)
        payload = self.record_bytes(tok)
        res.bytes_read = int(payload.sum())
        res.blocks_read = int(((payload + 4095) // 4096).sum())
        res.wall_time = time.perf_counter() - t0
        return res

    # ---- persistent re-rank server (espn_gpu.h) ----
    def server_start(self, query_precision: str = "auto", idle_us: int = 0) -> None:
        """Launch the persistent MaxSim server: fused tcgen05 batches of this
        table are then submitted to it (plan + wait kernels per batch, no
        per-batch MaxSim launch).  It exits after idle_us without work (0 =
        50 ms) and is relaunched by the next served call."""
        _check(L.lib().espn_gpu_server_start(self._h, _QPREC[query_precision], int(idle_us)))

    def server_stop(self) -> None:
        _check(L.lib().espn_gpu_server_stop(self._h))

    def server_pause(self) -> None:
        """Stop the kernel but stay in served mode (capture graphs now;
        server_start relaunches it before replaying them)."""
        _check(L.lib().espn_gpu_server_pause(self._h))

    @property
    def server_running(self) -> bool:
        return bool(L.lib().espn_gpu_server_running(self._h))

    def workspace(self, max_queries: int, max_candidates: int, max_query_tokens: int = 32) -> "Reranker":
        return Reranker(self, max_queries, max_candidates, max_query_tokens)

    def close(self) -> None:
        rr = getattr(self, "_pipeline_rr", None)  # workspace cached by pipeline.run_query / run_batch_queries
        if rr is not None:
            rr.close()
            self._pipeline_rr = None
        if getattr(self, "_h", None):
            L.lib().espn_gpu_table_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decode(codes: np.ndarray, dtype: str) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint16)
    if dtype in ("f16", "fp16"):
        return codes.view(np.float16).astype(np.float32)
    return (codes.astype(np.uint32) << 16).view(np.float32)


def encode(values: np.ndarray, dtype: str) -> np.ndarray:
    v = np.asarray(values, dtype=np.float32)
    if dtype in ("f16", "fp16"):
        return v.astype(np.float16).view(np.uint16)
    u = v.view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


class Reranker:
    """A table plus one workspace (per-stream scratch): the batched re-rank
    entry point.  One in-flight batch at a time."""

    def __init__(self, store: GpuStore, max_queries: int, max_candidates: int, max_query_tokens: int = 32,
                 max_list: int = 0, staging_bytes: int = 0):
        self.store = store
        desc = L.WorkspaceDesc(max_queries=max_queries, max_candidates=max_candidates,
                               max_query_tokens=max_query_tokens, max_list=max_list, staging_bytes=staging_bytes)
        h = C.c_void_p()
        _check(L.lib().espn_gpu_workspace_create(store.handle, C.byref(desc), C.byref(h)))
        self._h = h
        self.max_queries = max_queries
        self.max_candidates = max_candidates

    @property
    def handle(self):
        return self._h

    def rerank_arrays(self, query_tokens, cand_ids, cand_cls, cand_offsets, config: PipelineConfig,
                      kernel: str = "auto", device_io: bool = False, write_bow: bool = False,
                      out=None, stream=None, sync: bool = True, needed_counts=None, prefetched: bool = False,
                      fetch_stats: bool = False, separate_topk: bool = False, query_precision: str = "auto"):
        """Batched stages 3-6.  query_tokens (B, q, d) fp32; cand_* CSR over
        queries with cand_offsets (B+1, host uint64).  Host numpy arrays by
        default (copied in and out inside the call); device torch tensors
        with device_io=True.  Returns (ids[B,k], scores[B,k], counts[B], bow).
        query_precision: "auto" (the fp32 query as given; tcgen05 as hi + lo,
        espn_gpu.h ESPN_RERANK_QUERY_*), "split" (hi + lo everywhere) or
        "rounded" (query rounded to the table dtype first)."""
        offs = np.ascontiguousarray(np.asarray(cand_offsets, dtype=np.uint64))
        B = offs.shape[0] - 1
        k = int(config.final_k)
        if device_io:
            import torch
            nq = int(query_tokens.shape[1])
            if out is None:
                dev = query_tokens.device
                out = (torch.empty((B, k), dtype=torch.int32, device=dev),
                       torch.empty((B, k), dtype=torch.float32, device=dev),
                       torch.empty((B,), dtype=torch.int32, device=dev),
                       torch.empty((int(offs[-1]),), dtype=torch.float32, device=dev) if write_bow else None)
        else:
            query_tokens = np.ascontiguousarray(query_tokens, dtype=np.float32)
            cand_ids = np.ascontiguousarray(cand_ids, dtype=np.uint32).ravel()
            cand_cls = np.ascontiguousarray(cand_cls, dtype=np.float32).ravel()
            # the C side trusts these sizes (it copies B*q*d and C entries)
            if B < 0 or (B and int(offs[0]) != 0) or np.any(np.diff(offs.astype(np.int64)) < 0):
                raise InvalidInputError("cand_offsets must start at 0 and be non-decreasing")
            n_c = int(offs[-1]) if B else 0
            if cand_ids.size < n_c or cand_cls.size < n_c:
                raise InvalidInputError(f"cand_ids / cand_cls hold {cand_ids.size} / {cand_cls.size} entries, "
                                        f"cand_offsets needs {n_c}")
            if B == 0:
                nq = int(query_tokens.shape[1]) if query_tokens.ndim == 3 and query_tokens.shape[1] else 1
            elif query_tokens.ndim == 3:
                if query_tokens.shape[0] != B or query_tokens.shape[2] != self.store.d:
                    raise InvalidInputError(f"query_tokens shape {query_tokens.shape} != (B={B}, q, d={self.store.d})")
                nq = int(query_tokens.shape[1])
            else:
                if query_tokens.size == 0 or query_tokens.size % (B * self.store.d):
                    raise InvalidInputError("query_tokens must hold B * q * d values")
                nq = int(query_tokens.size // B // self.store.d)
            if out is None:
                out = (np.zeros((B, k), np.uint32), np.zeros((B, k), np.float32), np.zeros(B, np.uint32),
                       np.full(int(offs[-1]), np.nan, np.float32) if write_bow else None)
        flags = 0
        if config.partial_rerank_enabled:
            flags |= L.ESPN_RERANK_PARTIAL
        if device_io:
            flags |= L.ESPN_RERANK_DEVICE_IO
        if write_bow:
            flags |= L.ESPN_RERANK_WRITE_BOW
        if not sync:
            flags |= L.ESPN_RERANK_ASYNC
        if prefetched:
            flags |= L.ESPN_RERANK_PREFETCHED
        if separate_topk:
            flags |= L.ESPN_RERANK_SEPARATE_TOPK
        flags |= _QPREC[query_precision]
        args = L.RerankArgs(n_queries=B, n_query_tokens=nq, query_tokens=_ptr(query_tokens),
                            cand_ids=_ptr(cand_ids), cand_cls=_ptr(cand_cls), cand_offsets=offs.ctypes.data,
                            rerank_count=int(config.rerank_count), final_k=k, alpha=float(config.alpha),
                            flags=flags, kernel=_KERNELS[kernel])
        if needed_counts is not None:
            needed_counts = np.ascontiguousarray(needed_counts, dtype=np.uint32)
            args.needed_counts = needed_counts.ctypes.data
        fs = (L.FetchStats * B)() if fetch_stats else None
        o = L.RerankOut(ids=_ptr(out[0]), scores=_ptr(out[1]), counts=_ptr(out[2]),
                        bow_scores=_ptr(out[3]) if write_bow else None,
                        fetch_stats=C.addressof(fs) if fs is not None else None)
        self._keepalive = (query_tokens, cand_ids, cand_cls, offs, out, needed_counts)
        _check(L.lib().espn_gpu_rerank(self.store.handle, self._h, C.byref(args), C.byref(o),
                                       C.c_void_p(stream) if stream else None))
        if fs is not None:
            self.last_fetch_stats = [{f: int(getattr(x, f)) for f, _ in L.FetchStats._fields_} for x in fs]
        return out

    # ---- multi-GPU (espn_gpu.h "Multi-GPU") -------------------------
    def _sharded_args(self, query_tokens, cand_ids, cand_cls, cand_offsets, config, device_io, device_offsets,
                      sync, needed_counts, query_precision, out, kernel="auto"):
        if device_offsets:
            offs_p, B = _ptr(cand_offsets), int(cand_offsets.numel()) - 1
            nc_p = _ptr(needed_counts) if needed_counts is not None else None
            keep = ()
        else:
            offs = np.ascontiguousarray(np.asarray(cand_offsets, dtype=np.uint64))
            offs_p, B = offs.ctypes.data, offs.shape[0] - 1
            nc = np.ascontiguousarray(needed_counts, dtype=np.uint32) if needed_counts is not None else None
            nc_p = nc.ctypes.data if nc is not None else None
            keep = (offs, nc)
        k = int(config.final_k)
        if not device_io:
            query_tokens = np.ascontiguousarray(query_tokens, dtype=np.float32)
            cand_ids = np.ascontiguousarray(cand_ids, dtype=np.uint32).ravel()
            cand_cls = np.ascontiguousarray(cand_cls, dtype=np.float32).ravel()
            if query_tokens.ndim != 3 or query_tokens.shape[0] != B or query_tokens.shape[2] != self.store.d:
                raise InvalidInputError(f"query_tokens must be (B={B}, q, d={self.store.d})")
            if B and (cand_ids.size < int(keep[0][-1]) or cand_cls.size < int(keep[0][-1])):
                raise InvalidInputError("cand_ids / cand_cls shorter than cand_offsets[B]")
            if out is None:
                out = (np.zeros((B, k), np.uint32), np.zeros((B, k), np.float32), np.zeros(B, np.uint32))
        elif out is None:
            import torch
            dev = query_tokens.device
            out = (torch.empty((B, k), dtype=torch.int32, device=dev), torch.empty((B, k), dtype=torch.float32, device=dev),
                   torch.empty((B,), dtype=torch.int32, device=dev))
        flags = _QPREC[query_precision]
        if config.partial_rerank_enabled:
            flags |= L.ESPN_RERANK_PARTIAL
        if device_io:
            flags |= L.ESPN_RERANK_DEVICE_IO
        if device_offsets:
            flags |= L.ESPN_RERANK_DEVICE_OFFSETS
        if not sync:
            flags |= L.ESPN_RERANK_ASYNC
        args = L.RerankArgs(n_queries=B, n_query_tokens=int(query_tokens.shape[1]), query_tokens=_ptr(query_tokens),
                            cand_ids=_ptr(cand_ids), cand_cls=_ptr(cand_cls), cand_offsets=offs_p,
                            rerank_count=int(config.rerank_count), final_k=k, alpha=float(config.alpha),
                            flags=flags, kernel=_KERNELS[kernel], needed_counts=nc_p)
        o = L.RerankOut(ids=_ptr(out[0]), scores=_ptr(out[1]), counts=_ptr(out[2]))
        self._keep_sh = (query_tokens, cand_ids, cand_cls, keep, out)
        return args, o, out

    def rerank_sharded(self, query_tokens, cand_ids, cand_cls, cand_offsets, config: PipelineConfig, comm: "NcclComm",
                       device_io: bool = False, device_offsets: bool = False, out=None, stream=None, sync: bool = True,
                       needed_counts=None, query_precision: str = "auto", kernel: str = "auto"):
        """espn_gpu_rerank_sharded: every rank passes the SAME global batch
        (global doc ids) and gets the global ranked lists back; the table's
        placement (doc-id shard or full replica) decides the split.  Returns
        (ids[B,k], scores[B,k], counts[B])."""
        args, o, out = self._sharded_args(query_tokens, cand_ids, cand_cls, cand_offsets, config, device_io,
                                          device_offsets, sync, needed_counts, query_precision, out, kernel)
        _check(L.lib().espn_gpu_rerank_sharded(self.store.handle, self._h, C.byref(args), C.byref(o), comm.handle,
                                               C.c_void_p(stream) if stream else None))
        return out

    def shard_pack(self, query_tokens, cand_ids, cand_cls, cand_offsets, config: PipelineConfig, nranks: int,
                   rank: int, device_io: bool = True, stream=None, query_precision: str = "auto",
                   kernel: str = "auto"):
        """Phase 1 without NCCL: this rank's packed block (device pointer, int32
        words) in the workspace's send buffer."""
        args, o, _ = self._sharded_args(query_tokens, cand_ids, cand_cls, cand_offsets, config, device_io, False,
                                        True, None, query_precision, None, kernel)
        ptr, words = C.c_void_p(), C.c_uint64()
        _check(L.lib().espn_gpu_shard_pack(self.store.handle, self._h, C.byref(args), int(nranks), int(rank),
                                           C.c_void_p(stream) if stream else None, C.byref(ptr), C.byref(words)))
        return int(ptr.value or 0), int(words.value)

    def shard_merge(self, query_tokens, cand_ids, cand_cls, cand_offsets, config: PipelineConfig, recv, nranks: int,
                    device_io: bool = True, out=None, stream=None, query_precision: str = "auto"):
        """Phase 3 without NCCL: merge nranks gathered blocks (device tensor
        `recv`) into the global ranked lists."""
        args, o, out = self._sharded_args(query_tokens, cand_ids, cand_cls, cand_offsets, config, device_io, False,
                                          True, None, query_precision, out)
        _check(L.lib().espn_gpu_shard_merge(self.store.handle, self._h, C.byref(args), _ptr(recv), int(nranks),
                                            C.byref(o), C.c_void_p(stream) if stream else None))
        return out

    def prefetch_hints(self, hint_ids, hint_offsets, stream=None, device_offsets: bool = False):
        """espn_gpu_prefetch_hints: stage the host-tier rows of an approximate
        id list (the IVF snapshot after delta clusters, CSR over queries) on
        `stream`; the next rerank_arrays(..., prefetched=True) consumes it with
        its final candidates.  hint_ids: device tensor (uint32/int32) or host
        numpy array."""
        if isinstance(hint_ids, np.ndarray):  # host ids: copied by the library
            hint_ids = np.ascontiguousarray(hint_ids, dtype=np.uint32)
            flags = 0
        else:
            flags = L.ESPN_RERANK_DEVICE_IO
        if device_offsets:
            offs_p, B = _ptr(hint_offsets), int(hint_offsets.numel()) - 1
            flags |= L.ESPN_RERANK_DEVICE_OFFSETS
        else:
            offs = np.ascontiguousarray(np.asarray(hint_offsets, dtype=np.uint64))
            offs_p, B = offs.ctypes.data, offs.shape[0] - 1
            self._keep_hints = (offs, hint_ids)
        _check(L.lib().espn_gpu_prefetch_hints(self.store.handle, self._h, B, _ptr(hint_ids), offs_p, flags,
                                               C.c_void_p(stream) if stream else None))

    def prefetch_rows(self, ids, id_offsets, rows, row_byte_off, stream=None):
        """espn_gpu_prefetch_rows: stage rows the caller read from the store
        file (the disk tier) -- doc ids[j]'s plain codes at byte row_byte_off[j]
        of the host buffer `rows` (numpy uint8, or a pinned torch tensor) --
        keyed by doc; the next rerank_arrays(..., prefetched=True) finds them."""
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        offs = np.ascontiguousarray(np.asarray(id_offsets, dtype=np.uint64))
        boff = np.ascontiguousarray(np.asarray(row_byte_off, dtype=np.uint64))
        if boff.shape[0] < ids.shape[0]:
            raise InvalidInputError("one row offset per id")
        if isinstance(rows, np.ndarray):
            rows_p, nbytes = rows.ctypes.data, int(rows.nbytes)
        else:  # torch tensor (pinned host memory: asynchronous upload)
            rows_p, nbytes = int(rows.data_ptr()), int(rows.numel() * rows.element_size())
        self._keep_rows = (ids, offs, boff, rows)
        _check(L.lib().espn_gpu_prefetch_rows(self.store.handle, self._h, offs.shape[0] - 1, ids.ctypes.data,
                                              offs.ctypes.data, rows_p, boff.ctypes.data, nbytes,
                                              C.c_void_p(stream) if stream else None))

    def prefetch(self, query_tokens, cand_ids, cand_cls, cand_offsets, config: PipelineConfig, stream=None,
                 needed_counts=None, device_offsets: bool = False):
        """espn_gpu_prefetch: stage the NEXT batch's host-tier rows on `stream`
        (a side stream) while the current batch scores; the next
        rerank_arrays(..., device_io=True, prefetched=True) of the same arrays
        consumes it.  Device torch tensors; offsets host (numpy) unless
        device_offsets."""
        if device_offsets:
            offs_p, B = _ptr(cand_offsets), int(cand_offsets.numel()) - 1
            nc_p = _ptr(needed_counts) if needed_counts is not None else None
        else:
            offs = np.ascontiguousarray(np.asarray(cand_offsets, dtype=np.uint64))
            offs_p, B = offs.ctypes.data, offs.shape[0] - 1
            nc = np.ascontiguousarray(needed_counts, dtype=np.uint32) if needed_counts is not None else None
            nc_p = nc.ctypes.data if nc is not None else None
            self._pf_keep = (offs, nc)
        flags = L.ESPN_RERANK_DEVICE_IO | (L.ESPN_RERANK_DEVICE_OFFSETS if device_offsets else 0)
        args = L.RerankArgs(n_queries=B, n_query_tokens=int(query_tokens.shape[1]), query_tokens=_ptr(query_tokens),
                            cand_ids=_ptr(cand_ids), cand_cls=_ptr(cand_cls), cand_offsets=offs_p,
                            rerank_count=int(config.rerank_count), final_k=int(config.final_k),
                            alpha=float(config.alpha), flags=flags, needed_counts=nc_p)
        _check(L.lib().espn_gpu_prefetch(self.store.handle, self._h, C.byref(args),
                                         C.c_void_p(stream) if stream else None))

    def sync(self, stream=None) -> None:
        _check(L.lib().espn_gpu_workspace_sync(self._h, C.c_void_p(stream) if stream else None))

    def counters(self) -> dict:
        c = L.Counters()
        _check(L.lib().espn_gpu_get_counters(self._h, C.byref(c)))
        return {f: (float(getattr(c, f)) if f.endswith("_ms") else int(getattr(c, f))) for f, _ in L.Counters._fields_}

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().espn_gpu_workspace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (the bytes every rank passes to NcclComm)."""
    buf = (C.c_uint8 * 128)()
    _check(L.lib().espn_nccl_get_unique_id(C.addressof(buf)))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created by the library (ncclCommInitRank on
    `device`); hand the same `uid` (nccl_unique_id() on one rank, broadcast)
    to every rank."""

    def __init__(self, nranks: int, uid: bytes, rank: int, device: int = 0, handle=None):
        if handle is not None:
            self._h = C.c_void_p(handle)
            return
        if len(uid) != 128:
            raise InvalidInputError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(L.lib().espn_nccl_comm_init(int(nranks), C.addressof(buf), int(rank), int(device), C.byref(h)))
        self._h = h

    @classmethod
    def init_all(cls, devices) -> List["NcclComm"]:
        """ncclCommInitAll: one communicator per device of this process."""
        devs = (C.c_int * len(devices))(*[int(x) for x in devices])
        hs = (C.c_void_p * len(devices))()
        _check(L.lib().espn_nccl_comm_init_all(len(devices), C.addressof(devs), C.addressof(hs)))
        return [cls(0, b"", 0, handle=hs[i]) for i in range(len(devices))]

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().espn_nccl_comm_destroy(self._h)
            self._h = None


def record_io(store: GpuStore, token_counts) -> Tuple[np.ndarray, np.ndarray]:
    """Per-record (bytes, blocks) of the reference store (store.hpp:61-65,
    SPEC.md "Block accounting"): buffered reads move the exact payload
    record_bytes = (d_cls + t*d) * value_width and touch ceil(bytes / 4096)
    blocks."""
    rec = store.record_bytes(np.asarray(token_counts, np.uint64)).astype(np.uint64)
    return rec, (rec + np.uint64(4095)) // np.uint64(4096)


def _stats_for(store: GpuStore, ids: np.ndarray, n_needed: int, query_id: int, elapsed: float,
               prefetched_ids=None) -> QueryStats:
    """QueryStats (pipeline.hpp:36-54) exactly as the reference defines them
    for one query -- the same set arithmetic as the oracle's eo_rerank_query:
    needed = first n_needed final candidates; prefetched = the ids the
    prefetcher fetched (the query's snapshot hints; none without prefetch);
    hits = needed ∩ prefetched; missed = needed minus prefetched; byte and block
    counters per record over prefetched / missed / needed docs.  The tier view
    (rows resident in HBM vs staged over PCIe) is the separate device
    accounting, Reranker.last_fetch_stats."""
    ids = np.asarray(ids, np.uint32)
    needed = ids[:n_needed]
    pf = np.unique(np.asarray(prefetched_ids if prefetched_ids is not None else np.zeros(0), np.uint32))
    st = QueryStats(query_id=query_id, needed_count=int(n_needed), rerank_time=elapsed, total_time=elapsed)
    st.prefetched_count = int(np.asarray(prefetched_ids).size) if prefetched_ids is not None else 0
    hit = np.isin(needed, pf) if pf.size else np.zeros(needed.size, bool)
    st.missed_count = int(n_needed - hit.sum())
    st.hit_rate = float(hit.sum()) / n_needed if n_needed else 0.0
    tok_n = store.token_counts(needed)
    if tok_n is not None:
        rec, blk = record_io(store, tok_n)
        st.needed_payload_bytes = int(rec.sum())
        st.critical_fetch_bytes = int(rec[~hit].sum())
        st.critical_blocks_read = int(blk[~hit].sum())
    if prefetched_ids is not None and np.asarray(prefetched_ids).size:
        tok_p = store.token_counts(np.asarray(prefetched_ids, np.uint32))
        if tok_p is not None:
            st.prefetch_bytes = int(record_io(store, tok_p)[0].sum())
    return st


def rerank_batch(queries: Sequence[QueryEmbedding], candidate_lists: Sequence[CandidateList],
                 store: GpuStore, config: PipelineConfig, kernel: str = "auto") -> BatchResult:
    """run_batch (pipeline.hpp:81-85) restricted to stages 3-6: one device pass
    over the whole batch; per-query results identical to single-query calls."""
    if len(queries) != len(candidate_lists):
        raise InvalidInputError("queries and candidate lists differ in length")
    B = len(queries)
    res = BatchResult()
    if B == 0:
        return res
    d = store.d
    nq = queries[0].rows
    for q in queries:
        if q.cols != d:
            raise InvalidInputError(f"query dim {q.cols} != table dim {d}")
        if q.rows != nq:
            raise InvalidInputError("all queries of a batch must have the same token count")
    qt = np.stack([np.asarray(q.tokens, np.float32).reshape(q.rows, q.cols) for q in queries])
    offs = np.zeros(B + 1, np.uint64)
    for i, cl in enumerate(candidate_lists):
        offs[i + 1] = offs[i] + len(cl.entries)
    ids = np.fromiter((c.doc_id for cl in candidate_lists for c in cl.entries), np.uint32, int(offs[-1]))
    cls = np.fromiter((c.cls_score for cl in candidate_lists for c in cl.entries), np.float32, int(offs[-1]))
    rr = Reranker(store, B, max(int(offs[-1]), 1), max(nq, 1))
    try:
        t0 = time.perf_counter()
        oid, osc, ocnt, _ = rr.rerank_arrays(qt, ids, cls, offs, config, kernel=kernel, fetch_stats=True)
        fstats = rr.last_fetch_stats
        wall = time.perf_counter() - t0
    finally:
        rr.close()
    lat = []
    for b in range(B):
        n = int(ocnt[b])
        res.rankings.append(RankedList([ScoredDoc(int(oid[b, i]), float(osc[b, i])) for i in range(n)]))
        a0, a1 = int(offs[b]), int(offs[b + 1])
        need = min(a1 - a0, int(config.rerank_count))
        res.stats.append(_stats_for(store, ids[a0:a1], need, queries[b].query_id, wall))
        lat.append(wall)
    lat = np.asarray(lat)
    res.batch = BatchStats(n_queries=B, mean_latency=float(lat.mean()), p50_latency=float(np.percentile(lat, 50)),
                           p99_latency=float(np.percentile(lat, 99)), wall_time=wall,
                           total_critical_fetch_bytes=sum(s.critical_fetch_bytes for s in res.stats))
    return res


def rerank_candidates(query: QueryEmbedding, candidates: CandidateList, store: GpuStore,
                      config: PipelineConfig, kernel: str = "auto") -> Tuple[RankedList, QueryStats]:
    """Stages 3-6 of run_query (pipeline.hpp:56-64) for one query:
    the missing "candidates in -> ranked out" seam."""
    r = rerank_batch([query], [candidates], store, config, kernel=kernel)
    return r.rankings[0], r.stats[0]


# ---- quality harness (metrics.hpp:10-20) -----------
def _top_ids(ranked, k: int):
    if isinstance(ranked, RankedList):
        return [e.doc_id for e in ranked.entries[:k]]
    return [int(x) for x in list(ranked)[:k]]  # a plain id sequence (e.g. a row of rerank_arrays ids)


def mrr_at_k(results: Dict[int, object], qrels: Dict[int, set], k: int) -> float:
    """Mean over the qrels queries (id order) of 1/rank of the first relevant
    doc within the top k; a query without results counts 0 (metrics.hpp:10-12)."""
    if k < 1:
        raise InvalidInputError("k must be >= 1 (SPEC.md:74)")
    if not qrels:
        return 0.0
    s = 0.0
    for qid in sorted(qrels):
        rel = qrels[qid]
        for r, d in enumerate(_top_ids(results[qid], k) if qid in results else []):
            if d in rel:
                s += 1.0 / (r + 1)
                break
    return s / len(qrels)


def recall_at_k(results: Dict[int, object], qrels: Dict[int, set], k: int) -> float:
    """Mean over the qrels queries of |relevant in top k| / |relevant| (metrics.hpp:14-15)."""
    if k < 1:
        raise InvalidInputError("k must be >= 1 (SPEC.md:82)")
    if not qrels:
        return 0.0
    s = 0.0
    for qid in sorted(qrels):
        rel = qrels[qid]
        if qid in results and rel:
            s += sum(1 for d in _top_ids(results[qid], k) if d in rel) / len(rel)
    return s / len(qrels)


def load_qrels(src) -> Dict[int, set]:
    """TREC qrels (metrics.hpp:17-20): `query_id 0 doc_id relevance` per line,
    relevance > 0 marks a relevant doc, blank lines skipped, else FormatError.
    `src` is a path or an iterable of lines."""
    if isinstance(src, (str, Path)):
        try:
            with open(src) as f:
                return load_qrels(f.read().splitlines())
        except OSError as e:
            raise IoError(f"cannot open qrels file {src}: {e}") from None
    q: Dict[int, set] = {}
    for n, line in enumerate(src, 1):
        f = line.split()
        if not f:
            continue
        try:
            if len(f) != 4:
                raise ValueError
            qid, _, did, rel = (int(x) for x in f)
            if not (0 <= qid <= 0xFFFFFFFF and 0 <= did <= 0xFFFFFFFF):
                raise ValueError
        except ValueError:
            raise FormatError(f"qrels line {n}: expected `query_id 0 doc_id relevance`") from None
        if rel > 0:
            q.setdefault(qid, set()).add(did)
    return q
