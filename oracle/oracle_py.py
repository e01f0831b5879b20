"""ctypes binding of the CPU oracle (oracle/espn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference legs.  Never imported
by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libespn_oracle.so"
REF_HALF = HERE / "_ref" / "libref_half.so"

F16, BF16 = 0, 1


class Table(C.Structure):
    _fields_ = [
        ("n_docs", C.c_uint64), ("d", C.c_uint32), ("dtype", C.c_uint32),
        ("row_ptr", C.c_void_p), ("rows", C.c_void_p), ("d_cls", C.c_uint32),
        ("value_width", C.c_uint32), ("alignment", C.c_uint32), ("direct_io", C.c_uint32),
    ]


class Config(C.Structure):
    _fields_ = [("rerank_count", C.c_uint32), ("final_k", C.c_uint32), ("alpha", C.c_float),
                ("prefetch_enabled", C.c_int32), ("partial_rerank_enabled", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("prefetched_count", C.c_uint64), ("needed_count", C.c_uint64),
                ("missed_count", C.c_uint64), ("hit_rate", C.c_double),
                ("prefetch_bytes", C.c_uint64), ("critical_fetch_bytes", C.c_uint64),
                ("critical_blocks_read", C.c_uint64), ("needed_payload_bytes", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        h = C.CDLL(str(LIB))
        vp, u32, u64, f32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_float
        h.eo_float_to_half.restype = C.c_uint16; h.eo_float_to_half.argtypes = [f32]
        h.eo_half_to_float.restype = f32; h.eo_half_to_float.argtypes = [C.c_uint16]
        h.eo_float_to_bf16.restype = C.c_uint16; h.eo_float_to_bf16.argtypes = [f32]
        h.eo_bf16_to_float.restype = f32; h.eo_bf16_to_float.argtypes = [C.c_uint16]
        h.eo_encode.argtypes = [vp, vp, C.c_size_t, C.c_int]
        h.eo_decode.argtypes = [vp, vp, C.c_size_t, C.c_int]
        h.eo_dot_f32.restype = f32; h.eo_dot_f32.argtypes = [vp, vp, u32]
        h.eo_maxsim_score.restype = f32; h.eo_maxsim_score.argtypes = [vp, u32, vp, u32, u32]
        h.eo_aggregate_score.restype = f32; h.eo_aggregate_score.argtypes = [f32, f32, f32]
        h.eo_rank.restype = C.c_int; h.eo_rank.argtypes = [vp, vp, C.c_size_t, vp, vp]
        h.eo_gather.restype = C.c_int; h.eo_gather.argtypes = [C.POINTER(Table), vp, C.c_size_t, vp, vp]
        h.eo_validate_config.restype = C.c_int; h.eo_validate_config.argtypes = [C.POINTER(Config)]
        h.eo_rerank_query.restype = C.c_int
        h.eo_rerank_query.argtypes = [C.POINTER(Table), vp, u32, vp, vp, u32, vp, u32, C.POINTER(Config),
                                      vp, vp, vp, C.POINTER(Stats)]
        h.eo_rerank_batch.restype = C.c_int
        h.eo_rerank_batch.argtypes = [C.POINTER(Table), vp, u32, u32, vp, vp, vp, C.POINTER(Config), vp, vp, vp,
                                      C.c_int]
        h.eo_maxsim_batch.restype = C.c_int
        h.eo_maxsim_batch.argtypes = [C.POINTER(Table), vp, u32, u32, vp, vp, vp, C.c_int]
        h.eo_record_bytes.restype = u64; h.eo_record_bytes.argtypes = [C.POINTER(Table), u64]
        _lib = h
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data if a is not None and a.size else None


class OracleTable:
    """CSR table as the oracle sees it (host numpy arrays kept alive)."""

    def __init__(self, row_ptr, rows, d, dtype=F16, d_cls=128, value_width=2, alignment=4096, direct_io=False):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        self.rows = np.ascontiguousarray(rows, dtype=np.uint16)
        self.d = int(d)
        self.dtype = dtype
        self.s = Table(n_docs=self.row_ptr.shape[0] - 1, d=self.d, dtype=dtype, row_ptr=_p(self.row_ptr),
                       rows=_p(self.rows), d_cls=d_cls, value_width=value_width, alignment=alignment,
                       direct_io=1 if direct_io else 0)

    @property
    def n_docs(self):
        return int(self.row_ptr.shape[0] - 1)

    def doc(self, i) -> np.ndarray:
        a, b = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return decode(self.rows[a * self.d:b * self.d], self.dtype).reshape(b - a, self.d)


def encode(x, dtype=F16) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    out = np.empty(x.shape, np.uint16)
    lib().eo_encode(_p(x), _p(out), x.size, dtype)
    return out


def decode(c, dtype=F16) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.uint16).ravel()
    out = np.empty(c.shape, np.float32)
    lib().eo_decode(_p(c), _p(out), c.size, dtype)
    return out


def round_to(x, dtype=F16) -> np.ndarray:
    x = np.asarray(x, np.float32)
    return decode(encode(x, dtype), dtype).reshape(x.shape)


def maxsim_score(q: np.ndarray, doc: np.ndarray) -> float:
    q = np.ascontiguousarray(q, np.float32)
    doc = np.ascontiguousarray(doc, np.float32)
    return float(lib().eo_maxsim_score(_p(q), q.shape[0], _p(doc), doc.shape[0], q.shape[1]))


def aggregate_score(cls, bow, alpha) -> float:
    return float(lib().eo_aggregate_score(cls, bow, alpha))


def rank(ids, scores):
    ids = np.ascontiguousarray(ids, np.uint32)
    scores = np.ascontiguousarray(scores, np.float32)
    oi = np.empty_like(ids)
    os_ = np.empty_like(scores)
    st = lib().eo_rank(_p(ids), _p(scores), ids.size, _p(oi), _p(os_))
    return st, oi, os_


def gather(t: OracleTable, ids):
    ids = np.ascontiguousarray(ids, np.uint32)
    rp = np.zeros(ids.size + 1, np.uint64)
    st = lib().eo_gather(C.byref(t.s), _p(ids), ids.size, _p(rp), None)
    if st:
        return st, None, None
    rows = np.zeros(int(rp[-1]) * t.d, np.uint16)
    lib().eo_gather(C.byref(t.s), _p(ids), ids.size, _p(rp), _p(rows))
    return 0, rp, rows


def rerank_query(t: OracleTable, q, cand_ids, cand_cls, rerank_count, final_k, alpha=1.0,
                 partial=False, prefetch_enabled=True, prefetched=None):
    q = np.ascontiguousarray(q, np.float32)
    ids = np.ascontiguousarray(cand_ids, np.uint32)
    cls = np.ascontiguousarray(cand_cls, np.float32)
    pf = np.ascontiguousarray(prefetched if prefetched is not None else np.zeros(0), np.uint32)
    cfg = Config(rerank_count, final_k, alpha, 1 if prefetch_enabled else 0, 1 if partial else 0)
    oi = np.zeros(max(final_k, 1), np.uint32)
    os_ = np.zeros(max(final_k, 1), np.float32)
    n = C.c_uint32(0)
    stats = Stats()
    st = lib().eo_rerank_query(C.byref(t.s), _p(q), q.shape[0], _p(ids), _p(cls), ids.size, _p(pf), pf.size,
                               C.byref(cfg), _p(oi), _p(os_), C.addressof(n), C.byref(stats))
    return st, oi[:n.value].copy(), os_[:n.value].copy(), stats


def rerank_batch(t: OracleTable, q, cand_ids, cand_cls, cand_off, rerank_count, final_k, alpha=1.0,
                 partial=False, nthreads=None):
    q = np.ascontiguousarray(q, np.float32)
    B, nq = q.shape[0], q.shape[1]
    ids = np.ascontiguousarray(cand_ids, np.uint32)
    cls = np.ascontiguousarray(cand_cls, np.float32)
    off = np.ascontiguousarray(cand_off, np.uint64)
    cfg = Config(rerank_count, final_k, alpha, 1, 1 if partial else 0)
    oi = np.zeros((B, final_k), np.uint32)
    os_ = np.zeros((B, final_k), np.float32)
    on = np.zeros(B, np.uint32)
    st = lib().eo_rerank_batch(C.byref(t.s), _p(q), B, nq, _p(ids), _p(cls), _p(off), C.byref(cfg), _p(oi), _p(os_),
                               _p(on), nthreads or os.cpu_count() or 1)
    return st, oi, os_, on


def maxsim_batch(t: OracleTable, q, cand_ids, cand_off, nthreads=None):
    q = np.ascontiguousarray(q, np.float32)
    ids = np.ascontiguousarray(cand_ids, np.uint32)
    off = np.ascontiguousarray(cand_off, np.uint64)
    # never NULL: the C batch runner tells a MaxSim job from a re-rank job by a
    # non-NULL output pointer, so an all-empty batch still needs one
    out = np.full(max(ids.size, 1), np.nan, np.float32)
    st = lib().eo_maxsim_batch(C.byref(t.s), _p(q), q.shape[0], q.shape[1], _p(ids), _p(off), out.ctypes.data,
                               nthreads or os.cpu_count() or 1)
    return st, out[:ids.size]


def ref_half():
    """The reference's own half.hpp codec (oracle/_ref), or None if not built."""
    if not REF_HALF.exists():
        return None
    h = C.CDLL(str(REF_HALF))
    h.ref_float_to_half.restype = C.c_uint16; h.ref_float_to_half.argtypes = [C.c_float]
    h.ref_half_to_float.restype = C.c_float; h.ref_half_to_float.argtypes = [C.c_uint16]
    h.ref_half_to_float_bits.restype = C.c_uint32; h.ref_half_to_float_bits.argtypes = [C.c_uint16]
    h.ref_float_bits_to_half.restype = C.c_uint16; h.ref_float_bits_to_half.argtypes = [C.c_uint32]
    return h
