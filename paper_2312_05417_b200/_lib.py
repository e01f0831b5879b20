"""ctypes binding of include/espn_gpu.h (the C-ABI of libespn_gpu.so).

The library is loaded from the package's lib/ directory only (built in-tree by
paper_2312_05417_b200.build).  There is deliberately no fallback: if the
shared object is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libespn_gpu.so"

ESPN_OK = 0
ESPN_E_INVALID_INPUT = 1
ESPN_E_INVALID_STATE = 2
ESPN_E_INVALID_CONFIG = 3
ESPN_E_FORMAT = 4
ESPN_E_IO = 5
ESPN_E_DATA_INTEGRITY = 6
ESPN_E_CUDA = 7

ESPN_DTYPE_F16 = 0
ESPN_DTYPE_BF16 = 1

ESPN_KERNEL_AUTO = 0
ESPN_KERNEL_TCGEN05 = 1
ESPN_KERNEL_SIMT = 2
ESPN_KERNEL_SMALL = 3

ESPN_TABLE_DEVICE_BORROWED = 0x1
ESPN_TABLE_ROWS_TILED = 0x2

ESPN_RERANK_PARTIAL = 0x1
ESPN_RERANK_DEVICE_IO = 0x2
ESPN_RERANK_ASYNC = 0x4
ESPN_RERANK_WRITE_BOW = 0x8
ESPN_RERANK_PROFILE = 0x10
ESPN_RERANK_DEVICE_OFFSETS = 0x20
ESPN_RERANK_PREFETCHED = 0x40
ESPN_RERANK_SEPARATE_TOPK = 0x80
ESPN_RERANK_QUERY_ROUNDED = 0x100
ESPN_RERANK_QUERY_SPLIT = 0x200
ESPN_TABLE_STREAMED = 0x4
ESPN_TABLE_DISK_TIER = 0x8
ESPN_READ_DIRECT, ESPN_READ_BUFFERED, ESPN_READ_MMAP = 0, 1, 2


class TableDesc(C.Structure):
    _fields_ = [
        ("n_docs", C.c_uint64), ("d", C.c_uint32), ("dtype", C.c_uint32),
        ("d_cls", C.c_uint32), ("value_width", C.c_uint32), ("alignment", C.c_uint32),
        ("flags", C.c_uint32), ("row_ptr", C.c_void_p), ("rows", C.c_void_p),
        ("device", C.c_int32), ("shard_count", C.c_uint32), ("shard_index", C.c_uint32),
        ("resident", C.c_void_p), ("reserved", C.c_uint32 * 4),
    ]


class TableInfo(C.Structure):
    _fields_ = [
        ("n_docs", C.c_uint64), ("n_tokens", C.c_uint64), ("d", C.c_uint32),
        ("dtype", C.c_uint32), ("max_tokens", C.c_uint32), ("min_tokens", C.c_uint32),
        ("hbm_bytes", C.c_uint64), ("host_bytes", C.c_uint64), ("resident_docs", C.c_uint64),
    ]


class WorkspaceDesc(C.Structure):
    _fields_ = [
        ("max_queries", C.c_uint32), ("max_candidates", C.c_uint32),
        ("max_query_tokens", C.c_uint32), ("max_list", C.c_uint32), ("staging_bytes", C.c_uint64),
        ("reserved", C.c_uint32 * 2),
    ]


class RerankArgs(C.Structure):
    _fields_ = [
        ("n_queries", C.c_uint32), ("n_query_tokens", C.c_uint32),
        ("query_tokens", C.c_void_p), ("cand_ids", C.c_void_p), ("cand_cls", C.c_void_p),
        ("cand_offsets", C.c_void_p), ("rerank_count", C.c_uint32), ("final_k", C.c_uint32),
        ("alpha", C.c_float), ("flags", C.c_uint32), ("kernel", C.c_uint32),
        ("needed_counts", C.c_void_p), ("reserved", C.c_uint32 * 3),
    ]


class FetchStats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("needed", "resident", "prefetched", "missed", "prefetch_bytes",
                                          "critical_bytes")]


class RerankOut(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p), ("scores", C.c_void_p), ("counts", C.c_void_p),
        ("bow_scores", C.c_void_p), ("fetch_stats", C.c_void_p),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("batches", C.c_uint64), ("queries", C.c_uint64), ("pairs_scored", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("profiled_batches", C.c_uint64),
        ("maxsim_ms", C.c_double), ("topk_ms", C.c_double), ("maxsim_device_ns", C.c_uint64),
        ("maxsim_device_launches", C.c_uint64),
    ]


# name -> (restype, argtypes); every symbol declared in include/espn_gpu.h
SIGNATURES = {
    "espn_gpu_table_open": (C.c_int, [C.POINTER(TableDesc), C.POINTER(C.c_void_p)]),
    "espn_gpu_table_close": (C.c_int, [C.c_void_p]),
    "espn_gpu_table_load_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "espn_gpu_table_info": (C.c_int, [C.c_void_p, C.POINTER(TableInfo)]),
    "espn_gpu_workspace_create": (C.c_int, [C.c_void_p, C.POINTER(WorkspaceDesc), C.POINTER(C.c_void_p)]),
    "espn_gpu_workspace_destroy": (C.c_int, [C.c_void_p]),
    "espn_gpu_rerank": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RerankArgs), C.POINTER(RerankOut), C.c_void_p]),
    "espn_gpu_workspace_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "espn_gpu_workspace_cand_status": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "espn_gpu_prefetch": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RerankArgs), C.c_void_p]),
    "espn_gpu_prefetch_hints": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                          C.c_void_p]),
    "espn_gpu_prefetch_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_uint64, C.c_void_p]),
    "espn_gpu_gather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "espn_gpu_gather_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64]),
    "espn_gpu_merge_topk": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_gpu_get_counters": (C.c_int, [C.c_void_p, C.POINTER(Counters)]),
    "espn_gpu_debug_timeline": (C.c_int, [C.c_int, C.c_void_p, C.c_int]),
    "espn_gpu_synth_table": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_gpu_gather_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_gpu_server_start": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32]),
    "espn_gpu_server_stop": (C.c_int, [C.c_void_p]),
    "espn_gpu_server_pause": (C.c_int, [C.c_void_p]),
    "espn_gpu_server_running": (C.c_int, [C.c_void_p]),
    "espn_gpu_server_debug": (C.c_int, [C.c_void_p, C.c_void_p]),
    "espn_nccl_get_unique_id": (C.c_int, [C.c_void_p]),
    "espn_nccl_comm_init": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "espn_nccl_comm_init_all": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p]),
    "espn_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "espn_gpu_rerank_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RerankArgs), C.POINTER(RerankOut),
                                          C.c_void_p, C.c_void_p]),
    "espn_gpu_rerank_sharded_multi": (C.c_int, [C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(RerankArgs),
                                                C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_gpu_shard_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RerankArgs), C.c_uint32, C.c_uint32,
                                      C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "espn_gpu_shard_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RerankArgs), C.c_void_p, C.c_uint32,
                                       C.POINTER(RerankOut), C.c_void_p]),
    "espn_gpu_maxsim_f32": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                      C.c_int]),
    "espn_gpu_rank": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int]),
    "espn_last_error": (C.c_char_p, []),
    "espn_abi_version": (C.c_int, []),
}

_lib = None


def lib() -> C.CDLL:
    """Load libespn_gpu.so (once).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2312_05417_b200.build` "
                "(the re-rank path has no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def last_error() -> str:
    return (lib().espn_last_error() or b"").decode("utf-8", "replace")


# ---- include/espn_store.h: the on-disk .espn store (libespn_store.so, host only) ----
STORE_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libespn_store.so"


class StoreHeader(C.Structure):
    _fields_ = [("version", C.c_uint32), ("d", C.c_uint32), ("d_cls", C.c_uint32), ("value_width", C.c_uint32),
                ("alignment", C.c_uint32), ("count", C.c_uint64)]


class ManifestRecord(C.Structure):  # store.hpp:13-18
    _fields_ = [("byte_offset", C.c_uint64), ("byte_length", C.c_uint32), ("token_count", C.c_uint32)]


STORE_SIGNATURES = {
    "espn_store_build": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_store_load_manifest": (C.c_int, [C.c_char_p, C.POINTER(StoreHeader), C.c_void_p]),
    "espn_store_read_table": (C.c_int, [C.c_char_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "espn_store_save_manifest": (C.c_int, [C.c_char_p, C.POINTER(StoreHeader), C.c_void_p]),
    "espn_store_open": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p), C.POINTER(StoreHeader)]),
    "espn_store_close": (C.c_int, [C.c_void_p]),
    "espn_store_records": (C.c_int, [C.c_void_p, C.c_void_p]),
    "espn_store_fetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
    "espn_store_read_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]),
    "espn_store_last_error": (C.c_char_p, []),
}

_store_lib = None


def store_lib() -> C.CDLL:
    """Load libespn_store.so (once).  Raises if it is missing."""
    global _store_lib
    if _store_lib is None:
        if not STORE_LIB_PATH.exists():
            raise RuntimeError(f"{STORE_LIB_PATH} not found: build it with `python -m paper_2312_05417_b200.build`")
        h = C.CDLL(str(STORE_LIB_PATH))
        for name, (res, args) in STORE_SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _store_lib = h
    return _store_lib


def store_last_error() -> str:
    return (store_lib().espn_store_last_error() or b"").decode("utf-8", "replace")


# ---- include/espn_host.h: the C++ host layer (libespn_host.so) ------------------------
HOST_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libespn_host.so"
HOST_SIGNATURES = {
    "espn_host_run_batches": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                        C.c_void_p, C.c_uint32, C.POINTER(C.c_double)]),
}
_host_lib = None


def host_lib() -> C.CDLL:
    """Load libespn_host.so (once; it links libespn_gpu.so).  Raises if missing."""
    global _host_lib
    if _host_lib is None:
        lib()  # the GPU library first (same copy the host layer links, via rpath $ORIGIN)
        if not HOST_LIB_PATH.exists():
            raise RuntimeError(f"{HOST_LIB_PATH} not found: build it with `python -m paper_2312_05417_b200.build`")
        h = C.CDLL(str(HOST_LIB_PATH))
        for name, (res, args) in HOST_SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _host_lib = h
    return _host_lib
