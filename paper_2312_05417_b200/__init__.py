"""B200-native ESPN re-ranking hot path (gather -> MaxSim -> top-k).

The compute lives in lib/libespn_gpu.so (CUDA for sm_100a behind the C-ABI in
include/espn_gpu.h); this package is the reference-shaped host mirror.
"""
from .api import (  # noqa: F401
    BatchResult, BatchStats, Candidate, CandidateList, DataIntegrityError, EmbeddingMatrix, Error,
    FetchResult, FormatError, GpuStore, InvalidConfigError, InvalidInputError, InvalidStateError,
    IoError, PipelineConfig, QueryEmbedding, QueryStats, RankedList, Reranker, ScoredDoc,
    rerank_batch, rerank_candidates,
)

__all__ = [
    "BatchResult", "BatchStats", "Candidate", "CandidateList", "DataIntegrityError", "EmbeddingMatrix",
    "Error", "FetchResult", "FormatError", "GpuStore", "InvalidConfigError", "InvalidInputError",
    "InvalidStateError", "IoError", "PipelineConfig", "QueryEmbedding", "QueryStats", "RankedList",
    "Reranker", "ScoredDoc", "rerank_batch", "rerank_candidates",
]
