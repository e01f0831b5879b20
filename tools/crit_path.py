# Profiling experiment: pieces of the f1 critical path (rerank of a staged batch, host arrays).
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2312_05417_b200 import api, synth
rp, codes = synth.make_table(200000, 32, 1, 63, seed=41)
q, src = synth.make_queries(rp, codes, 32, 64, nq=32, seed=42)
ids, cls, off = synth.make_candidates(200000, 64, 1000, src=src, seed=43)
for res_frac in (1.0, 0.0):
    resident = (np.random.default_rng(1).random(200000) < res_frac).astype(np.uint8)
    store = api.GpuStore(rp, codes, 32, "f16", resident=None if res_frac == 1.0 else resident)
    rr = api.Reranker(store, 64, 64000, 32, staging_bytes=512 << 20)
    cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
    side = torch.cuda.Stream()
    for mode in ("plain", "hinted_all"):
        ts = []
        for r in range(12):
            if mode == "hinted_all":
                rr.prefetch_hints(ids, off, stream=side.cuda_stream)
                side.synchronize()
            t0 = time.perf_counter()
            out = rr.rerank_arrays(q, ids, cls, off, cfg, prefetched=(mode == "hinted_all"), fetch_stats=True)
            ts.append(time.perf_counter() - t0)
        t_nofs = []
        for r in range(12):
            if mode == "hinted_all":
                rr.prefetch_hints(ids, off, stream=side.cuda_stream)
                side.synchronize()
            t0 = time.perf_counter()
            out = rr.rerank_arrays(q, ids, cls, off, cfg, prefetched=(mode == "hinted_all"))
            t_nofs.append(time.perf_counter() - t0)
        print(f"resident={res_frac} {mode}: call {np.median(ts[2:])*1e3:.3f} ms (no fetch_stats {np.median(t_nofs[2:])*1e3:.3f} ms)")
    rr.close(); store.close()
