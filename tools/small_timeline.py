"""Per-CTA phase timeline of the single-launch small-batch kernel (ESPN_DEBUG=8):
configs[0] shape (100k docs, t <= 32, d=32, batch 1 x 1000 candidates)."""
import os
import sys
import ctypes as C
from pathlib import Path

os.environ["ESPN_DEBUG"] = "8"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2312_05417_b200 import _lib as L, api, synth  # noqa: E402

rp, codes = synth.make_table(100000, 32, 1, 32, seed=3)
store = api.GpuStore(rp, codes, 32)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rr = api.Reranker(store, B, B * 1000, 32)
cfg = api.PipelineConfig(rerank_count=1000, final_k=10)
lib = L.lib()
buf = (C.c_uint64 * (8 + 1024))()
rows = []
for it in range(30):
    q, src = synth.make_queries(rp, codes, 32, B, seed=10 + it)
    ids, cls, off = synth.make_candidates(100000, B, 1000, src=src, seed=50 + it)
    lib.espn_gpu_debug_timeline(0, buf, 1)  # reset
    rr.rerank_arrays(q, ids, cls, off, cfg, kernel="small")
    lib.espn_gpu_debug_timeline(0, buf, 2)
    st = np.array(buf[8:], dtype=np.uint64).reshape(256, 4)
    used = st[:, 0] > 0
    s = st[used].astype(np.float64)
    last = (st[used, 3] >> 63).astype(bool)
    s[:, 3] = (st[used, 3] & ((1 << 63) - 1)).astype(np.float64)
    t0 = s[:, 0].min()
    if it >= 5:
        rows.append([s[:, 0].max() - t0, np.median(s[:, 1] - s[:, 0]), np.median(s[:, 2] - s[:, 1]),
                     np.median(s[~last, 3] - s[~last, 2]), s[last, 3].max() - s[last, 2].max(),
                     s[:, 3].max() - t0, used.sum()])
r = np.array(rows)
print("ns (median over 25 calls): start spread | inputs ready | scored | arrive | last-CTA merge | total | CTAs")
print(" ".join(f"{x:9.0f}" for x in np.median(r, axis=0)))
