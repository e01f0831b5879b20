# Measurement behind ESPN_KERNEL_AUTO: tcgen05 vs CUDA-core (SIMT) MaxSim per dim,
# C2-shaped batch (64 queries x 1000 candidates, t~U{1..63}) on a 2M-doc table.
#   python tools/kernel_choice.py
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2312_05417_b200 import _lib as L, api, synth
dev = torch.device("cuda", 0)
lib = L.lib()
N, B, K = 2_000_000, 64, 1000
out = []
for d in (8, 16, 32, 48, 64, 128):
    if d in (16, 32, 64, 128):  # device generator (tensor-core dims, tile layout)
        n = N
        rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        assert lib.espn_gpu_synth_table(n, d, 0, 1, 63, 7, 1, 0, rp.data_ptr(), None, None) == 0
        rows = torch.empty(int(rp[-1]) * d, dtype=torch.int16, device=dev)
        assert lib.espn_gpu_synth_table(n, d, 0, 1, 63, 7, 1, 0, rp.data_ptr(), rows.data_ptr(), None) == 0
        store = api.GpuStore.from_device(rp, rows, d, "f16", rows_tiled=True)
    else:  # other dims: host generator, smaller table
        n = 300_000
        hrp, hcodes = synth.make_table(n, d, 1, 63, seed=7)
        rp = rows = None
        store = api.GpuStore(hrp, hcodes, d, "f16")
    rr = api.Reranker(store, B, B * K, 32)
    rng = np.random.default_rng(1)
    q = torch.from_numpy((rng.standard_normal((B, 32, d)) / np.sqrt(d)).astype(np.float32)).to(dev)
    ids = torch.from_numpy(np.stack([rng.choice(n, K, replace=False) for _ in range(B)]).astype(np.int32).ravel()).to(dev)
    cls = torch.from_numpy(np.sort(rng.random(B * K).astype(np.float32))[::-1].copy()).to(dev)
    off = np.arange(B + 1, dtype=np.uint64) * K
    cfg = api.PipelineConfig(rerank_count=K, final_k=10)
    row = {"d": d, "n_docs": n}
    for kern in ("tcgen05", "simt"):
        try:
            for _ in range(3):
                rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kern, device_io=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                rr.rerank_arrays(q, ids, cls, off, cfg, kernel=kern, device_io=True, sync=False)
            e1.record()
            rr.sync()
            torch.cuda.synchronize()
            row[kern + "_ms"] = e0.elapsed_time(e1) / 20
        except api.Error as e:
            row[kern + "_ms"] = None
            row[kern + "_why"] = str(e)[:80]
    out.append(row)
    print(json.dumps(row), flush=True)
    rr.close(); store.close()
    del rows, rp
    torch.cuda.empty_cache()
