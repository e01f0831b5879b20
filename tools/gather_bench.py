# K1 standalone gather (espn_gpu_gather, StoreHandle::fetch_batch restated)
# on the C2 table: 64 x 1000 random doc ids per call (one batch's candidates).
#   python tools/gather_bench.py [--reps 20]
# Algorithmic bytes per call = gathered tokens x 64 B read + the same written.
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import bench
from paper_2312_05417_b200 import _lib as L, api

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--n", type=int, default=64000)
a = ap.parse_args()
cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
lib = L.lib()
N, d = cfg["n_docs"], cfg["d"]
row_ptr = torch.zeros(N + 1, dtype=torch.int64, device=dev)
assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, row_ptr.data_ptr(), None, None) == 0
rows = torch.empty(int(row_ptr[-1]) * d, dtype=torch.int16, device=dev)
assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, row_ptr.data_ptr(),
                                rows.data_ptr(), None) == 0
store = api.GpuStore.from_device(row_ptr, rows, d, "f16", rows_tiled=True)
rng = np.random.default_rng(3)
sets = [torch.from_numpy(rng.integers(0, N, a.n).astype(np.int32)).to(dev) for _ in range(4)]
rp = torch.zeros(a.n + 1, dtype=torch.int64, device=dev)
out = torch.empty(a.n * 64 * d, dtype=torch.int16, device=dev)
times, toks = [], []
for r in range(a.reps + 3):
    ids = sets[r % 4]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.espn_gpu_gather(store.handle, ids.data_ptr(), a.n, out.data_ptr(), rp.data_ptr(), a.n * 64, None)
    t1 = time.perf_counter()
    assert rc == 0, L.last_error()
    if r >= 3:
        times.append(t1 - t0)
        toks.append(int(rp[-1]))
tok = float(np.mean(toks))
alg = tok * d * 2 * 2
print(json.dumps({"ids_per_call": a.n, "tokens_per_call": tok, "alg_bytes_per_call": alg,
                  "call_ms_median": float(np.median(times)) * 1e3,
                  "call_gbs": alg / float(np.median(times)) / 1e9,
                  "note": "call = count kernel + scan + host sync + copy kernel + sync; the copy kernel alone is in "
                          "the ncu launch list"}))
