"""Profiling experiment (not product): per warp role of the MaxSim kernel,
the share of its time spent waiting on mbarriers (ESPN_DEBUG bit 8, summed
over all CTAs and batches) for the served C2 step -- the role that never
waits is the bottleneck.  The accounting is compiled in only with
-DESPN_ROLE_PROFILE (it costs ~15% even when not executed):
  ESPN_NVCC_DEFINES=-DESPN_ROLE_PROFILE python -c "from paper_2312_05417_b200 import build as b; b.build_lib(force=True)"
  python tools/role_profile.py [on|off]
(rebuild without the define afterwards)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["ESPN_DEBUG"] = "8"
serve = (sys.argv[1] if len(sys.argv) > 1 else "on") == "on"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_05417_b200 import _lib as L, api  # noqa: E402

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
B, K, R, k = cfg["batch"], cfg["K"], cfg["R"], cfg["k"]
batches = bench.make_batches(cfg, 8, B)
dbs = [dict(q=torch.from_numpy(b["q"]).to(dev), ids=torch.from_numpy(b["ids"].view(np.int32)).to(dev),
            cls=torch.from_numpy(b["cls"]).to(dev), off=b["off"]) for b in batches]
pcfg = api.PipelineConfig(rerank_count=R, final_k=k)
lanes = []
for _ in range(3):
    rr = api.Reranker(store, B, B * K, 32, max_list=K)
    out = (torch.zeros((B, k), dtype=torch.int32, device=dev), torch.zeros((B, k), dtype=torch.float32, device=dev),
           torch.zeros(B, dtype=torch.int32, device=dev), None)
    lanes.append((rr, torch.cuda.Stream(), out))
if serve:
    store.server_start(idle_us=2_000_000)
buf = (C.c_uint64 * (8 + 1024))()
KINDS = ["full", "empty", "tfull", "tempty", "ufull", "uempty", "edone", "bdone", "bfree", "patched"]


def run(n):
    for i in range(n):
        rr, s, out = lanes[i % 3]
        db = dbs[i % len(dbs)]
        rr.rerank_arrays(db["q"], db["ids"], db["cls"], db["off"], pcfg, device_io=True, out=out,
                         stream=s.cuda_stream, sync=False)
    for rr, s, _ in lanes:
        s.synchronize()
        rr.sync(s.cuda_stream)


run(30)
if serve:
    store.server_stop()
lib.espn_gpu_debug_timeline(0, None, 1)  # reset
if serve:
    store.server_start(idle_us=2_000_000)
run(200)
if serve:
    store.server_stop()
lib.espn_gpu_debug_timeline(0, buf, 2)
a = np.array(buf[8:8 + 34], dtype=np.float64).reshape(17, 2)
names = ["epi q0 h0", "epi q1 h0", "epi q2 h0", "epi q3 h0", "epi q0 h1", "epi q1 h1", "epi q2 h1", "epi q3 h1",
         "MMA", "producer 0", "producer 1", "loader", "combine", "dedup", "rank", "query tile", "pad patch"]
print(f"server={'on' if serve else 'off'}: per warp role, busy share = 1 - waiting / total (all CTAs, 200 batches)")
kb = np.array(buf[8 + 64:8 + 64 + 17 * 12], dtype=np.float64).reshape(17, 12)
for i, (n, (tot, w)) in enumerate(zip(names, a)):
    parts = ", ".join(f"{KINDS[j]} {100 * kb[i, j] / max(tot, 1):.1f}" for j in range(10) if kb[i, j] > 0.005 * tot)
    print(f"  {n:12s} total {tot / 1e9:8.3f} Gcyc  waiting {100 * w / max(tot, 1):5.1f} %  busy "
          f"{100 * (1 - w / max(tot, 1)):5.1f} %   [{parts}]")
