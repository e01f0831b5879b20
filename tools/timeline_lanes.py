# Profiling experiment: CTA-0 role trace (ESPN_DEBUG bit 8) of MaxSim launches
# in the bench's steady state -- 3 lanes (streams + workspaces) in flight, C2.
#   ESPN_DEBUG=8 python tools/timeline_lanes.py
import os
import sys
from pathlib import Path
os.environ.setdefault("ESPN_DEBUG", "8")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2312_05417_b200 import _lib as L, api

cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
lib = L.lib()
N, d = cfg["n_docs"], cfg["d"]
rp = torch.zeros(N + 1, dtype=torch.int64, device=dev)
assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(), None, None) == 0
rows = torch.empty(int(rp[-1]) * d, dtype=torch.int16, device=dev)
assert lib.espn_gpu_synth_table(N, d, 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(), rows.data_ptr(), None) == 0
store = api.GpuStore.from_device(rp, rows, d, "f16", rows_tiled=True)
B, K = cfg["batch"], cfg["K"]
bts = bench.make_batches(cfg, 6, B)
dbs = [dict(q=torch.from_numpy(b["q"]).to(dev), ids=torch.from_numpy(b["ids"].view(np.int32)).to(dev),
            cls=torch.from_numpy(b["cls"]).to(dev), off=b["off"]) for b in bts]
pcfg = api.PipelineConfig(rerank_count=cfg["R"], final_k=cfg["k"])
lanes = [(api.Reranker(store, B, B * K, 32), torch.cuda.Stream()) for _ in range(3)]
outs = [(torch.empty((B, 10), dtype=torch.int32, device=dev), torch.empty((B, 10), dtype=torch.float32, device=dev),
         torch.empty(B, dtype=torch.int32, device=dev), None) for _ in range(3)]
torch.cuda.synchronize()
for i in range(9):
    rr, st = lanes[i % 3]
    db = dbs[i % 6]
    rr.rerank_arrays(db["q"], db["ids"], db["cls"], db["off"], pcfg, device_io=True, out=outs[i % 3],
                     stream=st.cuda_stream, sync=False)
torch.cuda.synchronize()
for rr, st in lanes:
    rr.sync(st.cuda_stream)
print("done", flush=True)
