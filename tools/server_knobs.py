"""Profiling experiment (not product; results with knobs set are NOT valid
rankings): which path bounds the persistent MaxSim server on C2?  Runs the
served C2 step (3 workspaces / streams in flight, device inputs, ASYNC) with
one ESPN_DEBUG knob (common.cuh) and prints the per-batch service time:
  0 = production, 4 = no row copies (compute chain only), 1 = no epilogue,
  2 = no MMAs, 32 = no doc-boundary scan, 3 = neither MMA nor epilogue.
usage: python tools/server_knobs.py <dbg> [server on|off]"""
import os
import sys
from pathlib import Path

dbg = sys.argv[1] if len(sys.argv) > 1 else "0"
os.environ["ESPN_DEBUG"] = dbg
serve = (sys.argv[2] if len(sys.argv) > 2 else "on") == "on"
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
NL = 3
lanes = []
for _ in range(NL):
    rr = api.Reranker(store, B, B * K, 32, max_list=K)
    out = (torch.zeros((B, k), dtype=torch.int32, device=dev), torch.zeros((B, k), dtype=torch.float32, device=dev),
           torch.zeros(B, dtype=torch.int32, device=dev), None)
    lanes.append((rr, torch.cuda.Stream(), out))
if serve:
    store.server_start(idle_us=2_000_000)


def step(i):
    rr, s, out = lanes[i % NL]
    db = dbs[i % len(dbs)]
    rr.rerank_arrays(db["q"], db["ids"], db["cls"], db["off"], pcfg, device_io=True, out=out,
                     stream=s.cuda_stream, sync=False)


def drain():
    for rr, s, _ in lanes:
        s.synchronize()
        try:
            rr.sync(s.cuda_stream)
        except api.Error:
            pass  # knobs make the scores invalid: expected


for i in range(30):
    step(i)
drain()
n = 300
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize() if not serve else None
e0.record()
for _, s, _ in lanes:
    s.wait_event(e0)
for i in range(n):
    step(i)
for _, s, _ in lanes:
    ev = torch.cuda.Event()
    ev.record(s)
    torch.cuda.current_stream().wait_event(ev)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
drain()
if serve:
    store.server_stop()
print(f"dbg={dbg} server={'on' if serve else 'off'}: {ms / n * 1e3:.1f} us per batch, {B * n / ms * 1e3 / 1e6:.3f} M q/s")
