"""Kernel timing harness (dev tool): C2-shaped batch through the C-ABI with
ESPN_RERANK_PROFILE; prints mean MaxSim / top-k kernel ms.  Usage:
  ESPN_DEBUG=<bits> python tools/ktime.py [config] [n]"""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
from paper_2312_05417_b200 import _lib as L, api
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lib = L.lib(); dev = torch.device("cuda", 0)
rp = torch.zeros(cfg["n_docs"] + 1, dtype=torch.int64, device=dev)
assert lib.espn_gpu_synth_table(cfg["n_docs"], cfg["d"], 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(), None, None) == 0
rows = torch.empty(int(rp[-1]) * cfg["d"], dtype=torch.int16, device=dev)
assert lib.espn_gpu_synth_table(cfg["n_docs"], cfg["d"], 0, cfg["t_min"], cfg["t_max"], bench.SEED, 1, 0, rp.data_ptr(), rows.data_ptr(), None) == 0
store = api.GpuStore.from_device(rp, rows, cfg["d"], "f16", rows_tiled=True)
B, K = cfg["batch"], cfg["K"]
bts = bench.make_batches(cfg, 8, B)
rr = api.Reranker(store, B, B * K, 32)
k = cfg["k"]
out = [torch.zeros((B, k), dtype=torch.int32, device=dev), torch.zeros((B, k), dtype=torch.float32, device=dev), torch.zeros(B, dtype=torch.int32, device=dev)]
dbs = [dict(q=torch.from_numpy(b["q"]).to(dev), ids=torch.from_numpy(b["ids"].view(np.int32)).to(dev), cls=torch.from_numpy(b["cls"]).to(dev), off=b["off"], doff=torch.from_numpy(b["off"].astype(np.int64)).to(dev)) for b in bts]
GRAPH = os.environ.get("KT_GRAPH") == "1"
s = torch.cuda.current_stream().cuda_stream
def step(i, prof):
    db = dbs[i % len(dbs)]
    a = L.RerankArgs(n_queries=B, n_query_tokens=32, query_tokens=db["q"].data_ptr(), cand_ids=db["ids"].data_ptr(), cand_cls=db["cls"].data_ptr(), cand_offsets=db["doff"].data_ptr() if GRAPH else db["off"].ctypes.data, rerank_count=cfg["R"], final_k=k, alpha=1.0, flags=L.ESPN_RERANK_DEVICE_IO | L.ESPN_RERANK_ASYNC | (L.ESPN_RERANK_DEVICE_OFFSETS if GRAPH else 0) | (L.ESPN_RERANK_PROFILE if prof else 0), kernel=0)
    o = L.RerankOut(ids=out[0].data_ptr(), scores=out[1].data_ptr(), counts=out[2].data_ptr())
    rc = lib.espn_gpu_rerank(store.handle, rr.handle, C.byref(a), C.byref(o), C.c_void_p(s))
    assert rc == 0 or os.environ.get("ESPN_DEBUG"), L.last_error()
for i in range(10): step(i, False)
torch.cuda.synchronize()
try: rr.sync(s)
except Exception: pass
c0 = rr.counters()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time
graphs = []
if GRAPH:
    s_ = torch.cuda.Stream()
    for i in range(len(dbs)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s_):
            s = torch.cuda.current_stream().cuda_stream
            step(i, False)
        graphs.append(g)
    s = torch.cuda.current_stream().cuda_stream
    for g in graphs: g.replay()
    torch.cuda.synchronize()
e0.record()
h0 = time.perf_counter()
for i in range(n):
    if GRAPH: graphs[i % len(graphs)].replay()
    else: step(i, False)
host_us = (time.perf_counter() - h0) / n * 1e6
e1.record(); torch.cuda.synchronize()
step_us = e0.elapsed_time(e1) / n * 1e3
for i in range(n): step(i, True)
torch.cuda.synchronize()
try: rr.sync(s)
except Exception: pass
c1 = rr.counters()
nb = c1["profiled_batches"] - c0["profiled_batches"]
ms = (c1["maxsim_ms"] - c0["maxsim_ms"]) / nb
print(f"host {host_us:.1f} us/call  step {step_us:.1f} us  ESPN_DEBUG={os.environ.get('ESPN_DEBUG','0')} {sys.argv[1:] } maxsim {ms*1e3:.1f} us  topk {(c1['topk_ms']-c0['topk_ms'])/nb*1e3:.1f} us  ~{131.8e6/(ms/1e3)/1e9:.0f} GB/s")
