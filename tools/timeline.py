# Profiling experiment (not product): per-kernel device timeline of the C2
# step under CUDA-graph replay and eager ASYNC calls (ESPN_DEBUG bit 256).
#   python tools/timeline.py [--config c2] [--dbg 0x100]
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--dbg", default="0x100")
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--batches", type=int, default=4)
ap.add_argument("--shards", type=int, default=1)
args = ap.parse_args()
os.environ["ESPN_DEBUG"] = args.dbg
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import bench
from paper_2312_05417_b200 import _lib as L, api

cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
lib = L.lib()
G = args.shards
n_local = (cfg["n_docs"] + G - 1) // G
row_ptr = torch.zeros(n_local + 1, dtype=torch.int64, device=dev)
assert lib.espn_gpu_synth_table(n_local, cfg["d"], 0, cfg["t_min"], cfg["t_max"], bench.SEED, G, 0,
                                row_ptr.data_ptr(), None, None) == 0
n_tok = int(row_ptr[-1])
rows = torch.empty(n_tok * cfg["d"], dtype=torch.int16, device=dev)
assert lib.espn_gpu_synth_table(n_local, cfg["d"], 0, cfg["t_min"], cfg["t_max"], bench.SEED, G, 0,
                                row_ptr.data_ptr(), rows.data_ptr(), None) == 0
store = api.GpuStore.from_device(row_ptr, rows, cfg["d"], "f16", shard_count=G, shard_index=0, device=0,
                                 rows_tiled=True)
from paper_2312_05417_b200.sharding import split_by_owner
B, K, R, k, nq = cfg["batch"], cfg["K"], cfg["R"], cfg["k"], cfg["nq"]
bts = bench.make_batches(cfg, args.batches, B)
dbs = []
for bt in bts:
    ids, cls, off, need = split_by_owner(bt["ids"], bt["cls"], bt["off"], R, G, 0)
    dbs.append(dict(q=torch.from_numpy(bt["q"]).to(dev), ids=torch.from_numpy(ids.view(np.int32)).to(dev),
                    cls=torch.from_numpy(cls).to(dev),
                    doff=torch.from_numpy(off.astype(np.int64)).to(dev),
                    dneed=torch.from_numpy(need.astype(np.int32)).to(dev)))
rr = api.Reranker(store, B, B * K, nq, max_list=K)
out = torch.zeros(2 * B * k + B, dtype=torch.int32, device=dev)
base = out.data_ptr()
flags = L.ESPN_RERANK_DEVICE_IO | L.ESPN_RERANK_DEVICE_OFFSETS | L.ESPN_RERANK_ASYNC


def enqueue(db, sp):
    a = L.RerankArgs(n_queries=B, n_query_tokens=nq, query_tokens=db["q"].data_ptr(), cand_ids=db["ids"].data_ptr(),
                     cand_cls=db["cls"].data_ptr(), cand_offsets=db["doff"].data_ptr(), rerank_count=R, final_k=k,
                     alpha=1.0, flags=flags, kernel=L.ESPN_KERNEL_AUTO, needed_counts=db["dneed"].data_ptr())
    o = L.RerankOut(ids=base, scores=base + 4 * B * k, counts=base + 8 * B * k)
    assert lib.espn_gpu_rerank(store.handle, rr.handle, C.byref(a), C.byref(o), C.c_void_p(sp)) == 0, L.last_error()


tl = (C.c_uint64 * 8)()


def show(tag):
    lib.espn_gpu_debug_timeline(0, C.cast(tl, C.c_void_p), 1)
    v = list(tl)
    t0 = v[0]
    names = ["plan", "maxsim", "final"]
    s = " ".join(f"{n}[{(v[2*i]-t0)/1e3:6.2f},{(v[2*i+1]-t0)/1e3:6.2f}]" for i, n in enumerate(names))
    print(f"{tag}: {s}  total {(max(v[3], v[5])-t0)/1e3:.2f}us", flush=True)


cap = torch.cuda.Stream()
with torch.cuda.stream(cap):
    for i in range(3):
        enqueue(dbs[i % len(dbs)], cap.cuda_stream)
cap.synchronize()
graphs = []
for db in dbs:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        enqueue(db, torch.cuda.current_stream().cuda_stream)
    graphs.append(g)
st = torch.cuda.current_stream()
for i in range(20):
    graphs[i % len(graphs)].replay()
torch.cuda.synchronize()
lib.espn_gpu_debug_timeline(0, None, 1)
for r in range(args.reps):
    graphs[r % len(graphs)].replay()
    show(f"graph {r}")
# eager, back-to-back: timeline of the last of 5 queued calls
for r in range(3):
    for i in range(4):
        enqueue(dbs[i % len(dbs)], st.cuda_stream)
    torch.cuda.synchronize()
    lib.espn_gpu_debug_timeline(0, None, 1)
    enqueue(dbs[r % len(dbs)], st.cuda_stream)
    show(f"eager {r}")
# steady-state graph step time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
os.environ["ESPN_DEBUG"] = "0"
e0.record()
for i in range(200):
    graphs[i % len(graphs)].replay()
e1.record()
torch.cuda.synchronize()
print(f"graph step (timeline on): {e0.elapsed_time(e1) / 200 * 1e3:.2f} us")
# per-CTA profile of one graph replay
big = (C.c_uint64 * (8 + 1024))()
lib.espn_gpu_debug_timeline(0, None, 1)
graphs[0].replay()
lib.espn_gpu_debug_timeline(0, C.cast(big, C.c_void_p), 2)
v = list(big)
t0 = v[0]
cp = np.array(v[8:8 + 4 * 148], dtype=np.float64).reshape(148, 4)
end = (cp[:, 0] - t0) / 1e3
rk = (cp[:, 1] - t0) / 1e3
dd = (cp[:, 3] - t0) / 1e3
order = np.argsort(-end)
print("slowest CTAs: cta end rank_end dedup_end merges")
for c in order[:12]:
    print(f"  {c:4d} {end[c]:7.2f} {rk[c]:7.2f} {dd[c]:7.2f} {int(cp[c, 2])}")
print("end percentiles", np.percentile(end, [0, 50, 90, 100]).round(2))
print("merges per CTA hist", np.bincount(cp[:, 2].astype(int)))
lib.espn_gpu_debug_timeline(0, None, 1)
graphs[1].replay()
lib.espn_gpu_debug_timeline(0, C.cast(big, C.c_void_p), 3)
v = list(big)
f = v[8:16]
n = max(f[2], 1)
print(f"finalize: warps {f[2]} load {f[0]/n/1e3:.2f}us select {f[1]/n/1e3:.2f}us wait {f[4]/n/1e3:.2f}us "
      f"cands/query {f[3]/n:.1f} first-wait-start {(f[5]/n - v[0])/1e3:.2f}us")
