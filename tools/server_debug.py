"""Diagnostics of the persistent server's queue on one small batch."""
import sys, time, ctypes as C
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_05417_b200 import api, synth, _lib as L

def dbg(store, tag):
    o = (C.c_uint64 * 8)()
    rc = L.lib().espn_gpu_server_debug(store.handle, C.addressof(o))
    print(tag, rc, [hex(x) for x in o], flush=True)

rp, codes = synth.make_table(20000, 32, 1, 63, seed=1)
q, src = synth.make_queries(rp, codes, 32, 8, seed=2)
ids, cls, off = synth.make_candidates(20000, 8, 600, src=src, seed=3)
store = api.GpuStore(rp, codes, 32)
rr = api.Reranker(store, 8, int(off[-1]), 32)
cfg = api.PipelineConfig(rerank_count=500, final_k=10)
ref = rr.rerank_arrays(q, ids, cls, off, cfg)
store.server_start(idle_us=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
dbg(store, "after start")
time.sleep(0.01)
dbg(store, "after 10ms")
import torch
mode = sys.argv[2] if len(sys.argv) > 2 else "host"
dq, di, dc = torch.from_numpy(q).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), torch.from_numpy(cls).cuda()
st = torch.cuda.Stream()
for i in range(3):
    try:
        t0 = time.perf_counter()
        if mode == "host":
            got = rr.rerank_arrays(q, ids, cls, off, cfg)
        else:
            got = rr.rerank_arrays(dq, di, dc, off, cfg, device_io=True, stream=st.cuda_stream)
            got = [x.cpu().numpy() for x in got[:3]]
        print("call", i, "ok", np.array_equal(got[0].view(np.uint32), ref[0]), "%.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
    except Exception as e:
        print("call", i, "error", e, "%.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
    dbg(store, f"after call {i}")
time.sleep(0.2)
dbg(store, "after 200ms")
store.server_stop()
print("stopped", flush=True)
