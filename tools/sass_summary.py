"""SASS instruction counts per kernel of the built libespn_gpu.so -- the
evidence that the hot kernels use tcgen05 (UTCHMMA / UTCBAR / LDTM / UTCATOMSWS
= TMEM alloc), TMA bulk copies (UBLKCP) and mbarriers (SYNCS).
usage: python tools/sass_summary.py > profiles/sass_r2.json"""
import json
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2312_05417_b200" / "lib" / "libespn_gpu.so"
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "UTCATOMSWS", "UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "ATOMS", "REDG",
       "FFMA", "FMUL", "FADD", "FMNMX3", "FMNMX", "SHFL", "ELECT"]
out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
res, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        res[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o:
                res[cur][o] = res[cur].get(o, 0) + 1
keep = {k: v for k, v in res.items() if re.search(r"maxsim|small|gather_copy|plan_kernel|finalize|stage_kernel|topk", k)}
json.dump({"library": str(LIB.name), "kernels": keep}, sys.stdout, indent=1)
