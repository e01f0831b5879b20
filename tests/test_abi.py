"""CPU: the C-ABI library loads, exports every symbol include/espn_gpu.h
declares, the ctypes mirror matches the C struct layouts, and device calls
fail loudly (ESPN_E_CUDA) on a host without a GPU -- no CPU fallback."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "espn_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"ESPN_API\s+[\w\s\*]+?\b(espn_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["espn_gpu_table_open", "espn_gpu_rerank", "espn_gpu_gather", "espn_gpu_merge_topk",
              "espn_gpu_workspace_create", "espn_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2312_05417_b200 import _lib as L
    lib = L.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in L.SIGNATURES, f"ctypes mirror lacks {s}"
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (espn_\w+)", out))
    assert exported == set(declared_symbols()), exported ^ set(declared_symbols())
    assert lib.espn_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against the header and compare sizeof/offsetof with ctypes."""
    from paper_2312_05417_b200 import _lib as L
    structs = {"espn_table_desc": L.TableDesc, "espn_table_info": L.TableInfo,
               "espn_workspace_desc": L.WorkspaceDesc, "espn_rerank_args": L.RerankArgs,
               "espn_rerank_out": L.RerankOut, "espn_counters": L.Counters}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c99", "-o", str(exe), str(src)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.split("\n") if l)
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; covered by the gpu tests")
    import numpy as np
    from paper_2312_05417_b200 import api
    rp = np.array([0, 2], np.uint64)
    with pytest.raises(api.Error, match="no CUDA device"):
        api.GpuStore(rp, np.zeros(64, np.uint16), 32)


def test_product_does_not_import_oracle():
    pat = re.compile(r"^\s*(import\s+oracle|from\s+oracle|import\s+oracle_py|from\s+oracle_py)|libespn_oracle",
                     re.M)
    for p in (ROOT / "paper_2312_05417_b200").rglob("*.py"):
        assert not pat.search(p.read_text()), p
    for p in (ROOT / "paper_2312_05417_b200" / "csrc").rglob("*"):
        if p.is_file():
            assert "espn_oracle" not in p.read_text(), p
    assert "espn_oracle" not in (ROOT / "paper_2312_05417_b200" / "build.py").read_text()


def test_store_library_exports_and_layouts(tmp_path):
    """include/espn_store.h: libespn_store.so exports exactly the declared
    symbols and the ctypes mirror matches the header's struct layouts."""
    from paper_2312_05417_b200 import _lib as L
    hdr = ROOT / "include" / "espn_store.h"
    syms = set(re.findall(r"ESPN_API\s+[\w\s\*]+?\b(espn_\w+)\s*\(", hdr.read_text()))
    assert syms == set(L.STORE_SIGNATURES)
    lib = L.store_lib()
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.STORE_LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert set(re.findall(r"\bT (espn_\w+)", out)) == syms
    for s in syms:
        assert hasattr(lib, s)
    structs = {"espn_store_header": L.StoreHeader, "espn_manifest_record": L.ManifestRecord}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{hdr}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    (tmp_path / "p.c").write_text("\n".join(lines))
    subprocess.run(["gcc", "-std=c99", "-o", str(tmp_path / "p"), str(tmp_path / "p.c")], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(tmp_path / "p")], capture_output=True, text=True,
                                                         check=True).stdout.split("\n") if l)
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"
    from paper_2312_05417_b200 import api
    assert C.sizeof(L.ManifestRecord) == api._RECORD_DT.itemsize == 16
