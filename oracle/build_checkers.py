"""Builds the CHECKERS (test infrastructure only): the CPU oracle
(oracle/_build/libespn_oracle.so), the reference-codec shim (oracle/_ref, only
where /root/reference exists) and the C++ API test driver
(tests/cpp/host_api_test, links the oracle).  Never imported by the product
package; called by __graft_entry__.build() and the tests.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(ROOT))
from paper_2312_05417_b200.build import CXX, HOST_LIB, LIB_DIR, REF_INC, REFAPI_LIB  # noqa: E402


def build_oracle() -> None:
    """Oracle (test infrastructure) + the reference codec shim when the
    reference tree is present (this container only)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    if Path("/root/reference/proj/include/espn/half.hpp").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)


def build_cpp_tests() -> Path:
    """tests/cpp/host_api_test: drives the C++ API on the GPU and checks it
    against the CPU oracle (test infrastructure: links oracle/_build)."""
    out = ROOT / "tests" / "cpp" / "host_api_test"
    src = ROOT / "tests" / "cpp" / "host_api_test.cpp"
    deps = [src, HOST_LIB, ROOT / "include" / "espn_b200.hpp", HERE / "espn_oracle.h", HERE / "_build" / "libespn_oracle.so"]
    if out.exists() and all(p.stat().st_mtime <= out.stat().st_mtime for p in deps):
        return out
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle"), "-o", str(out),
           str(src), "-L", str(LIB_DIR), "-lespn_host", "-lespn_gpu", "-lespn_store", "-L", str(ROOT / "oracle" / "_build"),
           "-lespn_oracle", f"-Wl,-rpath,{LIB_DIR}", f"-Wl,-rpath,{ROOT / 'oracle' / '_build'}",
           "-Wl,-rpath,$ORIGIN/../../paper_2312_05417_b200/lib", "-Wl,-rpath,$ORIGIN/../../oracle/_build"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building tests/cpp/host_api_test")
    return out


def build_refapi_test() -> Path | None:
    """tests/cpp/refapi_test: a program written against the reference's
    UNMODIFIED headers, linked with lib/libespn_refapi.so, checked against the
    oracle.  Compiled where the reference headers exist (this container); the
    binary ships with the tree and runs on the GPU box."""
    out = ROOT / "tests" / "cpp" / "refapi_test"
    if not REF_INC.exists():
        return out if out.exists() else None
    src = ROOT / "tests" / "cpp" / "refapi_test.cpp"
    deps = [src, REFAPI_LIB, HERE / "espn_oracle.h", HERE / "_build" / "libespn_oracle.so"]
    if out.exists() and all(p.stat().st_mtime <= out.stat().st_mtime for p in deps):
        return out
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", str(REF_INC), "-I", str(ROOT / "oracle"), "-o", str(out), str(src),
           "-L", str(LIB_DIR), "-lespn_refapi", "-L", str(ROOT / "oracle" / "_build"), "-lespn_oracle",
           "-Wl,-rpath,$ORIGIN/../../paper_2312_05417_b200/lib", "-Wl,-rpath,$ORIGIN/../../oracle/_build"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building tests/cpp/refapi_test")
    return out
