"""In-tree build of the native library (no JIT cache, so the .so travels with
the repo snapshot to the GPU box).

    python -m paper_2312_05417_b200.build        # libespn_gpu.so + libespn_host.so

libespn_gpu.so = csrc/espn_gpu.cu (+ headers) compiled for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`: plain -arch=sm_100a would also
emit compute_100 PTX, on which ptxas rejects tcgen05).  Host C++ lives in the
same translation unit; the library links only the CUDA runtime.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libespn_gpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "espn_gpu.h"]


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources())


def build_lib(verbose: bool = False, force: bool = False) -> Path:
    if not force and not needs_rebuild():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    # ESPN_NVCC_DEFINES: extra -D flags for measurement builds (e.g. -DESPN_ROLE_PROFILE
    # for tools/role_profile.py); production builds leave it unset
    extra = os.environ.get("ESPN_NVCC_DEFINES", "").split()
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(tmp), str(CSRC / "espn_gpu.cu"),
           "-lcudart"]
    if verbose:
        cmd.insert(1, "-Xptxas")
        cmd.insert(2, "-v")
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libespn_gpu.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


HOST_LIB = LIB_DIR / "libespn_host.so"
CUDA_INC = "/usr/local/cuda/include"
CUDA_LIB = "/usr/local/cuda/lib64"
HOST_SRC = CSRC / "host" / "espn_b200.cpp"
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-fvisibility=default"]


def build_host(force: bool = False) -> Path:
    """libespn_host.so: the C++ espn::gpu API (include/espn_b200.hpp) over the
    C-ABI, linked against libespn_gpu.so (rpath $ORIGIN)."""
    build_store_lib()
    deps = [HOST_SRC, ROOT / "include" / "espn_b200.hpp", ROOT / "include" / "espn_gpu.h",
            ROOT / "include" / "espn_host.h", LIB, STORE_LIB]
    if not force and HOST_LIB.exists() and all(p.stat().st_mtime <= HOST_LIB.stat().st_mtime for p in deps):
        return HOST_LIB
    cmd = [CXX, *CXX_FLAGS, "-shared", "-I", str(ROOT / "include"), "-I", CUDA_INC, "-o", str(HOST_LIB),
           str(HOST_SRC), "-L", str(LIB_DIR), "-lespn_gpu", "-lespn_store", "-L", CUDA_LIB, "-lcudart",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libespn_host.so")
    return HOST_LIB


STORE_SRC = CSRC / "host" / "espn_store.cpp"
STORE_LIB = LIB_DIR / "libespn_store.so"


def build_store_lib(force: bool = False) -> Path:
    """libespn_store.so: the on-disk .espn store (include/espn_store.h), pure
    host C++ -- builds and runs without a GPU."""
    deps = [STORE_SRC, ROOT / "include" / "espn_store.h", ROOT / "include" / "espn_gpu.h"]
    if not force and STORE_LIB.exists() and all(p.stat().st_mtime <= STORE_LIB.stat().st_mtime for p in deps):
        return STORE_LIB
    LIB_DIR.mkdir(exist_ok=True)
    cmd = [CXX, *CXX_FLAGS, "-shared", "-fvisibility=hidden", "-I", str(ROOT / "include"), "-o", str(STORE_LIB),
           str(STORE_SRC)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libespn_store.so")
    return STORE_LIB


REFAPI_SRC = CSRC / "host" / "espn_ref_api.cpp"
REFAPI_LIB = LIB_DIR / "libespn_refapi.so"
REF_INC = Path("/root/reference/proj/include")


def build_refapi(force: bool = False) -> Path | None:
    """lib/libespn_refapi.so: the reference's declarations (its UNMODIFIED
    headers) defined over the B200 path -- espn_ref_api.cpp plus the C++ host
    layer compiled with the reference's carrier types.  Built where the
    reference headers exist (this container); the .so ships with the tree."""
    if not REF_INC.exists():
        return REFAPI_LIB if REFAPI_LIB.exists() else None
    build_store_lib()
    deps = [REFAPI_SRC, HOST_SRC, ROOT / "include" / "espn_b200.hpp", ROOT / "include" / "espn_gpu.h",
            ROOT / "include" / "espn_store.h", ROOT / "include" / "espn_host.h", LIB, STORE_LIB]
    if not force and REFAPI_LIB.exists() and all(p.stat().st_mtime <= REFAPI_LIB.stat().st_mtime for p in deps):
        return REFAPI_LIB
    cmd = [CXX, *CXX_FLAGS, "-ffp-contract=off", "-shared", "-DESPN_B200_WITH_REFERENCE_HEADERS",
           "-I", str(ROOT / "include"), "-I", str(REF_INC), "-I", CUDA_INC, "-o", str(REFAPI_LIB), str(REFAPI_SRC),
           str(HOST_SRC), "-L", str(LIB_DIR), "-lespn_gpu", "-lespn_store", "-L", CUDA_LIB, "-lcudart",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libespn_refapi.so against the reference headers")
    return REFAPI_LIB


def check_reference_headers() -> bool:
    """Compile the C++ host API against the reference's own headers (source
    compatibility of the drop-in), where /root/reference exists."""
    inc = Path("/root/reference/proj/include")
    if not inc.exists():
        return False
    cmd = [CXX, *CXX_FLAGS, "-fsyntax-only", "-DESPN_B200_WITH_REFERENCE_HEADERS", "-I", str(ROOT / "include"),
           "-I", CUDA_INC, "-I", str(inc), str(HOST_SRC)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("C++ host API does not compile against the reference headers")
    return True


if __name__ == "__main__":
    build_lib(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_host(force="-f" in sys.argv)
    build_store_lib(force="-f" in sys.argv)
    build_refapi(force="-f" in sys.argv)
    print(LIB)
