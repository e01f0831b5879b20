"""The C++ host API (include/espn_b200.hpp): compiles against the reference's
own headers (source compatibility of the drop-in, CPU) and, on the GPU, runs
tests/cpp/host_api_test (C++ API vs the CPU oracle)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_host_api_compiles_against_reference_headers():
    from paper_2312_05417_b200 import build
    if not Path("/root/reference/proj/include/espn/pipeline.hpp").exists():
        pytest.skip("reference headers not present on this machine")
    assert build.check_reference_headers()


def test_host_library_builds_and_exports():
    from paper_2312_05417_b200 import build
    lib = build.build_host()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True).stdout
    for sym in ["rerank_candidates", "rerank_batch", "throw_status", "fetch_batch"]:
        assert sym in out, sym


@pytest.mark.gpu
def test_cpp_api_against_oracle(cuda_ok):
    from paper_2312_05417_b200 import build
    import build_checkers
    build.build_host()
    build_checkers.build_oracle()
    exe = build_checkers.build_cpp_tests()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


REFAPI_SYMBOLS = ["maxsim_score", "aggregate_score", "4rank", "dot_f32", "validate_embedding", "validate_cls",
                  "validate_query", "store_paths", "build_store", "save_manifest", "load_manifest", "open_store",
                  "StoreHandle11fetch_batch", "kmeans", "nearest_centroid", "train_ivf", "save_ivf", "load_ivf",
                  "SearchCursor7advance", "SearchCursor8snapshot", "SearchCursor6finish", "begin_search",
                  "validate_config", "run_query", "run_batch", "measure_hit_rate", "mrr_at_k", "recall_at_k",
                  "load_qrels", "PipelineConfig5delta", "IvfIndex4size"]


def test_refapi_defines_the_reference_declarations():
    """lib/libespn_refapi.so (built against the UNMODIFIED reference headers)
    defines every function the reference declares on and around the path."""
    from paper_2312_05417_b200 import build
    lib = build.build_refapi()
    if lib is None:
        pytest.skip("reference headers absent and no prebuilt libespn_refapi.so")
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True).stdout
    names = [ln.split()[-1] for ln in out.splitlines() if " T " in ln]
    for sym in REFAPI_SYMBOLS:
        assert any(sym in n and n.startswith(("_ZN4espn", "_ZNK4espn")) for n in names), sym


@pytest.mark.gpu
def test_refapi_program_against_oracle(cuda_ok):
    """tests/cpp/refapi_test: written against the reference's own headers,
    linked with libespn_refapi.so, checked against the oracle on the GPU."""
    exe = ROOT / "tests" / "cpp" / "refapi_test"
    if not exe.exists():
        import build_checkers
        exe = build_checkers.build_refapi_test()
    assert exe is not None and exe.exists(), "tests/cpp/refapi_test was not built (needs the reference headers)"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
