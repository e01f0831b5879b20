"""On-disk .espn store (store.hpp:13-54).

CPU tests: the SPEC's known answers, the byte layout re-parsed independently
with numpy/struct, round trips at both value widths and both table dtypes,
and the error classes.  The gpu-marked test opens a store as the HBM table
and checks it re-ranks exactly like the in-memory table it was built from.
"""
import json
import struct

import numpy as np
import pytest

from paper_2312_05417_b200 import api, synth

HDR = struct.Struct("<8sIIIIIIQ")  # magic, version, d, d_cls, width, alignment, reserved, count


def _corpus(rng, n, d, t_lo=1, t_hi=40, d_cls=128):
    t = rng.integers(t_lo, t_hi + 1, n)
    row_ptr = np.zeros(n + 1, np.uint64)
    row_ptr[1:] = np.cumsum(t)
    rows = rng.standard_normal((int(row_ptr[-1]), d)).astype(np.float32)
    cls = rng.standard_normal((n, d_cls)).astype(np.float32)
    return row_ptr, rows, cls


def _parse(base):
    """Independent reader of the layout in include/espn_store.h."""
    raw = open(f"{base}.manifest", "rb").read()
    magic, ver, d, d_cls, w, al, _, count = HDR.unpack_from(raw)
    assert magic == b"ESPNSTR1" and ver == 1
    recs = np.frombuffer(raw, api._RECORD_DT, count, HDR.size)
    assert len(raw) == HDR.size + 16 * count
    return dict(d=d, d_cls=d_cls, w=w, al=al, recs=recs, data=open(f"{base}.espn", "rb").read())


def test_spec_kat_one_doc_one_block(tmp_path):
    # 1 doc, d_cls=128, d=32, t=10, width 2, alignment 4096 -> 896 bytes, 1 block
    rng = np.random.default_rng(1)
    row_ptr, rows, cls = _corpus(rng, 1, 32, 10, 10)
    m = api.build_store(tmp_path / "kat", row_ptr, rows, 32, 128, 2, 4096, cls)
    assert m.count() == 1 and m.d == 32 and m.d_cls == 128 and m.value_width == 2 and m.alignment == 4096
    r = m.records[0]
    assert int(r["byte_length"]) == 128 * 2 + 10 * 32 * 2 == 896
    assert int(r["byte_offset"]) == 0 and int(r["token_count"]) == 10
    assert -(-int(r["byte_length"]) // 4096) == 1
    p = _parse(tmp_path / "kat")
    assert len(p["data"]) == 4096  # one block, zero padded
    assert p["data"][896:] == bytes(4096 - 896)
    payload = np.frombuffer(p["data"][:896], np.float16)
    np.testing.assert_array_equal(payload[:128], cls[0].astype(np.float16))
    np.testing.assert_array_equal(payload[128:].reshape(10, 32), rows.astype(np.float16))
    js = json.load(open(f"{tmp_path / 'kat'}.manifest.json"))
    assert js["count"] == 1 and js["records"][0] == [0, 896, 10]


def test_alignment_one_is_packed(tmp_path):
    # alignment=1 -> file size == sum of payload bytes
    rng = np.random.default_rng(2)
    row_ptr, rows, cls = _corpus(rng, 37, 16)
    m = api.build_store(tmp_path / "a1", row_ptr, rows, 16, 128, 4, 1, cls)
    p = _parse(tmp_path / "a1")
    assert len(p["data"]) == int(m.records["byte_length"].astype(np.int64).sum())
    off = np.concatenate([[0], np.cumsum(m.records["byte_length"].astype(np.uint64))[:-1]])
    np.testing.assert_array_equal(m.records["byte_offset"], off)


@pytest.mark.parametrize("al", [512, 4096])
def test_aligned_offsets_and_blocks(tmp_path, al):
    rng = np.random.default_rng(3)
    row_ptr, rows, cls = _corpus(rng, 50, 32, 1, 80)
    m = api.build_store(tmp_path / "al", row_ptr, rows, 32, 128, 2, al, cls)
    r = m.records
    assert np.all(r["byte_offset"] % al == 0)
    np.testing.assert_array_equal(r["byte_length"], m.record_bytes(np.diff(row_ptr)))
    blocks = -(-r["byte_length"].astype(np.int64) // al)
    np.testing.assert_array_equal(np.diff(r["byte_offset"].astype(np.int64)), blocks[:-1] * al)
    assert len(_parse(tmp_path / "al")["data"]) == int(r["byte_offset"][-1]) + int(blocks[-1]) * al


@pytest.mark.parametrize("width", [2, 4])
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_round_trip(tmp_path, width, dtype):
    # decode(fetch(build(x))) == x at width 4; == fp16(x) at width 2
    rng = np.random.default_rng(4)
    d = 64
    row_ptr, rows, cls = _corpus(rng, 29, d)
    api.build_store(tmp_path / "rt", row_ptr, rows, d, 128, width, 4096, cls)
    rp, codes, cls_out = api.read_store_table(tmp_path / "rt", dtype, with_cls=True)
    np.testing.assert_array_equal(rp, row_ptr)
    stored = rows.astype(np.float16).astype(np.float32) if width == 2 else rows
    if dtype == "f16":
        want = stored.astype(np.float16).view(np.uint16).ravel()
    else:  # bf16, round to nearest even from the stored value
        b = stored.view(np.uint32).ravel().astype(np.uint64)
        want = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
    np.testing.assert_array_equal(codes, want)
    want_cls = cls.astype(np.float16).astype(np.float32) if width == 2 else cls
    np.testing.assert_array_equal(cls_out, want_cls)


def test_width2_bytes_are_rne_fp16(tmp_path):
    # values straddling fp16 rounding boundaries, subnormals and overflow-to-max
    vals = np.array([1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 2.0 ** -24, 2.0 ** -25 * 1.5, 65504.0,
                     -0.0, 6.1e-5, -3.14159, 1e-8, 0.1], np.float32)
    rows = np.tile(vals, (1, 1)).reshape(1, -1)[:, :8]
    row_ptr = np.array([0, 1], np.uint64)
    api.build_store(tmp_path / "rne", row_ptr, rows, 8, 4, 2, 1, np.zeros((1, 4), np.float32))
    data = _parse(tmp_path / "rne")["data"]
    np.testing.assert_array_equal(np.frombuffer(data[8:], np.uint16), rows.astype(np.float16).view(np.uint16).ravel())


def test_no_cls_writes_zeros(tmp_path):
    rng = np.random.default_rng(5)
    row_ptr, rows, _ = _corpus(rng, 3, 16)
    api.build_store(tmp_path / "nc", row_ptr, rows, 16, 32, 4, 1)
    _, _, c = api.read_store_table(tmp_path / "nc", with_cls=True)
    assert c.shape == (3, 32) and not c.any()


def test_empty_store(tmp_path):
    m = api.build_store(tmp_path / "e", np.zeros(1, np.uint64), np.zeros((0, 32), np.float32), 32)
    assert m.count() == 0
    rp, codes, _ = api.read_store_table(tmp_path / "e")
    assert rp.tolist() == [0] and codes.size == 0


def test_errors(tmp_path):
    rng = np.random.default_rng(6)
    row_ptr, rows, cls = _corpus(rng, 4, 16)
    with pytest.raises(api.InvalidConfigError):
        api.build_store(tmp_path / "x", row_ptr, rows, 16, 128, 2, 1000, cls)
    with pytest.raises(api.InvalidConfigError):
        api.build_store(tmp_path / "x", row_ptr, rows, 16, 128, 3, 4096, cls)
    bad = row_ptr.copy()
    bad[2] = bad[1]  # doc 1 has t = 0
    with pytest.raises(api.InvalidInputError):
        api.build_store(tmp_path / "x", bad, rows, 16, 128, 2, 4096, cls)
    nan = rows.copy()
    nan[3, 2] = np.nan
    with pytest.raises(api.InvalidInputError):
        api.build_store(tmp_path / "x", row_ptr, nan, 16, 128, 2, 4096, cls)
    with pytest.raises(api.IoError):
        api.build_store(tmp_path / "no_such_dir" / "x", row_ptr, rows, 16, 128, 2, 4096, cls)
    with pytest.raises(api.Error):
        api.load_manifest(tmp_path / "missing")
    # corrupt magic -> format error
    api.build_store(tmp_path / "ok", row_ptr, rows, 16, 128, 2, 4096, cls)
    raw = bytearray(open(f"{tmp_path / 'ok'}.manifest", "rb").read())
    raw[0:8] = b"NOTESPN!"
    open(f"{tmp_path / 'bad'}.manifest", "wb").write(raw)
    open(f"{tmp_path / 'bad'}.espn", "wb").write(open(f"{tmp_path / 'ok'}.espn", "rb").read())
    with pytest.raises(api.FormatError):
        api.load_manifest(tmp_path / "bad")
    # truncated manifest -> format error
    open(f"{tmp_path / 'bad'}.manifest", "wb").write(open(f"{tmp_path / 'ok'}.manifest", "rb").read()[:-5])
    with pytest.raises(api.FormatError):
        api.load_manifest(tmp_path / "bad")
    # truncated data file -> io error on read
    open(f"{tmp_path / 'bad'}.manifest", "wb").write(open(f"{tmp_path / 'ok'}.manifest", "rb").read())
    open(f"{tmp_path / 'bad'}.espn", "wb").write(open(f"{tmp_path / 'ok'}.espn", "rb").read()[:4096 * 2 + 10])
    with pytest.raises(api.IoError):
        api.read_store_table(tmp_path / "bad")


@pytest.mark.gpu
def test_open_store_reranks_like_in_memory_table(tmp_path, cuda_ok):
    rng = np.random.default_rng(7)
    d, n, nq, B, K = 32, 500, 32, 4, 60
    row_ptr, rows, cls = _corpus(rng, n, d, 1, 60)
    api.build_store(tmp_path / "g", row_ptr, rows, d, 128, 2, 4096, cls)
    st = api.GpuStore.open_store(tmp_path / "g", "f16")
    assert (st.d_cls, st.value_width, st.alignment) == (128, 2, 4096)
    mem = api.GpuStore(row_ptr, rows.astype(np.float16).view(np.uint16).ravel(), d, "f16")
    q = rng.standard_normal((B, nq, d)).astype(np.float32)
    ids, ccls, off = synth.make_candidates(n, B, K, seed=8)
    cfg = api.PipelineConfig(rerank_count=K, final_k=10)
    outs = []
    for s in (st, mem):
        rr = api.Reranker(s, B, B * K, nq)
        outs.append([np.copy(x) for x in rr.rerank_arrays(q, ids, ccls, off, cfg, write_bow=True)])
        rr.close()
        s.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


def test_python_wrapper_bounds_checks(tmp_path):
    rp = np.array([0, 3, 5], np.uint64)
    with pytest.raises(api.InvalidInputError):
        api.build_store(tmp_path / "b", rp, np.zeros((4, 8), np.float32), 8)  # 5 rows needed
    with pytest.raises(api.InvalidInputError):
        api.build_store(tmp_path / "b", rp, np.zeros((5, 8), np.float32), 8, 16, cls=np.zeros((1, 16), np.float32))
    with pytest.raises(api.InvalidInputError):
        api.build_store(tmp_path / "b", np.array([1, 3], np.uint64), np.zeros((3, 8), np.float32), 8)


@pytest.mark.parametrize("mode", ["direct", "buffered", "mmap"])
def test_store_reader_fetch_rows(tmp_path, mode):
    """api.StoreReader (the file-backed StoreHandle, store.hpp:56-112) -- the
    host side of the disk tier: request order, duplicates, the BOW rows at
    row_offsets() are the store's fp16 codes, direct-mode counters aligned."""
    rp, codes = synth.make_table(300, 32, 1, 40, seed=4)
    base = tmp_path / "r"
    api.build_store(base, rp, api.decode(codes, "f16"), 32, d_cls=16, alignment=512)
    rd = api.StoreReader(base, mode=mode, queue_depth=4)
    ids = np.array([5, 299, 5, 0, 17], np.uint32)
    buf, off, ctr = rd.fetch(ids)
    roff = rd.row_offsets(off)
    for j, i in enumerate(ids):
        t = int(rp[i + 1] - rp[i])
        got = np.frombuffer(buf[int(roff[j]):int(roff[j]) + t * 64].tobytes(), np.uint16)
        assert np.array_equal(got, codes[int(rp[i]) * 32:int(rp[i + 1]) * 32])
        assert int(off[j + 1] - off[j]) == (16 + t * 32) * 2
    if mode == "direct":
        assert ctr["bytes_read"] % 512 == 0 and ctr["bytes_read"] >= int(off[-1])
    with pytest.raises(api.InvalidInputError):
        rd.fetch(np.array([300], np.uint32))
    rd.close()
