"""The disk tier (ESPN_TABLE_DISK_TIER + espn_gpu_prefetch_rows): the paper's
premise that the embeddings live on SSD.  Only the resident docs ever exist
in memory; a batch's other needed docs are read from the .espn store file
with the reference's own file-backed StoreHandle (StoreReader, O_DIRECT,
queue_depth reads in flight; store.hpp:56-112), handed to the device, staged
and found by the PREFETCHED re-rank.  Rankings are bit-identical to the same
table fully in HBM."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05417_b200 import api, synth  # noqa: E402


def _case(tmp_path, n=4000, seed=3, d=32):
    rp, codes = synth.make_table(n, d, 1, 63, seed=seed)
    base = tmp_path / "disk"
    api.build_store(base, rp, api.decode(codes, "f16"), d, d_cls=16, alignment=512)
    resident = (np.random.default_rng(seed).random(n) < 0.2).astype(np.uint8)
    return rp, codes, base, resident


def _needed_misses(ids, off, R, resident, partial=False):
    """Per query: the needed candidates (first min(R, n_b)) not in HBM."""
    per, offs = [], [0]
    for b in range(len(off) - 1):
        a0, a1 = int(off[b]), int(off[b + 1])
        need = ids[a0:a0 + min(a1 - a0, R)]
        m = need[resident[need] == 0]
        per.append(m)
        offs.append(offs[-1] + m.size)
    return np.concatenate(per).astype(np.uint32) if per else np.zeros(0, np.uint32), np.asarray(offs, np.uint64)


@pytest.mark.parametrize("mode", ["direct", "buffered"])
def test_disk_tier_rerank_equals_hbm(tmp_path, cuda_ok, mode):
    rp, codes, base, resident = _case(tmp_path)
    n = rp.shape[0] - 1
    disk = api.GpuStore.open_store(base, resident=resident, disk_tier=True, chunk_bytes=1 << 16)
    assert disk.tiered and disk.resident_docs == int(resident.sum()) and disk.host_bytes == 0
    ref = api.GpuStore(rp, codes, 32, d_cls=16, alignment=512)
    reader = api.StoreReader(base, mode=mode, queue_depth=16)
    B, K = 4, 700
    rr = api.Reranker(disk, B, B * K, 32)
    rh = api.Reranker(ref, B, B * K, 32)
    for it, (R, partial) in enumerate(((700, False), (300, True), (700, False))):
        q, src = synth.make_queries(rp, codes, 32, B, seed=10 + it)
        ids, cls, off = synth.make_candidates(n, B, K, src=src, seed=20 + it)
        cfg = api.PipelineConfig(rerank_count=R, final_k=10, alpha=0.5, partial_rerank_enabled=partial)
        miss, moff = _needed_misses(ids, off, R, resident)
        buf, roff, ctr = reader.fetch(miss)
        assert ctr["bytes_read"] >= int(roff[-1])  # the reference's counters (aligned in direct mode)
        rr.prefetch_rows(miss, moff, buf, reader.row_offsets(roff))
        got = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", prefetched=True, fetch_stats=True)
        want = rh.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05")
        for g, w in zip(got[:3], want[:3]):
            assert np.array_equal(np.asarray(g).view(np.uint32), np.asarray(w).view(np.uint32)), it
        for b, fs in enumerate(rr.last_fetch_stats):
            nm = int(moff[b + 1] - moff[b])
            assert fs["prefetched"] == nm and fs["missed"] == 0, (it, b, fs)
        assert np.array_equal(got[0][:, 0], src.astype(np.uint32))
    rr.close(); rh.close(); reader.close(); disk.close(); ref.close()


def test_disk_tier_requires_prefetch_and_no_gather(tmp_path, cuda_ok):
    rp, codes, base, resident = _case(tmp_path, n=2000, seed=7)
    n = rp.shape[0] - 1
    disk = api.GpuStore.open_store(base, resident=resident, disk_tier=True)
    reader = api.StoreReader(base, mode="direct")
    rr = api.Reranker(disk, 2, 600, 32)
    q, src = synth.make_queries(rp, codes, 32, 2, seed=1)
    ids, cls, off = synth.make_candidates(n, 2, 300, src=src, seed=2)
    cfg = api.PipelineConfig(rerank_count=300, final_k=10)
    with pytest.raises(api.InvalidStateError):  # not prefetched: the rows are only in the file
        rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05")
    miss, moff = _needed_misses(ids, off, 300, resident)
    half = miss[: miss.size // 2]  # only some of them
    buf, roff, _ = reader.fetch(half)
    rr.prefetch_rows(half, np.array([0, half.size, half.size], np.uint64), buf, reader.row_offsets(roff))
    with pytest.raises(api.InvalidStateError):
        rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", prefetched=True)
    buf, roff, _ = reader.fetch(miss)  # then the full set works on the same workspace
    rr.prefetch_rows(miss, moff, buf, reader.row_offsets(roff))
    gi, _, gc, _ = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", prefetched=True)
    assert list(gc) == [10, 10] and np.array_equal(gi[:, 0], src.astype(np.uint32))
    with pytest.raises(api.InvalidStateError):
        disk.fetch_batch(np.arange(10, dtype=np.uint32))
    # host-tier hints are no-ops for disk docs (nothing to copy from memory)
    rr.prefetch_hints(ids, off)
    with pytest.raises(api.InvalidStateError):
        rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", prefetched=True)
    rr.close(); reader.close(); disk.close()


def test_prefetch_rows_input_checks(tmp_path, cuda_ok):
    rp, codes, base, resident = _case(tmp_path, n=1000, seed=11)
    disk = api.GpuStore.open_store(base, resident=resident, disk_tier=True)
    rr = api.Reranker(disk, 2, 400, 32)
    ids = np.array([1, 2, 3], np.uint32)
    with pytest.raises(api.InvalidInputError):  # rows past the buffer
        rr.prefetch_rows(ids, np.array([0, 3], np.uint64), np.zeros(64, np.uint8), np.zeros(3, np.uint64))
    with pytest.raises(api.InvalidInputError):  # misaligned offset
        rr.prefetch_rows(ids, np.array([0, 3], np.uint64), np.zeros(1 << 16, np.uint8), np.array([0, 8, 16], np.uint64))
    with pytest.raises(api.InvalidInputError):  # decreasing offsets
        rr.prefetch_rows(ids, np.array([0, 2, 1], np.uint64), np.zeros(1 << 16, np.uint8), np.zeros(3, np.uint64))
    rr.close()
    small = api.Reranker(disk, 2, 400, 32, staging_bytes=4096)  # rows larger than the staging slot
    nd = disk.n_docs
    many = np.arange(nd, dtype=np.uint32)[:200]
    tok = disk.token_counts(many).astype(np.uint64)
    boff = np.concatenate([[0], np.cumsum(tok * 64)[:-1]]).astype(np.uint64)
    with pytest.raises(api.InvalidConfigError):
        small.prefetch_rows(many, np.array([0, 200, 200], np.uint64), np.zeros(int(tok.sum()) * 64, np.uint8), boff)
    small.close(); disk.close()


@pytest.mark.parametrize("frac", [0.0, 0.5, 1.0])
def test_disk_tier_random_batches(tmp_path, cuda_ok, frac):
    """Random batches (ragged / empty lists, partial re-rank, alpha, the same
    doc missing in several queries -- staged once) through the disk tier,
    bit-identical to the table fully in HBM; resident fractions 0 (every
    needed doc from the file), 0.5 and 1 (nothing to stage)."""
    n = 3000
    rp, codes = synth.make_table(n, 32, 1, 63, seed=5)
    base = tmp_path / "fz"
    api.build_store(base, rp, api.decode(codes, "f16"), 32, d_cls=16, alignment=512)
    rng = np.random.default_rng(int(frac * 10) + 1)
    resident = (rng.random(n) < frac).astype(np.uint8)
    disk = api.GpuStore.open_store(base, resident=resident, disk_tier=True)
    ref = api.GpuStore(rp, codes, 32, d_cls=16, alignment=512)
    reader = api.StoreReader(base, mode="direct", queue_depth=8)
    rr = api.Reranker(disk, 8, 8 * 600, 32)
    rh = api.Reranker(ref, 8, 8 * 600, 32)
    for case in range(6):
        B = int(rng.choice([1, 3, 8]))
        q, src = synth.make_queries(rp, codes, 32, B, seed=30 + case)
        ids_l, cls_l, offs = [], [], [0]
        pool = rng.permutation(n)[:700].astype(np.uint32)  # overlapping lists: shared misses
        for b in range(B):
            m = int(rng.choice([0, 1, 50, 600]))
            c = rng.choice(pool, size=m, replace=False).astype(np.uint32)
            if m and src[b] not in c:
                c[0] = src[b]
            s = rng.random(m).astype(np.float32)
            o = np.lexsort((c, -s))
            ids_l.append(c[o]); cls_l.append(s[o]); offs.append(offs[-1] + m)
        ids = np.concatenate(ids_l).astype(np.uint32)
        cls = np.concatenate(cls_l).astype(np.float32)
        off = np.asarray(offs, np.uint64)
        partial = bool(rng.random() < 0.5)
        R = int(rng.integers(10, 601)) if partial else 600
        cfg = api.PipelineConfig(rerank_count=R, final_k=10, alpha=float(rng.choice([0.5, 1.0])),
                                 partial_rerank_enabled=partial)
        miss, moff = _needed_misses(ids, off, R, resident)
        buf, roff, _ = reader.fetch(miss)
        rr.prefetch_rows(miss, moff, buf, reader.row_offsets(roff))
        got = rr.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05", prefetched=True)
        want = rh.rerank_arrays(q, ids, cls, off, cfg, kernel="tcgen05")
        for g, w in zip(got[:3], want[:3]):
            assert np.array_equal(np.asarray(g).view(np.uint32), np.asarray(w).view(np.uint32)), (frac, case)
    rr.close(); rh.close(); reader.close(); disk.close(); ref.close()
