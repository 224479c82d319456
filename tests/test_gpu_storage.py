"""Device storage kernels (csrc/sort.cu, csrc/setops.cu) against the
reference's golden storage fixtures and the numpy oracle at scale."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import storage as ost  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    from paper_2604_20073_b200 import device

    device.lib()
    return device


def to_dev(rows, arity):
    from paper_2604_20073_b200 import device

    arr = np.asarray(rows, dtype=np.uint32).reshape(-1, arity).T.copy()
    return torch.from_numpy(arr).to(device.device())


def host(t):
    return t.cpu().numpy().astype(np.int64).T


def test_sort_dedup_golden(dev, golden):
    for case in golden("storage.json")["sort_dedup"]:
        rows = to_dev(case["rows"], case["arity"])
        for bits in (5, 32):
            got = dev.sort_dedup(rows, bits, order=case["order"])
            assert host(got).tolist() == case["out"]


def test_compute_delta_golden(dev, golden):
    for case in golden("storage.json")["compute_delta"]:
        a = case["arity"]
        segs = [to_dev(case["body"], a), to_dev(case["head"], a)]
        got = dev.compute_delta(to_dev(case["new"], a), segs, 5)
        assert host(got).tolist() == case["out"]


def test_merge_sequences_golden(dev, golden):
    from paper_2604_20073_b200.columns import ColumnarRelation, as_tuples

    # storage.json's 80 sequences + the acceptance suite's 1000 (merges.json.gz)
    for case in golden("storage.json")["merge"] + golden("merges.json.gz"):
        a = case["arity"]
        rel = ColumnarRelation.empty(a, case["order"])
        for step in case["steps"]:
            rel = rel.merge_delta(to_dev(step["delta"], a), flush_limit=case["flush"])
            assert [list(r) for r in as_tuples(rel.head)] == step["head"]
            assert [list(r) for r in as_tuples(rel.body)] == step["body"]
            assert rel.hist.keys.cpu().tolist() == step["hist_keys"]
            assert rel.hist.degrees.cpu().tolist() == step["hist_degrees"]
            assert rel.hist.prefix.cpu().tolist() == step["hist_prefix"]
            rel.check_invariants()


def test_histogram_updates_golden(dev, golden):
    from paper_2604_20073_b200.columns import Histogram

    for seq in golden("storage.json")["histogram"]:
        h = Histogram.empty()
        for step in seq:
            col = torch.tensor(step["delta"], dtype=torch.int64).to(torch.uint32).to(dev.device())
            h = h.updated(col)
            assert h.keys.cpu().tolist() == step["keys"]
            assert h.degrees.cpu().tolist() == step["degrees"]
            assert h.prefix.cpu().tolist() == step["prefix"]


@pytest.mark.parametrize("arity,bits,n,domain", [
    (1, 20, 1_000_003, 1 << 20),
    (2, 24, 3_000_000, 1 << 12),
    (3, 21, 2_000_000, 1 << 7),
    (4, 32, 500_000, 1 << 32),       # 128-bit keys: chunked LSD with a row permutation
    (5, 13, 700_000, 7),             # heavy duplication, 65 bits
    (8, 32, 100_000, 3),
])
def test_sort_dedup_at_scale(dev, arity, bits, n, domain):
    rng = np.random.default_rng(arity * 1000 + bits)
    rows = rng.integers(0, domain, size=(n, arity), dtype=np.uint64).astype(np.int64)
    got = dev.sort_dedup(to_dev(rows, arity), bits)
    assert np.array_equal(host(got), ost.sort_dedup(rows))
    assert dev.is_sorted_strict(got)


def test_compute_delta_and_merge_at_scale(dev):
    rng = np.random.default_rng(5)
    full = ost.sort_dedup(rng.integers(0, 3000, size=(2_000_000, 2)))
    head = ost.difference(ost.sort_dedup(rng.integers(3000, 3100, size=(20_000, 2))), full)
    new = rng.integers(0, 3200, size=(1_500_000, 2))
    want = ost.compute_delta(new, head, full)
    got = dev.compute_delta(to_dev(new, 2), [to_dev(full, 2), to_dev(head, 2)], 12)
    assert np.array_equal(host(got), want)
    merged = dev.merge(to_dev(full, 2), got)
    assert np.array_equal(host(merged), ost.merge_sorted(full, want))


def test_histogram_at_scale(dev):
    rng = np.random.default_rng(11)
    col = np.sort(rng.zipf(1.3, size=3_000_000) % 100_000).astype(np.uint32)
    keys, deg, prefix = dev.histogram(torch.from_numpy(col).to(dev.device()))
    uk, cnt = np.unique(col, return_counts=True)
    assert np.array_equal(keys.cpu().numpy(), uk)
    assert np.array_equal(deg.cpu().numpy(), cnt)
    assert np.array_equal(prefix.cpu().numpy(), np.cumsum(cnt))


def test_empty_and_single_rows(dev):
    e = to_dev([], 3)
    assert dev.sort_dedup(e, 8).shape == (3, 0)
    assert dev.compute_delta(e, [to_dev([(1, 2, 3)], 3)], 8).shape == (3, 0)
    one = to_dev([(4, 5, 6)], 3)
    assert host(dev.sort_dedup(one, 8)).tolist() == [[4, 5, 6]]
    assert dev.compute_delta(one, [one], 8).shape[1] == 0
    assert dev.is_sorted_strict(one)
    top = to_dev([(0xFFFFFFFE, 0), (0, 0xFFFFFFFE), (0xFFFFFFFE, 0)], 2)
    assert host(dev.sort_dedup(top, 32)).tolist() == [[0, 0xFFFFFFFE], [0xFFFFFFFE, 0]]


def test_compute_delta_chunked_equals_single(dev, monkeypatch):
    from paper_2604_20073_b200 import columns

    rng = np.random.default_rng(17)
    full_rows = ost.sort_dedup(rng.integers(0, 500, size=(200_000, 2)))
    rel = columns.ColumnarRelation.from_sorted(2, (0, 1), to_dev(full_rows, 2))
    staged = to_dev(rng.integers(0, 700, size=(900_000, 2)), 2)
    whole = columns.compute_delta(staged, rel)
    monkeypatch.setattr(columns, "DELTA_CHUNK", 70_001)  # 13 chunks, exercises the re-merge
    chunked = columns.compute_delta(staged, rel)
    assert torch.equal(whole, chunked)
    want = ost.compute_delta(host(staged), np.empty((0, 2), np.int64), full_rows)
    assert np.array_equal(host(chunked), want)


@pytest.mark.parametrize("arity,bits", [(1, 21), (2, 12), (3, 32)])  # 3x32 bits: row-compare path
def test_anti_join_and_merge_across_tile_boundaries(dev, arity, bits):
    """Every staged row equal to a full row must be recognised even when the
    pair straddles a merge-path tile boundary (1024 outputs per tile)."""
    rng = np.random.default_rng(arity)
    top = min(1 << bits, 1 << 20)
    full = ost.sort_dedup(rng.integers(0, top, size=(300_000, arity)))
    extra = ost.difference(ost.sort_dedup(rng.integers(0, top, size=(50_000, arity))), full)
    staged = np.concatenate([full, full[::3], extra])
    got = dev.compute_delta(to_dev(staged, arity), [to_dev(full, arity)], bits)
    assert np.array_equal(host(got), extra)
    # interleaved disjoint halves merge back to the whole
    a, b = full[0::2], full[1::2]
    assert np.array_equal(host(dev.merge(to_dev(a, arity), to_dev(b, arity))), full)


def test_anti_join_small_staged_vs_large_full(dev):
    """Binary-search regime (segment > 24x staged) agrees with the oracle."""
    rng = np.random.default_rng(23)
    full = ost.sort_dedup(rng.integers(0, 1 << 16, size=(2_000_000, 2)))
    staged = np.concatenate([full[rng.choice(len(full), 20_000)], rng.integers(0, 1 << 16, size=(20_000, 2))])
    want = ost.compute_delta(staged, np.empty((0, 2), np.int64), full)
    for bits in (16, 32):  # packed keys (2x16) and, at 2x32, still packed
        got = dev.compute_delta(to_dev(staged, 2), [to_dev(full, 2)], bits)
        assert np.array_equal(host(got), want)
    full3 = np.concatenate([full, full[:, :1]], axis=1)
    staged3 = np.concatenate([staged, staged[:, :1]], axis=1)
    got3 = dev.compute_delta(to_dev(staged3, 3), [to_dev(full3, 3)], 32)  # row-compare path
    assert np.array_equal(host(got3)[:, :2], want)


@pytest.mark.parametrize("n,nf", [(0, 50), (1, 0), (7, 0), (3000, 0), (1, 1), (5000, 20000), (300_000, 2_000)])
def test_histogram_union_matches_two_step(dev, n, nf):
    """srdl_histogram_union == histogram(delta) and its union with a full
    histogram (equal keys summed), overlapping and disjoint key sets."""
    rng = np.random.default_rng(n + 7 * nf)
    col = np.sort(rng.zipf(1.4, size=n) % 50_000).astype(np.uint32)
    full = np.sort(rng.integers(0, 60_000, size=nf)).astype(np.uint32)
    fk, fd, _ = dev.histogram(torch.from_numpy(full).to(dev.device()))
    (dk, dd, dp), (uk, ud, up) = dev.histogram_union(torch.from_numpy(col).to(dev.device()), fk, fd)
    ck, cc = np.unique(col, return_counts=True)
    assert np.array_equal(dk.cpu().numpy(), ck)
    assert np.array_equal(dd.cpu().numpy(), cc)
    assert np.array_equal(dp.cpu().numpy(), np.cumsum(cc))
    if n:
        both = np.concatenate([col, full])
        bk, bc = np.unique(both, return_counts=True)
        assert np.array_equal(uk.cpu().numpy(), bk)
        assert np.array_equal(ud.cpu().numpy(), bc)
        assert np.array_equal(up.cpu().numpy(), np.cumsum(bc))


@pytest.mark.parametrize("arity,bits", [(1, 21), (2, 16), (3, 32)])
@pytest.mark.parametrize("layout", ["random", "sorted", "sorted_dups"])
@pytest.mark.parametrize("n", [2, 1000, 200_000, 5_000_000])
def test_sort_paths_device_and_host_branch(dev, arity, bits, layout, n):
    """sort_dedup / compute_delta decide 'already sorted' on the device below
    2^22 rows (radix passes skip themselves) and on the host above; both
    branches, every key-packing path (1 chunk, 3x32-bit multi-chunk), sorted
    and unsorted input, and the distinct=True re-sort."""
    rng = np.random.default_rng(n + arity)
    hi = min(1 << bits, 1 << 20)
    rows = rng.integers(0, hi, size=(n, arity))
    if layout != "random":
        rows = np.unique(rows, axis=0) if layout == "sorted" else rows[np.lexsort(rows.T[::-1])]
    want = np.unique(rows, axis=0)
    t = to_dev(rows.reshape(-1), arity)
    got = dev.sort_dedup(t, bits)
    assert np.array_equal(host(got), want)
    full = want[::3]
    fd = to_dev(full.reshape(-1), arity)
    delta = dev.compute_delta(t, [fd], bits)
    keep = ~np.isin(np.arange(len(want)), np.arange(0, len(want), 3))
    assert np.array_equal(host(delta), want[keep])
    if arity > 1:  # distinct rows re-sorted under the reversed column order
        order = list(range(arity))[::-1]
        rs = dev.sort_dedup(got, bits, order=order, distinct=True)
        ref = want[:, order]
        assert np.array_equal(host(rs), ref[np.lexsort(ref.T[::-1])])


@pytest.mark.parametrize("arity,bits,n", [(2, 27, 2_000_000), (2, 9, 5_000), (3, 21, 1_000_000), (4, 12, 300_000)])
def test_sort_reorder_equals_full_sort(dev, arity, bits, n):
    """srdl_sort_reorder (one stable sort on the leading target columns of a
    sorted delta) gives exactly the full sort under every column order."""
    import itertools

    rng = np.random.default_rng(arity * 100 + bits)
    rows = np.unique(rng.integers(0, 1 << bits, size=(n, arity)), axis=0).T.astype(np.uint32)
    t = torch.from_numpy(np.ascontiguousarray(rows)).to(dev.device())
    for order in itertools.permutations(range(arity)):
        got = dev.sort_reorder(t, bits, order)
        want = dev.sort_dedup(t, bits, order=order, distinct=True)
        assert torch.equal(got, want), order


@pytest.mark.parametrize("n", [1, 4096, 4097, 5000, 100_003, 3_000_001, 40_000_000])
@pytest.mark.parametrize("wide", [False, True])
def test_scans_match_cumsum(dev, n, wide):
    """Single-pass chained scans (u32 / u64, exclusive with total, inclusive,
    in place) against torch.cumsum, across one and many tiles."""
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randint(0, 7, (n,), device="cuda", generator=g, dtype=torch.int64)
    ref = torch.cumsum(x, 0)
    src = x if wide else x.to(torch.int32).view(torch.uint32)
    out, total = dev.scan(src, exclusive=True)
    got = out.view(torch.int64) if wide else out.view(torch.int32).to(torch.int64)
    assert torch.equal(got, ref - x)
    assert int(total.view(torch.int64 if wide else torch.int32)[0]) == int(ref[-1])
    inc, _ = dev.scan(src, exclusive=False)
    got = inc.view(torch.int64) if wide else inc.view(torch.int32).to(torch.int64)
    assert torch.equal(got, ref)
    for _ in range(3):  # repeated calls reuse the epoch-stamped status
        out2, _ = dev.scan(src, exclusive=True)
        assert torch.equal(out2, out)
