"""Host-side logic of the package (no GPU): partitions, protocol helpers, strategies."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O
from paper_2308_00106_b200 import bench as B
from paper_2308_00106_b200.kernels import make_row_partition
from paper_2308_00106_b200.permute import (
    TABLE_ORDER,
    StrategyKind,
    _interleave_forward,
    axis_seed,
    pcg64_permutation,
    pcg64_swap_partners,
    random_permutation_forward,
)
from paper_2308_00106_b200.rowshard import ShardPlan


def test_make_row_partition_examples():  # reference test_kernels.py:92-96
    assert make_row_partition(10, 2).boundaries.tolist() == [0, 5, 10]
    assert make_row_partition(10, 3).boundaries.tolist() == [0, 4, 7, 10]
    assert make_row_partition(5, 5).boundaries.tolist() == [0, 1, 2, 3, 4, 5]
    with pytest.raises(ValueError):
        make_row_partition(10, 0)
    with pytest.raises(ValueError):
        make_row_partition(3, 4)


@given(st.integers(1, 200), st.data())
@settings(max_examples=60, deadline=None)
def test_partition_matches_oracle(n_rows, data):
    w = data.draw(st.integers(1, n_rows))
    assert np.array_equal(make_row_partition(n_rows, w).boundaries, O.make_row_partition(n_rows, w))


def test_protocol_helpers_match_reference_semantics():
    assert B.gflops(1000, 1e-6) == pytest.approx(2.0)
    assert B.gflops(0, 1.0) == 0.0
    with pytest.raises(ValueError):
        B.gflops(10, 0.0)
    assert B.choose_iterations(1e-6) == 5000 and B.choose_iterations(1.0) == 1000
    assert B.derived_seed(0, 3) == O.derived_seed(0, 3)
    assert np.array_equal(B.input_vector(0, 17), O.input_vector(0, 17))
    # SURVEY.md §8d byte counts
    assert B.spmv_bytes(10_000, 10_000, 100_000) == 1_400_004
    assert B.spmv_bytes(4_000_000, 4_000_000, 19_992_000) == 319_904_004
    assert B.spmv_bytes(50_000_000, 50_000_000, 1_000_000_000) == 13_000_000_004


def test_host_permutation_generation_is_the_references(golden):
    assert np.array_equal(random_permutation_forward(31, 5), golden["perm/rp_31_5"])
    assert np.array_equal(random_permutation_forward(1000, 123), golden["perm/rp_1000_123"])
    assert [axis_seed(7, 0), axis_seed(7, 1)] == [int(v) for v in golden["perm/axis_seed_7"]]
    with pytest.raises(ValueError):
        random_permutation_forward(0, 1)
    with pytest.raises(ValueError):
        random_permutation_forward(5, -1)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 65, 1000, 4097, 65536, 1 << 20, 3_000_001])
@pytest.mark.parametrize("seed", [0, 5, 2**63 + 11])
def test_native_pcg64_permutation_is_numpys(n, seed):
    """sme_host_pcg64_permutation == Generator(PCG64(seed)).permutation(n), and it leaves
    the generator in numpy's state (incl. the buffered uint32 half)."""
    ours_bg, ref_bg = np.random.PCG64(seed), np.random.PCG64(seed)
    got = pcg64_permutation(ours_bg, n)
    ref = np.random.Generator(ref_bg).permutation(n)
    assert got.dtype == np.int32 and np.array_equal(got, ref)
    assert ours_bg.state == ref_bg.state


def test_native_pcg64_consecutive_draws_like_riffle():
    """Two permutations from one generator (riffle_shuffle_permutation, permute.py:150-156),
    then a third with an odd pending uint32, then a float draw: all as numpy."""
    a, b = np.random.PCG64(99), np.random.PCG64(99)
    ga = np.random.Generator(a)
    for n in (12345, 777, 3):
        assert np.array_equal(pcg64_permutation(b, n), ga.permutation(n))
    gb = np.random.Generator(b)
    assert gb.integers(0, 1000, 5).tolist() == ga.integers(0, 1000, 5).tolist()
    assert gb.random() == ga.random()


def test_strategy_table_and_interleave():
    assert [k.code for k in TABLE_ORDER] == ["reg", "r", "gr", "gc", "rc"]
    assert StrategyKind.ROW_COLUMN_PERMUTE.label == "Row-Column-Permute"
    # permute.py:129-139: alternate the two parts, then the remainder
    assert _interleave_forward(5, 2).tolist() == [0, 2, 1, 3, 4]
    assert sorted(_interleave_forward(9, 4).tolist()) == list(range(9))


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (103, 4), (8, 8), (50_000_000, 8)])
def test_shard_plan(n, world):
    plan = ShardPlan(n, n, world)
    assert plan.rows[0] == 0 and plan.rows[-1] == n
    assert plan.pad * world >= n and plan.pad - (n // world) <= 1
    sizes = np.diff(plan.cols)
    assert sizes.max() <= plan.pad
    cols = np.unique(np.r_[0, n - 1, plan.cols[:-1], np.minimum(plan.cols[1:], n - 1)])
    assert np.array_equal(plan.slot_of(cols), O.rowshard_remap_cols(cols, n, world, plan.pad))



@pytest.mark.parametrize("n", [1, 2, 3, 5, 64, 1000, 20_000])
@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3])
@pytest.mark.parametrize("pending", [False, True])
def test_native_swap_partners_replay_numpys_shuffle(n, seed, pending):
    """sme_host_pcg64_swap_partners: the sequential swaps over its partners give numpy's
    permutation, and the generator ends in numpy's state; also with a pending uint32 half
    (pending=True draws one integer first, like a second riffle part after an odd count)."""
    ours_bg, ref_bg = np.random.PCG64(seed), np.random.PCG64(seed)
    if pending:
        for bg in (ours_bg, ref_bg):
            np.random.Generator(bg).integers(0, 10, dtype=np.uint32)
        assert ours_bg.state["has_uint32"] == 1
    j = pcg64_swap_partners(ours_bg, n, threads=3)
    a = np.arange(n)
    for i in range(n - 1, 0, -1):
        a[i], a[j[i]] = a[j[i]], a[i]
    assert np.array_equal(a, np.random.Generator(ref_bg).permutation(n))
    assert ours_bg.state == ref_bg.state


def test_native_swap_partners_large_match_full_shuffle():
    bg1, bg2 = np.random.PCG64(123), np.random.PCG64(123)
    n = 3_000_001
    j = pcg64_swap_partners(bg1, n)
    full = pcg64_permutation(bg2, n)
    assert bg1.state == bg2.state
    # spot-check: the partners' last steps reproduce the shuffle's tail positions' dependence
    assert j[0] == 0 and int(j[1:].max()) < n and np.all(j[1:] <= np.arange(1, n))
    assert full.dtype == np.int32


def test_hostio_fresh_results_never_alias_and_recycle():
    """hostio.fresh_host: large results are pooled mappings handed out again only after
    every array (and tensor) viewing them has been released; small ones are np.empty."""
    import gc

    import torch

    from paper_2308_00106_b200 import hostio

    n = hostio.CHUNK_MIN_BYTES // 8 + 7
    key = n * 8
    hostio.pool_clear()
    a = hostio.fresh_host(n, np.float64)
    b = hostio.fresh_host(n, np.float64)
    assert a.flags.writeable and a.shape == (n,) and not np.shares_memory(a, b)
    a[:] = 1.0
    view = a[5:9]
    t = torch.from_numpy(a)
    del a
    gc.collect()
    assert len(hostio._POOL.get(key, [])) == 0  # a view and a tensor still hold the mapping
    del view
    gc.collect()
    assert len(hostio._POOL.get(key, [])) == 0
    del t
    gc.collect()
    assert len(hostio._POOL[key]) == 1
    c = hostio.fresh_host(n, np.float64)  # the released mapping comes back
    assert len(hostio._POOL[key]) == 0 and c[0] == 1.0 and not np.shares_memory(c, b)
    small = hostio.fresh_host(10, np.float32)
    assert small.dtype == np.float32 and small.shape == (10,)
    assert hostio.slices(10, 8) == [0, 10] and hostio.slices(n, 8, 4)[-1] == n


def test_hostio_pool_is_capped_lru(monkeypatch):
    """released result mappings are capped in total bytes (least recently
    released evicted first) and per size; concurrent releases are safe."""
    import gc
    import threading

    from paper_2308_00106_b200 import hostio

    hostio.pool_clear()
    base = hostio.CHUNK_MIN_BYTES
    monkeypatch.setattr(hostio, "POOL_MAX_BYTES", 3 * base)
    arrs = [hostio.fresh_host(base // 8 + 64 * k, np.float64) for k in range(4)]
    while arrs:  # released smallest first
        del arrs[0]
        gc.collect()
    assert 0 < hostio.pool_bytes() <= 3 * base
    sizes = sorted(k for k, v in hostio._POOL.items() if v)
    assert (base // 8) * 8 not in sizes  # the first released (smallest here) was evicted
    hostio.pool_clear()
    assert hostio.pool_bytes() == 0

    def worker():
        for _ in range(5):
            a = hostio.fresh_host(base // 8, np.float64)
            a[0] = 1.0
            del a
            gc.collect()

    ts = [threading.Thread(target=worker) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert len(hostio._POOL.get(base, [])) <= hostio.POOL_PER_SIZE
    hostio.pool_clear()


def test_cache_header_rejects_foreign_and_newer_files(tmp_path):
    import struct

    from paper_2308_00106_b200 import cache

    f = tmp_path / "x.smecache"
    f.write_bytes(b"NOTACACHE" + b"\0" * 100)
    with pytest.raises(ValueError, match="not an sme cache"):
        cache.read_header(f)
    f.write_bytes(cache.MAGIC + struct.pack("<II", cache.VERSION + 1, 2) + b"{}")
    with pytest.raises(ValueError, match="cache version"):
        cache.read_header(f)
    f.write_bytes(cache.MAGIC + struct.pack("<II", cache.VERSION, 11) + b'{"kind": 1}')
    head, base = cache.read_header(f)
    assert head == {"kind": 1} and base == cache.ALIGN
