"""The CPU oracle is pinned to the reference's own outputs (golden vectors) — CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import golden_cases


def cases(golden):
    return golden_cases(golden)


def test_golden_has_cases(golden):
    assert "c1" in cases(golden) and "long" in cases(golden) and len(cases(golden)) >= 30


def test_oracle_permutation_pipeline_matches_reference(golden):
    for c in cases(golden):
        g = lambda k: golden[f"{c}/{k}"]  # noqa: E731
        n_rows, n_cols = (int(v) for v in g("shape"))
        pr, pc = O.permute_coo(g("row"), g("col"), g("p_r"), g("p_c"))
        assert np.array_equal(pr, g("perm_row")), c
        assert np.array_equal(pc, g("perm_col")), c
        ptr0, col0, val0 = O.coo_to_csr(n_rows, g("row"), g("col"), g("val"))
        assert np.array_equal(ptr0, g("csr0_ptr")) and np.array_equal(col0, g("csr0_col")), c
        assert np.array_equal(val0.view(np.uint64), g("csr0_val").view(np.uint64)), c
        ptr1, col1, val1 = O.coo_to_csr(n_rows, pr, pc, g("val"))
        assert np.array_equal(ptr1, g("csr_ptr")) and np.array_equal(col1, g("csr_col")), c
        assert np.array_equal(val1.view(np.uint64), g("csr_val").view(np.uint64)), c
        assert np.array_equal(O.permute_vector(g("x"), g("p_c")), g("x_perm")), c


def test_oracle_sampled_rows_match_reference(golden):
    for c in ("c1", "long", "s7"):
        g = lambda k: golden[f"{c}/{k}"]  # noqa: E731
        rows = np.arange(int(g("shape")[0]))[:: max(1, int(g("shape")[0]) // 50)]
        got = O.permute_csr_rows(g("csr0_ptr"), g("csr0_col"), g("csr0_val"), g("p_r"), g("p_c"), rows)
        ptr, col, val = g("csr_ptr"), g("csr_col"), g("csr_val")
        for r, (cc, vv) in zip(rows, got):
            a, b = ptr[r], ptr[r + 1]
            assert np.array_equal(cc, col[a:b]) and np.array_equal(vv, val[a:b])


def test_oracle_spmv_bitwise_matches_reference(golden):
    for c in cases(golden):
        g = lambda k: golden[f"{c}/{k}"]  # noqa: E731
        y0 = O.spmv_csr(g("csr0_ptr"), g("csr0_col"), g("csr0_val"), g("x"))
        y = O.spmv_csr(g("csr_ptr"), g("csr_col"), g("csr_val"), g("x_perm"))
        assert np.array_equal(y0.view(np.uint64), g("y0").view(np.uint64)), c
        assert np.array_equal(y.view(np.uint64), g("y").view(np.uint64)), c
        n = int(g("shape")[0])
        par = O.spmv_csr_parallel(g("csr_ptr"), g("csr_col"), g("csr_val"), g("x_perm"), min(4, n))
        assert np.array_equal(par.view(np.uint64), g("par4").view(np.uint64)), c
        assert O.relative_error(y, g("y_expected")) <= 1e-12, c


def test_oracle_histograms_and_entropy_match_reference(golden):
    for c in cases(golden):
        g = lambda k: golden[f"{c}/{k}"]  # noqa: E731
        if f"{c}/hist" not in golden:
            continue
        n_rows, n_cols = (int(v) for v in g("shape"))
        br, bc = (int(v) for v in g("bins2d"))
        h0 = O.histogram_2d_counts(g("row"), g("col"), n_rows, n_cols, br, bc)
        h = O.histogram_2d_counts(g("perm_row"), g("perm_col"), n_rows, n_cols, br, bc)
        assert np.array_equal(h0, g("hist0")) and np.array_equal(h, g("hist")), c
        assert O.entropy_of_counts(h0) == float(g("H0")), c
        assert O.entropy_of_counts(h) == float(g("H")), c
        b1r, b1c = min(512, n_rows), min(512, n_cols)
        assert np.array_equal(O.row_histogram_counts(g("perm_row"), n_rows, b1r), g("rowhist")), c
        assert np.array_equal(O.col_histogram_counts(g("perm_col"), n_cols, b1c), g("colhist")), c


def test_oracle_entropy_kats(golden):
    cnt = golden["ent/counts"]
    assert O.entropy_of_counts(cnt) == float(golden["ent/H2"])
    assert O.entropy_of_counts(cnt, np.e) == float(golden["ent/He"])
    assert O.entropy_of_counts(cnt, 10.0) == float(golden["ent/H10"])
    assert O.entropy_of_counts([1, 1, 2]) == 1.5  # test_entropy.py:103-104
    assert O.entropy_of_counts([0, 9, 0, 0]) == 0.0
    with pytest.raises(ValueError):
        O.entropy_of_counts([0, 0])


def test_oracle_permutation_generators(golden):
    assert np.array_equal(O.random_permutation(31, 5), golden["perm/rp_31_5"])
    assert np.array_equal(O.random_permutation(1000, 123), golden["perm/rp_1000_123"])
    assert [O.axis_seed(7, 0), O.axis_seed(7, 1)] == [int(v) for v in golden["perm/axis_seed_7"]]
    assert O.derived_seed(0, 3) == int(golden["perm/derived_0_3"][0])
    assert np.array_equal(O.input_vector(0, 17), golden["perm/input_vector_0_17"])
    # inverse / compose KATs (test_permute.py:68-76)
    assert O.inverse([2, 0, 1]).tolist() == [1, 2, 0]
    p = O.random_permutation(31, 5)
    assert np.array_equal(O.compose(p, O.inverse(p)), np.arange(31))
    assert O.permute_vector([10.0, 20.0, 30.0], [2, 0, 1]).tolist() == [20.0, 30.0, 10.0]


def test_oracle_duplicates_and_kats():
    assert O.find_duplicate([0, 0], [1, 1]) == (0, 1)
    assert O.find_duplicate([0, 1, 0], [1, 1, 2]) is None
    with pytest.raises(ValueError, match="duplicate entry at \\(0, 1\\)"):
        O.coo_to_csr(2, [0, 0], [1, 1], [1.0, 2.0])
    ptr, col, val = O.coo_to_csr(2, [0, 1, 0, 1], [0, 0, 1, 1], [1.0, 3.0, 2.0, 4.0])
    assert ptr.tolist() == [0, 2, 4] and col.tolist() == [0, 1, 0, 1] and val.tolist() == [1.0, 2.0, 3.0, 4.0]
    assert O.bin_edges(10, 3).tolist() == [0, 3, 6, 10]
    assert O.bin_index([9], 10, 3).tolist() == [2]
    assert O.make_row_partition(10, 3).tolist() == [0, 4, 7, 10]


def test_oracle_generators_are_well_formed():
    ptr, col, val = O.laplacian5(5)
    assert ptr[-1] == 5 * 25 - 4 * 5 and col.size == val.size == ptr[-1]
    dense = np.zeros((25, 25))
    for r in range(25):
        dense[r, col[ptr[r] : ptr[r + 1]]] = val[ptr[r] : ptr[r + 1]]
    assert np.allclose(dense, dense.T) and np.all(np.diag(dense) == 4.0)
    cols, vals = O.random_rows(np.arange(50), 1000, 20, 12345)
    assert cols.shape == (50, 20)
    assert np.all(np.diff(cols, axis=1) > 0) and cols.min() >= 0 and cols.max() < 1000
    assert vals.min() >= -1.0 and vals.max() < 1.0
    c2, _ = O.random_rows(np.arange(3), 25, 20, 7)  # forces extra draw rounds
    assert np.all(np.diff(c2, axis=1) > 0)
    for n_cols in (1000, 25, 50_000_000):
        rows = np.arange(0, 3000, 7)
        fc, fv = O.random_rows_fast(rows, n_cols, 20, 99)
        sc, sv = O.random_rows(rows, n_cols, 20, 99)
        assert np.array_equal(fc, sc) and np.array_equal(fv, sv)


def test_oracle_rowshard_map_is_a_padded_bijection():
    n, parts = 103, 4
    pad = -(-n // parts)
    slots = O.rowshard_remap_cols(np.arange(n), n, parts, pad)
    assert len(set(slots.tolist())) == n and slots.max() < parts * pad
    b = O.make_row_partition(n, parts)
    for k in range(parts):
        assert slots[b[k]] == k * pad
