"""int64 row_ptr ("wide" CSR, nnz >= 2^31 - 1): the `_i64` entry points of include/sme.h.

The reference keeps row_ptr as int64 at every size (matio.py:97-99); the GPU layout
switches from int32 to int64 offsets at nnz = 2^31 - 1 (SURVEY.md §7, §8(d) s_p = 8).
Small matrices are forced wide (_cuda.FORCE_WIDE_ROW_PTR) so that every wide entry point
is checked against the int32 path (bit for bit: same kernels, same orders) and against
the oracle.  test_wide_above_2_31 builds a real 2.16e9-nonzero matrix when the device has
the memory, and checks K4, the seg layout and the SpMV on sampled rows against the oracle.
"""

import contextlib

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _cuda, cache, kernels, synth
from paper_2308_00106_b200.seg import seg_of

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12


@contextlib.contextmanager
def wide():
    old = _cuda.FORCE_WIDE_ROW_PTR
    _cuda.FORCE_WIDE_ROW_PTR = True
    try:
        yield
    finally:
        _cuda.FORCE_WIDE_ROW_PTR = old


def ragged_csr(seed=5, n_cols=20_000):
    """Row lengths covering every sort path (<= 32 tile, 33..256 warp, 257..4096 block,
    > 4096 long) and empty rows, so every fill path of the seg layout runs too."""
    rng = np.random.default_rng(seed)
    lens = np.concatenate([rng.integers(0, 33, 300), [0, 0, 40, 100, 256, 257, 600, 4096, 4097, 9000],
                           rng.integers(0, 8, 200)])
    rng.shuffle(lens)
    ptr = np.zeros(lens.size + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, int(L), replace=False)) for L in lens if L])
    val = rng.random(col.size) * 2 - 1
    return ptr, col, val, n_cols


def both(ptr, col, val, n_cols):
    narrow = P.CsrMatrix(len(ptr) - 1, n_cols, ptr, col, val)
    with wide():
        w = P.CsrMatrix(len(ptr) - 1, n_cols, ptr, col, val)
    assert narrow.d_row_ptr.dtype == torch.int32 and w.d_row_ptr.dtype == torch.int64 and w.wide
    return narrow, w


def same_csr(a, b):
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))


def test_wide_validation_errors():
    ptr, col, val, n = ragged_csr()
    with wide():
        bad = col.copy()
        r = int(np.argmax(np.diff(ptr) > 3))
        bad[ptr[r] + 1] = bad[ptr[r]]
        with pytest.raises(ValueError, match="strictly increasing"):
            P.CsrMatrix(len(ptr) - 1, n, ptr, bad, val)
        p2 = ptr.copy()
        p2[-1] += 1
        with pytest.raises(ValueError):
            P.CsrMatrix(len(ptr) - 1, n, p2, np.append(col, 0), np.append(val, 0.0))
        with pytest.raises(ValueError, match="outside"):
            P.CsrMatrix(len(ptr) - 1, n, ptr, np.where(np.arange(col.size) == 7, n, col), val)


def test_wide_coo_to_csr_and_back():
    ptr, col, val, n = ragged_csr(6)
    rows = O.csr_to_coo_rows(ptr)
    order = np.random.default_rng(1).permutation(col.size)
    narrow = P.coo_to_csr(P.CooMatrix(len(ptr) - 1, n, rows[order], col[order], val[order]))
    with wide():
        w = P.coo_to_csr(P.CooMatrix(len(ptr) - 1, n, rows[order], col[order], val[order]))
        back = P.csr_to_coo(w)
    assert w.wide and not narrow.wide
    same_csr(narrow, w)
    optr, ocol, oval = O.coo_to_csr(len(ptr) - 1, rows[order], col[order], val[order])
    assert np.array_equal(w.row_ptr, optr) and np.array_equal(w.col_idx, ocol)
    assert np.array_equal(back.row_idx, rows)
    with wide(), pytest.raises(ValueError, match="duplicate"):
        P.CooMatrix(3, 3, [0, 1, 1], [2, 0, 0], [1.0, 2.0, 3.0])


@pytest.mark.parametrize("premap", [False, True])
def test_wide_permute_csr_k4(premap, monkeypatch):
    from paper_2308_00106_b200 import permute as PM

    if premap:  # the column-sliced pre-map passes (C4's path) on a small matrix
        monkeypatch.setattr(PM, "_premap_slices", lambda m: 3)
    ptr, col, val, n = ragged_csr(7)
    narrow, w = both(ptr, col, val, n)
    p_r = P.random_permutation(narrow.n_rows, 11)
    p_c = P.random_permutation(n, 12)
    bn = P.permute_csr(narrow, p_r, p_c)
    bw = P.permute_csr(w, p_r, p_c)
    assert bw.wide
    same_csr(bn, bw)
    rows = np.arange(narrow.n_rows)
    ref = O.permute_csr_rows(ptr, col, val, p_r.forward, p_c.forward, rows)
    assert np.array_equal(bw.col_idx, np.concatenate([c for c, _ in ref]))
    assert np.array_equal(bw.values.view(np.uint64), np.concatenate([v for _, v in ref]).view(np.uint64))


def test_wide_histograms():
    ptr, col, val, n = ragged_csr(8)
    narrow, w = both(ptr, col, val, n)
    for br, bc in [(128, 128), (7, 300), (500, 64)]:
        hn, hw = P.histogram_2d(narrow, br, bc), P.histogram_2d(w, br, bc)
        assert np.array_equal(hn.counts, hw.counts)
        assert np.array_equal(hw.counts, O.histogram_2d_counts(O.csr_to_coo_rows(ptr), col, len(ptr) - 1, n, br, bc))
    assert np.array_equal(P.row_histogram(narrow, 16).counts, P.row_histogram(w, 16).counts)


@pytest.mark.parametrize("kernel,panels", [("vector", None), ("seg", 1), ("seg", 3), ("seg", 8)])
def test_wide_spmv_bitwise_equal_to_int32(kernel, panels):
    ptr, col, val, n = ragged_csr(9)
    narrow, w = both(ptr, col, val, n)
    x = O.input_vector(3, n)
    if kernel == "seg":
        for m in (narrow, w):
            seg_of(m, panels)
            m._cache["seg_panels"] = panels
    yn = np.asarray(P.spmv_csr(narrow, x, kernel))
    yw = np.asarray(P.spmv_csr(w, x, kernel))
    assert np.array_equal(yn.view(np.uint64), yw.view(np.uint64))
    assert O.relative_error(yw, O.spmv_csr(ptr, col, val, x)) <= F64_TOL
    yp = np.asarray(P.spmv_csr_parallel(w, x, 4, kernel="vector"))
    assert O.relative_error(yp, O.spmv_csr(ptr, col, val, x)) <= F64_TOL


def test_wide_rejects_int32_only_kernels():
    ptr, col, val, n = ragged_csr(10)
    _, w = both(ptr, col, val, n)
    x = np.ones(n)
    for k in ("stream", "merge", "panel", "exact"):
        with pytest.raises(ValueError, match="int64 row_ptr"):
            P.spmv_csr(w, x, k)
    assert kernels.auto_kernel(w) in kernels.WIDE_KERNELS


def test_wide_cache_round_trip(tmp_path):
    ptr, col, val, n = ragged_csr(11)
    _, w = both(ptr, col, val, n)
    lay = seg_of(w, 2)
    path = cache.save(tmp_path / "w.sme", w, layout=lay)
    back = cache.load(path, verify=True)
    assert back.d_row_ptr.dtype == torch.int64
    same_csr(w, back)


def test_wide_above_2_31():
    """A real nnz >= 2^31 matrix: 108M rows x 20 random columns = 2.16e9 nonzeros (f64,
    ~96 GB with its permuted copy and seg layout).  K4 rows, the 2-D histogram total and
    the SpMV are checked against the oracle on sampled rows."""
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip(f"needs ~120 GB of free device memory ({free / 1e9:.0f} GB free)")
    n_rows, n_cols, k = 108_000_000, 50_000_000, 20
    A = synth.random_rows(n_rows, n_cols, k)
    assert A.nnz == n_rows * k >= 2**31 and A.wide
    p_r = P.random_permutation(n_rows, 21)
    p_c = P.random_permutation(n_cols, 22)
    B = P.permute_csr(A, p_r, p_c)
    assert B.wide and int(B.d_row_ptr[-1]) == A.nnz
    rng = np.random.default_rng(3)
    rows = np.sort(rng.choice(n_rows, 2000, replace=False))
    # oracle rows of B: generator rows inverse(p_r)[rows], columns through p_c, sorted
    inv_r = p_r.d_inverse[torch.from_numpy(rows).cuda()].cpu().numpy()
    src_col, src_val = O.random_rows_fast(inv_r, n_cols, k, synth.C4_SEED)
    fc = p_c.d_forward.cpu().numpy()
    mapped = fc[src_col.reshape(-1, k)]
    order = np.argsort(mapped, axis=1, kind="stable")
    o_col = np.take_along_axis(mapped, order, 1)
    o_val = np.take_along_axis(src_val.reshape(-1, k), order, 1)
    starts = torch.from_numpy(rows).cuda()
    bptr = B.d_row_ptr[starts]
    idx = (bptr[:, None] + torch.arange(k, device="cuda")[None, :]).reshape(-1)
    assert np.array_equal(B.d_col_idx[idx].cpu().numpy().reshape(-1, k), o_col)
    assert np.array_equal(B.d_values[idx].cpu().numpy().reshape(-1, k).view(np.uint64), o_val.view(np.uint64))
    h = P.histogram_2d(B, 128, 128)
    assert int(h.counts.sum()) == A.nnz
    del A
    torch.cuda.empty_cache()
    x = torch.rand(n_cols, dtype=torch.float64, device="cuda")
    y = P.spmv_csr(B, x)  # auto: seg (x is 400 MB)
    assert kernels.auto_kernel(B) == "seg"
    xs = x.cpu().numpy()
    sptr = np.arange(rows.size + 1, dtype=np.int64) * k
    y_o = O.spmv_csr(sptr, o_col.reshape(-1), o_val.reshape(-1), xs)
    assert O.relative_error(y[starts].cpu().numpy(), y_o) <= F64_TOL
