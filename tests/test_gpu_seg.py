"""The segmented-chunk layout (spmv_seg.cu / seg.py) against the CPU oracle.

Layout: decoding every panel's 32-bit words and chunk headers must give back
the CSR entries of that column range, bit for bit, in row-major order, plus
exactly the explicit zeros the layout promises.  SpMV: normwise relative
error <= 1e-12 (f64, kernels.py:131-142 / bench.py:34) and <= 1e-5 (f32).
"""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200.seg import CHUNK, SegLayout

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12
F32_TOL = 1e-5
MARK = (1 << 23) - 1


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda")


def csr_from_lens(rng, lens, n_cols, dtype=np.float64):
    ptr = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    parts = [np.sort(rng.choice(n_cols, int(L), replace=False)) for L in lens if L]
    col = np.concatenate(parts) if parts else np.zeros(0, np.int64)
    val = (rng.random(col.size) * 2 - 1).astype(dtype)
    return ptr, col, val


def decode(lay: SegLayout):
    """Per panel: (rows, cols, vals, is_zero, end_of_row) decoded from pk/hdr/val on the host."""
    pk = lay.pk.cpu().numpy().view(np.uint32).astype(np.int64)
    hdr = lay.hdr.cpu().numpy().astype(np.int64)
    val = lay.val.cpu().numpy()
    out = []
    for p in range(lay.n_panels):
        o, e = int(lay.offsets[p]), int(lay.entries[p])
        pos = np.arange(o, o + e)
        w = pk[o : o + e]
        lc, end, d = w >> 9, (w >> 8) & 1, w & 255
        rows = hdr[pos // CHUNK] + d
        zero = lc == MARK
        cols = np.where(zero, -1, lc + int(lay.bounds_host[p]))
        out.append((rows, cols, val[o : o + e], zero, end.astype(bool)))
    return out


def check_layout(lay, ptr, col, val, full_last=False):
    n_rows = len(ptr) - 1
    rows_all = O.csr_to_coo_rows(ptr)
    for p, (rows, cols, vals, zero, end) in enumerate(decode(lay)):
        lo, hi = int(lay.bounds_host[p]), int(lay.bounds_host[p + 1])
        assert np.all(np.diff(rows) >= 0), p  # row-major
        sel = (col >= lo) & (col < hi)
        assert np.array_equal(rows[~zero], rows_all[sel]), p
        assert np.array_equal(cols[~zero], col[sel]), p
        assert np.array_equal(vals[~zero].view(np.uint8), val[sel].view(np.uint8)), p
        assert np.all(vals[zero] == 0), p
        # explicit zeros: panel 0 every row without entries; later panels empty rows r % 2 == 0
        has = np.zeros(n_rows, bool)
        has[rows_all[sel]] = True
        every = p == 0 or (full_last and p == lay.n_panels - 1)
        want_zero = np.flatnonzero(~has) if every else np.flatnonzero(~has & (np.arange(n_rows) % 2 == 0))
        assert np.array_equal(rows[zero], want_zero), p
        # end flag exactly on the last entry of every row
        want_end = np.ones(rows.size, bool)
        want_end[:-1] = rows[1:] != rows[:-1]
        assert np.array_equal(end, want_end), p
        # every chunk spans < 256 rows (8-bit offsets) -- implied by decode, checked explicitly
        if rows.size:
            starts = rows[::CHUNK]
            ends = rows[np.minimum(np.arange(0, rows.size, CHUNK) + CHUNK - 1, rows.size - 1)]
            assert np.all(ends - starts <= 255)


def run_seg(m, x, n_panels, n_warps=None, full_last=False):
    lay = SegLayout(m, n_panels, n_warps, full_last=full_last)
    xd = torch.as_tensor(x).to(m.d_values.device, m.dtype)
    y = torch.full((m.n_rows,), float("nan"), dtype=m.dtype, device=xd.device)  # every row must be written
    lay.spmv_into(xd, y)
    return lay, y.double().cpu().numpy()


@pytest.mark.parametrize("full_last", [False, True])
@pytest.mark.parametrize("n_panels", [1, 2, 3, 7])
def test_layout_and_spmv_random_lengths(dev, rng, n_panels, full_last):
    n_rows, n_cols = 3000, 5000
    lens = rng.integers(0, 60, n_rows)
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols)
    lay, y = run_seg(m, x, n_panels, full_last=full_last)
    check_layout(lay, ptr, col, val, full_last)
    assert O.relative_error(y, O.spmv_csr(ptr, col, val, x)) <= F64_TOL


@pytest.mark.parametrize("n_warps", [1, 2, 3, 37, 1000])
def test_warp_splits_and_carries(dev, rng, n_warps):
    """Few warps: long chunk runs, rows carried across chunks and warp boundaries."""
    n_rows, n_cols = 2500, 4000
    lens = np.minimum((rng.pareto(1.1, n_rows) * 4).astype(np.int64), 3000)  # rows up to 3000 entries
    lens[rng.random(n_rows) < 0.4] = 0
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols) * 2 - 1
    want = O.spmv_csr(ptr, col, val, x)
    for n_panels in (1, 3):
        lay, y = run_seg(m, x, n_panels, n_warps)
        check_layout(lay, ptr, col, val)
        assert O.relative_error(y, want) <= F64_TOL, (n_warps, n_panels)


def test_sparse_panels_many_empty_rows(dev, rng):
    """Most rows empty in most panels: the r % 2 explicit zeros keep chunk spans < 256 rows."""
    n_rows, n_cols = 20000, 100000
    lens = (rng.random(n_rows) < 0.05).astype(np.int64) * rng.integers(1, 4, n_rows)
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols)
    lay, y = run_seg(m, x, 9)
    check_layout(lay, ptr, col, val)
    assert O.relative_error(y, O.spmv_csr(ptr, col, val, x)) <= F64_TOL


@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (300, 200), (5000, 5000)])
def test_permuted_pipeline_seg(dev, rng, shape):
    n_rows, n_cols = shape
    dens = min(1.0, 20.0 / n_cols)
    rows, cols = np.nonzero(rng.random(shape) < dens)
    vals = rng.random(rows.size) * 2 - 1
    p_r, p_c = O.random_permutation(n_rows, 1), O.random_permutation(n_cols, 2)
    m = P.CooMatrix(n_rows, n_cols, rows, cols, vals)
    csr = P.coo_to_csr(P.permute_matrix(m, P.Permutation(p_r), P.Permutation(p_c)))
    pr2, pc2 = O.permute_coo(rows, cols, p_r, p_c)
    optr, ocol, oval = O.coo_to_csr(n_rows, pr2, pc2, vals)
    xp = O.permute_vector(O.input_vector(0, n_cols), p_c)
    want = O.spmv_csr(optr, ocol, oval, xp)
    assert O.relative_error(P.spmv_csr(csr, xp, "seg"), want) <= F64_TOL
    for n_panels in sorted({1, min(2, n_cols), min(5, n_cols)}):
        lay, y = run_seg(csr, xp, n_panels)
        check_layout(lay, optr, ocol, oval)
        assert O.relative_error(y, want) <= F64_TOL


def test_empty_matrix_and_empty_rows(dev, rng):
    m = P.CsrMatrix(5, 4, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0))
    lay, y = run_seg(m, np.ones(4), 2)
    assert np.array_equal(y, np.zeros(5))
    ptr = np.array([0, 0, 2, 2, 3])
    m = P.CsrMatrix(4, 3, ptr, np.array([0, 2, 1]), np.array([1.0, 2.0, 3.0]))
    lay, y = run_seg(m, np.array([1.0, 10.0, 100.0]), 2)
    assert np.array_equal(y, [0.0, 201.0, 0.0, 30.0])


def test_nonfinite_x_only_reaches_its_rows(dev):
    """Explicit zeros never gather x: an inf in x must not turn empty rows into NaN."""
    ptr = np.array([0, 1, 1, 2])
    m = P.CsrMatrix(3, 8, ptr, np.array([1, 7]), np.array([2.0, 1.0]))
    x = np.ones(8)
    x[0] = np.inf
    lay, y = run_seg(m, x, 2)
    assert np.array_equal(y, [2.0, 0.0, 1.0])


def test_f32_seg_within_1e5(dev, rng):
    n = 6000
    lens = rng.integers(0, 40, n)
    ptr, col, val = csr_from_lens(rng, lens, n, np.float32)
    x = rng.random(n).astype(np.float32)
    m = P.CsrMatrix(n, n, ptr, col, val, dtype=np.float32)
    want = O.spmv_csr(ptr, col, val.astype(np.float64), x.astype(np.float64))
    for n_panels in (1, 4):
        lay, y = run_seg(m, x, n_panels)
        assert O.relative_error(y, want) <= F32_TOL


def test_host_vector_path_overlaps_and_matches(dev, rng):
    n = 8000
    lens = rng.integers(0, 30, n)
    ptr, col, val = csr_from_lens(rng, lens, n)
    m = P.CsrMatrix(n, n, ptr, col, val)
    m._cache["seg_panels"] = 4
    x = torch.from_numpy(rng.random(n)).pin_memory()
    y = P.spmv_csr(m, x, "seg")
    assert not y.is_cuda
    assert O.relative_error(y.numpy(), O.spmv_csr(ptr, col, val, x.numpy())) <= F64_TOL


def test_panel_width_limit_is_enforced(dev):
    n_cols = (1 << 23) + 5
    m = P.CsrMatrix(2, n_cols, np.array([0, 1, 2]), np.array([0, n_cols - 1]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="23-bit"):
        SegLayout(m, 1)
    lay, y = run_seg(m, np.ones(n_cols), 2)
    assert np.array_equal(y, [1.0, 2.0])


@pytest.mark.parametrize("kernel", ["seg", "vector", "panel"])
def test_pipelined_host_stream_equals_per_vector_calls(dev, rng, kernel):
    """spmv_csr_pipelined: the same outputs as one spmv_csr call per vector (bitwise:
    same kernels, same order), with copies of neighbouring steps overlapped."""
    n = 7000
    lens = rng.integers(0, 30, n)
    ptr, col, val = csr_from_lens(rng, lens, n)
    m = P.CsrMatrix(n, n, ptr, col, val)
    m._cache["seg_panels"] = 3
    m._cache["n_panels"] = 3
    xs = [torch.from_numpy(rng.random(n)).pin_memory() for _ in range(5)]
    ys = P.spmv_csr_pipelined(m, xs, kernel=kernel)
    assert len(ys) == 5
    for x, y in zip(xs, ys):
        want = P.spmv_csr(m, x.cuda(), kernel).cpu()
        assert torch.equal(y, want)
        assert O.relative_error(y.numpy(), O.spmv_csr(ptr, col, val, x.numpy())) <= F64_TOL
    # outputs in a ring of two host buffers (bench.py's e2e): the last two survive
    ring = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    P.spmv_csr_pipelined(m, xs, [ring[k & 1] for k in range(len(xs))], kernel=kernel)
    assert torch.equal(ring[(len(xs) - 1) & 1], ys[-1]) and torch.equal(ring[(len(xs) - 2) & 1], ys[-2])
    with pytest.raises(ValueError):
        P.spmv_csr_pipelined(m, [torch.zeros(n + 1)])


@pytest.mark.parametrize("n_panels", [1, 4])
def test_very_long_rows(dev, rng, n_panels):
    """Rows of 150k and 60k entries (a warp's range always holds whole rows, so one warp
    walks them chunk by chunk with the carry) next to short and empty rows."""
    n_rows, n_cols = 400, 200_000
    lens = rng.integers(0, 5, n_rows)
    lens[7], lens[300] = 150_000, 60_000
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols) * 2 - 1
    for n_warps in (None, 5):
        lay, y = run_seg(m, x, n_panels, n_warps)
        check_layout(lay, ptr, col, val)
        assert O.relative_error(y, O.spmv_csr(ptr, col, val, x)) <= F64_TOL


def test_split_row_plans_with_empty_ranges(dev, rng):
    """More warps than entries: most split ranges are empty and sit between carries of the
    same row (the property test's 2 x 281 case)."""
    n_rows, n_cols = 2, 281
    lens = np.array([270, 0])
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols) * 2 - 1
    for n_warps in (4736, 1000, 300):
        lay = SegLayout(m, 1, n_warps, split_rows=True)
        y = torch.full((n_rows,), float("nan"), dtype=m.dtype, device=dev)
        lay.spmv_into(torch.as_tensor(x).to(dev), y)
        assert O.relative_error(y.cpu().numpy(), O.spmv_csr(ptr, col, val, x)) <= F64_TOL, n_warps


@pytest.mark.parametrize("n_panels", [1, 3])
@pytest.mark.parametrize("n_warps", [7, 37, 300])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_split_row_plans(dev, rng, n_panels, n_warps, dtype):
    """Split-row plans: warp ranges end mid-row (a 150k-entry row spans many warps) and the
    ordered fix-up adds the open partials; same result as whole-row plans and the oracle."""
    n_rows, n_cols = 600, 200_000
    lens = rng.integers(0, 6, n_rows)
    lens[11], lens[400], lens[599] = 150_000, 40_000, 9_000
    ptr, col, val = csr_from_lens(rng, lens, n_cols, dtype)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val, dtype=dtype)
    x = (rng.random(n_cols) * 2 - 1).astype(dtype)
    want = O.spmv_csr(ptr, col, val.astype(np.float64), x.astype(np.float64))
    tol = F64_TOL if dtype == np.float64 else F32_TOL
    split = SegLayout(m, n_panels, n_warps, split_rows=True)
    whole = SegLayout(m, n_panels, n_warps, split_rows=False)
    assert split.split_rows and not whole.split_rows
    for lay in (split, whole):
        xd = torch.as_tensor(x).to(dev)
        y = torch.full((n_rows,), float("nan"), dtype=m.dtype, device=dev)
        lay.spmv_into(xd, y)
        assert O.relative_error(y.double().cpu().numpy(), want) <= tol
    # repeated calls are deterministic
    y1 = torch.empty(n_rows, dtype=m.dtype, device=dev)
    y2 = torch.empty(n_rows, dtype=m.dtype, device=dev)
    split.spmv_into(torch.as_tensor(x).to(dev), y1)
    split.spmv_into(torch.as_tensor(x).to(dev), y2)
    assert torch.equal(y1, y2)


def test_split_rows_chosen_automatically_for_dominant_rows(dev, rng):
    n_rows, n_cols = 2000, 50_000
    lens = rng.integers(0, 4, n_rows)
    lens[5] = 45_000
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    assert SegLayout(m, 1, 64).split_rows
    assert SegLayout(m, 1, 64, full_last=True).split_rows  # fused layouts too (epilogue as a row pass)
    assert not SegLayout(m, 1, 64, split_rows=False).split_rows
    lens[5] = 3
    ptr, col, val = csr_from_lens(rng, lens, n_cols)
    assert not SegLayout(P.CsrMatrix(n_rows, n_cols, ptr, col, val), 1, 64).split_rows


@pytest.mark.parametrize("kernel,dtype", [("seg", np.float64), ("vector", np.float64), ("seg", np.float32)])
def test_host_vectors_large_fresh_results(dev, rng, kernel, dtype):
    """numpy / CPU-tensor x above the staging threshold (hostio): slices staged through
    pinned memory, results in fresh pooled page-locked memory that never aliases a live
    result (the reference returns a new array per call, kernels.py:73-78)."""
    import gc

    from paper_2308_00106_b200 import hostio

    n = (hostio.CHUNK_MIN_BYTES // 8) + 12345  # x and y above the chunking threshold
    rows = np.repeat(np.arange(n), rng.integers(0, 4, n))
    cols = rng.integers(0, n, rows.size)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.ones(rows.size, dtype=bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, col = rows[keep], cols[keep]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    val = (rng.random(col.size) * 2 - 1).astype(dtype)
    m = P.CsrMatrix(n, n, ptr, col, val)
    m._cache["seg_panels"] = 3
    x1, x2 = rng.random(n), rng.random(n)
    want1 = O.spmv_csr(ptr, col, val.astype(np.float64), x1)
    want2 = O.spmv_csr(ptr, col, val.astype(np.float64), x2)
    tol = F64_TOL if dtype == np.float64 else F32_TOL
    for rep in range(3):  # the pool recycles released results
        y1 = P.spmv_csr(m, x1, kernel)
        y2 = P.spmv_csr(m, x2, kernel)
        assert isinstance(y1, np.ndarray) and y1.dtype == np.float64 and y1.shape == (n,)
        assert not np.shares_memory(y1, y2)
        assert O.relative_error(y1, want1) <= tol and O.relative_error(y2, want2) <= tol
        del y1
        gc.collect()
        yt = P.spmv_csr(m, torch.from_numpy(x1).to(torch.float64 if dtype == np.float64 else torch.float32), kernel)
        assert isinstance(yt, torch.Tensor) and not yt.is_cuda and yt.dtype == m.dtype
        assert O.relative_error(yt.double().numpy(), want1) <= tol
        assert O.relative_error(y2, want2) <= tol  # untouched by the later calls
        del y2, yt
        gc.collect()


@pytest.mark.parametrize("n_panels", [1, 3, 8])
def test_grouped_fill_equals_per_row_fill(dev, rng, n_panels):
    """The grouped layout fill (warp per 32 rows through shared memory, with the per-row
    path for groups too long for the image) builds the same layout, bit for bit, as the
    per-row fill."""
    from paper_2308_00106_b200 import _lib

    n = 5000
    lens = rng.integers(0, 40, n)
    lens[[7, 8, 900]] = [3000, 1500, 2500]  # groups over the image capacity
    lens[100:180] = 0  # empty rows: explicit zeros
    ptr, col, val = csr_from_lens(rng, lens, n)
    m = P.CsrMatrix(n, n, ptr, col, val)
    layouts = []
    for on in (1, 0):
        _lib.call("sme_seg_set_scatter_groups", on)
        try:
            layouts.append(SegLayout(m, n_panels))
        finally:
            _lib.call("sme_seg_set_scatter_groups", 1)
    a, b = layouts
    assert torch.equal(a.pk, b.pk) and torch.equal(a.val, b.val) and torch.equal(a.hdr, b.hdr)


@pytest.mark.parametrize("n_panels", [1, 3, 8, 17])
@pytest.mark.parametrize("shape", ["c4_like", "ragged"])
def test_ballot_fill_equals_per_row_fill(dev, rng, n_panels, shape):
    """The entry-parallel fill of groups without empty rows (sme_seg_set_fill_ballot: row
    of an entry from the mask of row starts in its 32-entry window) builds the same
    layout, bit for bit, as the lane-per-row walk and as the per-row fill — with C4-like
    20-entry rows and with ragged rows (1..60 entries, windows holding many row starts),
    some groups with empty rows (the other paths) and some past the image capacity."""
    from paper_2308_00106_b200 import _lib

    n = 6000
    if shape == "c4_like":
        lens = np.full(n, 20)
    else:
        lens = rng.integers(1, 61, n)
        lens[rng.random(n) < 0.3] = 1
        lens[[5, 2000]] = [900, 1300]  # groups over the image capacity
        lens[3000:3010] = 0  # empty rows: those groups take the walk
    ptr, col, val = csr_from_lens(rng, lens, n)
    m = P.CsrMatrix(n, n, ptr, col, val)
    layouts = []
    # (grouped, entry-parallel, direct stores): the default, the image variants, the per-row fill
    for groups, ballot, direct in ((1, 1, 1), (1, 0, 1), (1, 1, 0), (1, 0, 0), (0, 1, 1)):
        _lib.call("sme_seg_set_scatter_groups", groups)
        _lib.call("sme_seg_set_fill_ballot", ballot)
        _lib.call("sme_seg_set_fill_direct", direct)
        try:
            layouts.append(SegLayout(m, n_panels))
        finally:
            _lib.call("sme_seg_set_scatter_groups", 1)
            _lib.call("sme_seg_set_fill_ballot", 1)
            _lib.call("sme_seg_set_fill_direct", 1)
    a = layouts[0]
    for b in layouts[1:]:
        assert torch.equal(a.pk, b.pk) and torch.equal(a.val, b.val) and torch.equal(a.hdr, b.hdr)
    x = rng.random(n)
    want = O.spmv_csr(ptr, col, val, x)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    a.spmv_into(torch.from_numpy(x).to(dev), y)
    assert O.relative_error(y.cpu().numpy(), want) <= 1e-12
