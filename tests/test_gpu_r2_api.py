"""Round-2 API parity: deterministic COO SpMV, spmv_csr_parallel on every kernel,
`out=` validation, reentrant host calls, the reference's entropy base and
col_histogram behaviour."""

from __future__ import annotations

import math
import threading

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from conftest import make_random_coo_arrays
from paper_2308_00106_b200 import synth

pytestmark = pytest.mark.gpu


def _coo(rng, n_rows, n_cols, density, dtype=np.float64):
    r, c, v = make_random_coo_arrays(rng, n_rows, n_cols, density)
    order = rng.permutation(r.size)  # shuffled entry order: np.add.at's order matters
    return r[order], c[order], v[order].astype(dtype)


@pytest.mark.parametrize("shape,density", [((1000, 700), 0.01), ((20_000, 30_000), 0.0005), ((2000, 2000), 0.25),
                                           ((300, 5), 0.9)])
def test_spmv_coo_bitwise_equals_np_add_at(rng, shape, density):
    """The default COO kernel reproduces np.add.at (kernels.py:81-86) bit for bit, at
    up to 1M nonzeros in shuffled entry order, and is run-to-run identical."""
    r, c, v = _coo(rng, *shape, density)
    m = P.CooMatrix(*shape, r, c, v)
    x = rng.random(shape[1])
    want = O.spmv_coo(shape[0], r, c, v, x)
    got = P.spmv_coo(m, x)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    xd = torch.from_numpy(x).cuda()
    first = P.spmv_coo(m, xd)
    for _ in range(4):
        assert torch.equal(P.spmv_coo(m, xd), first)


def test_spmv_coo_f32_and_atomic_within_tolerance(rng):
    r, c, v = _coo(rng, 50_000, 40_000, 0.0005)
    x = rng.random(40_000)
    want = O.spmv_coo(50_000, r, c, v, x)
    m = P.CooMatrix(50_000, 40_000, r, c, v)
    assert O.relative_error(P.spmv_coo(m, x, kernel="atomic"), want) <= 1e-12
    m32 = P.CooMatrix(50_000, 40_000, r, c, v.astype(np.float32))
    want32 = O.spmv_coo(50_000, r, c, v.astype(np.float32).astype(np.float64),
                        x.astype(np.float32).astype(np.float64))
    got32 = P.spmv_coo(m32, torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert O.relative_error(got32, want32) <= 1e-5


def test_spmv_coo_atomic_run_to_run_bound(rng):
    """The atomic variant's run-to-run spread is bounded by the f64 reassociation
    error of a row (<= nnz_row * eps * sum|products|); it stays opt-in."""
    n = 2000
    r = np.repeat(np.arange(n), 500)
    c = np.tile(np.arange(500), n)
    v = rng.standard_normal(r.size)
    m = P.CooMatrix(n, 500, r, c, v)
    x = torch.from_numpy(rng.standard_normal(500)).cuda()
    runs = torch.stack([P.spmv_coo(m, x, kernel="atomic") for _ in range(5)])
    spread = (runs.max(0).values - runs.min(0).values).abs().max().item()
    bound = 500 * 2.0**-52 * float((torch.from_numpy(np.abs(v).reshape(n, 500)).cuda() * x.abs()).sum(1).max())
    assert spread <= bound


def test_spmv_csr_parallel_bitwise_with_auto_seg():
    """on a matrix where auto resolves to 'seg', spmv_csr_parallel is bitwise
    equal to spmv_csr (the reference's parallel == serial invariant, kernels.py:1-6)."""
    A = synth.rmat(16, 16, cap=100000, dtype=np.float64)  # ragged rows -> 'seg'
    assert P.kernels.auto_kernel(A) == "seg"
    x = torch.from_numpy(O.input_vector(0, A.n_cols)).cuda()
    y = P.spmv_csr(A, x)
    for w in (1, 3, 16):
        assert torch.equal(P.spmv_csr_parallel(A, x, w), y)
    B = synth.laplacian5(300)
    assert P.kernels.auto_kernel(B) == "vector"
    xb = torch.from_numpy(O.input_vector(0, B.n_cols)).cuda()
    assert torch.equal(P.spmv_csr_parallel(B, xb, 7), P.spmv_csr(B, xb))


def test_out_is_validated():
    A = synth.laplacian5(50)
    x = torch.ones(A.n_cols, dtype=torch.float64, device="cuda")
    good = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    assert P.spmv_csr(A, x, out=good) is good
    for bad in (torch.empty(A.n_rows, dtype=torch.float32, device="cuda"),
                torch.empty(A.n_rows - 1, dtype=torch.float64, device="cuda"),
                torch.empty(2 * A.n_rows, dtype=torch.float64, device="cuda")[::2],
                torch.empty(A.n_rows, dtype=torch.float64)):
        with pytest.raises(ValueError, match="out must"):
            P.spmv_csr(A, x, out=bad)


def test_concurrent_host_calls_on_one_matrix():
    """4 threads calling spmv_csr(m, x_i) with host vectors on ONE
    matrix each get their own result (large enough for the staged/pooled paths)."""
    g = 1500  # 2.25M rows: 18 MB vectors take the chunked staging and pooled results
    A = synth.laplacian5(g)
    n = A.n_rows
    xs = [np.random.default_rng(k).random(n) for k in range(4)]
    want = [P.spmv_csr(A, torch.from_numpy(x).cuda()).cpu().numpy() for x in xs]
    errors: list = []

    def worker(k):
        try:
            for it in range(6):
                y = P.spmv_csr(A, xs[k]) if it % 2 == 0 else P.spmv_csr(A, torch.from_numpy(xs[k]))
                y = np.asarray(y)
                if not np.array_equal(y, want[k]):
                    errors.append((k, it, float(np.abs(y - want[k]).max())))
        except Exception as e:  # pragma: no cover
            errors.append((k, repr(e)))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_entropy_base_and_errors_match_reference():
    h = P.histogram_2d(P.CooMatrix(3, 3, [0, 1, 2, 2], [0, 1, 2, 0], [1.0, 1.0, 1.0, 1.0]), 3, 3)
    p = np.array([1, 1, 1, 1]) / 4
    assert P.shannon_entropy(h, base=0.5) == pytest.approx(float(-(p * np.log(p)).sum() / math.log(0.5)), rel=1e-12)
    assert P.shannon_entropy(h, base=10.0) == pytest.approx(float(-(p * np.log(p)).sum() / math.log(10.0)),
                                                            rel=1e-12)
    with pytest.raises(ZeroDivisionError):
        P.shannon_entropy(h, base=1.0)
    with pytest.raises(ValueError, match="math domain"):
        P.shannon_entropy(h, base=-2.0)
    empty = P.histogram_2d(P.CooMatrix(3, 3, [], [], []), 3, 3)
    with pytest.raises(ValueError, match="empty"):
        P.shannon_entropy(empty, base=1.0)  # the empty check comes first, as in the reference


def test_col_histogram_zero_row_matrix():
    m = P.CooMatrix(0, 6, [], [], [])
    h = P.col_histogram(m, 3)
    assert h.counts.tolist() == [0, 0, 0]
    with pytest.raises(ValueError, match="column bin count 7 exceeds"):
        P.col_histogram(m, 7)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_warp_medium_row_sort_equals_block_sort_and_oracle(dtype):
    """K4 rows with 32 < len <= 512 take the warp-wide register sort; it must equal the
    CTA-wide shared-memory sort bit for bit and the oracle's coo_to_csr(permute_matrix)."""
    from paper_2308_00106_b200 import _lib

    rng = np.random.default_rng(3)
    n = 4000
    lens = np.concatenate([rng.integers(33, 513, 900), rng.integers(0, 33, 2900), rng.integers(513, 3000, 200)])
    rng.shuffle(lens)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n, size=int(l), replace=False)) for l in lens])
    val = rng.standard_normal(col.size).astype(dtype)
    A = P.CsrMatrix(n, n, ptr, col, val)
    fr, fc = rng.permutation(n), rng.permutation(n)
    outs = []
    for wmed in (4, 0):
        _lib.call("sme_sort_rows_set_wmed", wmed)
        try:
            outs.append(P.permute_csr(A, P.Permutation(fr), P.Permutation(fc)))
        finally:
            _lib.call("sme_sort_rows_set_wmed", 3)
    a, b = outs
    assert torch.equal(a.d_row_ptr, b.d_row_ptr) and torch.equal(a.d_col_idx, b.d_col_idx)
    assert torch.equal(a.d_values.view(torch.uint8), b.d_values.view(torch.uint8))
    pr, pc = O.permute_coo(O.csr_to_coo_rows(ptr), col, fr, fc)
    ptr_o, col_o, val_o = O.coo_to_csr(n, pr, pc, val.astype(np.float64))
    assert np.array_equal(a.row_ptr, ptr_o) and np.array_equal(a.col_idx, col_o)
    assert np.array_equal(a.values, val_o)
    # the COO path (staged source) sorts its rows the same way
    coo = P.CooMatrix(n, n, pr, pc, val)
    c = P.coo_to_csr(coo)
    assert torch.equal(c.d_col_idx, a.d_col_idx) and torch.equal(c.d_values.view(torch.uint8),
                                                                  a.d_values.view(torch.uint8))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cta_hybrid_row_sort_equals_smem_sort_and_oracle(dtype):
    """K4 rows of 257..4096 entries take the CTA-wide register / shuffle / shared-memory
    bitonic network (E = 2..16 keys per thread); it must equal the all-shared-memory sort
    bit for bit and the oracle, on the CSR (gathered source) and the COO (staged) paths,
    including a duplicate reported like the reference's lexsort would."""
    from paper_2308_00106_b200 import _lib

    rng = np.random.default_rng(4)
    n = 6000
    lens = np.concatenate([[257, 300, 511, 512, 513, 1000, 1023, 1024, 1025, 2047, 2048, 2049, 3000, 4095, 4096],
                           rng.integers(257, 4097, 60), rng.integers(0, 40, 2000)])
    lens = np.concatenate([lens, np.zeros(n - lens.size, dtype=lens.dtype)])
    rng.shuffle(lens)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n, size=int(l), replace=False)) for l in lens])
    val = rng.standard_normal(col.size).astype(dtype)
    A = P.CsrMatrix(n, n, ptr, col, val)
    fr, fc = rng.permutation(n), rng.permutation(n)
    outs = []
    for cta in (1, 0):
        _lib.call("sme_sort_rows_set_cta", cta)
        try:
            outs.append(P.permute_csr(A, P.Permutation(fr), P.Permutation(fc)))
        finally:
            _lib.call("sme_sort_rows_set_cta", 1)
    a, b = outs
    assert torch.equal(a.d_row_ptr, b.d_row_ptr) and torch.equal(a.d_col_idx, b.d_col_idx)
    assert torch.equal(a.d_values.view(torch.uint8), b.d_values.view(torch.uint8))
    pr, pc = O.permute_coo(O.csr_to_coo_rows(ptr), col, fr, fc)
    ptr_o, col_o, val_o = O.coo_to_csr(n, pr, pc, val.astype(np.float64))
    assert np.array_equal(a.row_ptr, ptr_o) and np.array_equal(a.col_idx, col_o)
    assert np.array_equal(a.values, val_o)
    c = P.coo_to_csr(P.CooMatrix(n, n, pr, pc, val))
    assert torch.equal(c.d_col_idx, a.d_col_idx)
    # a duplicate inside a long row: the reference's first duplicate in lexsort order
    r_long = int(np.argmax(lens))
    rows_d = np.append(pr, pr[ptr[r_long]])
    cols_d = np.append(pc, pc[ptr[r_long]])
    vals_d = np.append(val, val[0])
    with pytest.raises(ValueError, match="duplicate"):
        P.CooMatrix(n, n, rows_d, cols_d, vals_d)
