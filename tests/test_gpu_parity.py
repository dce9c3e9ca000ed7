"""Parity of the CUDA path with the reference (golden vectors) and the CPU oracle.

Bars: permutations, permuted CSR and histogram counts
bit-exact; SpMV normwise relative error <= 1e-12 (f64) / 1e-5 (f32, against
the f64 oracle on the f32-rounded inputs); the reduceat-order kernel bitwise.
"""

import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from conftest import golden_cases
from paper_2308_00106_b200 import rowshard, synth
from paper_2308_00106_b200.kernels import spmv_into

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12
F32_TOL = 1e-5


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def gcase(golden, c):
    return lambda k: golden[f"{c}/{k}"]


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda")


# ---------------------------------------------------------------------------
# golden vectors: the whole pipeline on every reference case
# ---------------------------------------------------------------------------
def test_pipeline_matches_reference_golden(golden, dev):
    for c in golden_cases(golden):
        g = gcase(golden, c)
        n_rows, n_cols = (int(v) for v in g("shape"))
        m = P.CooMatrix(n_rows, n_cols, g("row"), g("col"), g("val"))
        csr0 = P.coo_to_csr(m)
        assert np.array_equal(csr0.row_ptr, g("csr0_ptr")), c
        assert np.array_equal(csr0.col_idx, g("csr0_col")), c
        assert np.array_equal(bits(csr0.values), bits(g("csr0_val"))), c
        p_r, p_c = P.Permutation(g("p_r")), P.Permutation(g("p_c"))
        perm = P.permute_matrix(m, p_r, p_c)
        assert np.array_equal(perm.row_idx, g("perm_row")) and np.array_equal(perm.col_idx, g("perm_col")), c
        # fused permuted CSR (row gather + segmented sort) == coo_to_csr(permute_matrix(.))
        csr = P.coo_to_csr(perm)
        assert np.array_equal(csr.row_ptr, g("csr_ptr")), c
        assert np.array_equal(csr.col_idx, g("csr_col")), c
        assert np.array_equal(bits(csr.values), bits(g("csr_val"))), c
        # the general COO path with maps applied inside the build
        csr_b = P.CooMatrix(n_rows, n_cols, g("perm_row"), g("perm_col"), g("val"))
        assert P.coo_to_csr(csr_b) == csr, c
        x_perm = P.permute_vector(g("x"), p_c)
        assert np.array_equal(bits(x_perm), bits(g("x_perm"))), c
        for kernel in ("vector", "merge", "stream"):
            y = P.spmv_csr(csr, x_perm, kernel)
            assert P.relative_error(y, g("y")) <= F64_TOL, (c, kernel)
            assert O.relative_error(y, g("y")) <= F64_TOL, (c, kernel)
        y_exact = P.spmv_csr(csr, x_perm, "exact")
        assert np.array_equal(bits(y_exact), bits(g("y"))), c
        assert np.array_equal(bits(P.spmv_csr(csr0, g("x"), "exact")), bits(g("y0"))), c
        par = P.spmv_csr_parallel(csr, x_perm, min(4, n_rows))
        assert np.array_equal(bits(par), bits(P.spmv_csr(csr, x_perm))), c
        # round trip of Eq. (1): P_r y == (P_r A P_c)(P_c^-1 x)
        assert P.relative_error(P.spmv_csr(csr, x_perm, "merge"), g("y_expected")) <= F64_TOL, c
        if f"{c}/hist" in golden:
            br, bc = (int(v) for v in g("bins2d"))
            h_coo = P.histogram_2d(P.CooMatrix(n_rows, n_cols, g("perm_row"), g("perm_col"), g("val")), br, bc)
            h_csr = P.histogram_2d(csr, br, bc)
            h0 = P.histogram_2d(csr0, br, bc)
            assert np.array_equal(h_csr.counts, g("hist")), c
            assert np.array_equal(h0.counts, g("hist0")), c
            assert np.array_equal(P.histogram_2d(perm, br, bc).counts, g("hist")), c
            assert np.array_equal(h_coo.counts, g("hist")), c
            H = P.shannon_entropy(h_csr)
            assert H == pytest.approx(float(g("H")), rel=1e-12, abs=1e-12), c
            b1r, b1c = min(512, n_rows), min(512, n_cols)
            assert np.array_equal(P.row_histogram(csr, b1r).counts, g("rowhist")), c
            assert np.array_equal(P.col_histogram(csr, b1c).counts, g("colhist")), c


@pytest.mark.parametrize("mode", [0, 1])
def test_both_merge_kernels_match_reference(golden, dev, mode):
    from paper_2308_00106_b200.kernels import set_merge_mode

    set_merge_mode(mode)
    try:
        for c in golden_cases(golden):
            g = gcase(golden, c)
            n_rows, n_cols = (int(v) for v in g("shape"))
            csr = P.CsrMatrix(n_rows, n_cols, g("csr_ptr"), g("csr_col"), g("csr_val"))
            y = P.spmv_csr(csr, g("x_perm"), "merge")
            assert O.relative_error(y, g("y")) <= F64_TOL, (c, mode)
            again = P.spmv_csr(csr, g("x_perm"), "merge")
            assert np.array_equal(bits(y), bits(again)), (c, mode)  # deterministic
    finally:
        set_merge_mode(-1)


def test_coo_histogram_kernel_matches_reference(golden, dev):
    for c in golden_cases(golden):
        g = gcase(golden, c)
        if f"{c}/hist" not in golden:
            continue
        n_rows, n_cols = (int(v) for v in g("shape"))
        br, bc = (int(v) for v in g("bins2d"))
        m = P.CooMatrix(n_rows, n_cols, g("perm_row"), g("perm_col"), g("val"))
        m._csr = None  # force the COO kernel
        assert np.array_equal(P.histogram_2d(m, br, bc).counts, g("hist")), c


def test_entropy_known_answers(golden, dev):
    cnt = golden["ent/counts"]
    h = P.BinnedHistogram(cnt, (np.arange(cnt.size + 1),))
    assert P.shannon_entropy(h) == pytest.approx(float(golden["ent/H2"]), rel=1e-12)
    assert P.shannon_entropy(h, base=math.e) == pytest.approx(float(golden["ent/He"]), rel=1e-12)
    assert P.shannon_entropy(h, base=10.0) == pytest.approx(float(golden["ent/H10"]), rel=1e-12)
    one = lambda c: P.BinnedHistogram(np.asarray(c), (np.arange(len(c) + 1),))  # noqa: E731
    assert P.shannon_entropy(one([1, 1, 2])) == 1.5  # test_entropy.py:103-104 (exact)
    assert P.shannon_entropy(one([0, 9, 0, 0])) == 0.0
    for b in (2, 256, 1024):
        assert P.shannon_entropy(one(np.full(b, 3))) == pytest.approx(math.log2(b), abs=1e-12)
    with pytest.raises(ValueError, match="empty"):
        P.shannon_entropy(one([0, 0, 0]))


# ---------------------------------------------------------------------------
# reference unit-test semantics on the drop-in API
# ---------------------------------------------------------------------------
def test_reference_kats(dev):
    m = P.CooMatrix(2, 2, [0, 0, 1], [0, 1, 1], [1.0, 2.0, 3.0])
    assert P.spmv_csr(P.coo_to_csr(m), np.array([1.0, 1.0])).tolist() == [3.0, 3.0]
    ident = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
    assert P.spmv_csr(P.coo_to_csr(ident), np.array([4.0, 5.0, 6.0])).tolist() == [4.0, 5.0, 6.0]
    assert P.spmv_coo(ident, np.array([4.0, 5.0, 6.0])).tolist() == [4.0, 5.0, 6.0]
    assert P.spmv_coo(P.CooMatrix(3, 2, [], [], []), np.array([1.0, 2.0])).tolist() == [0.0, 0.0, 0.0]
    e = P.coo_to_csr(P.CooMatrix(3, 3, [0, 2], [1, 2], [5.0, 6.0]))
    assert e.row_ptr.tolist() == [0, 1, 1, 2]
    p = P.Permutation([2, 0, 1])
    assert P.inverse(p) == P.Permutation([1, 2, 0])
    assert P.permute_vector(np.array([10.0, 20.0, 30.0]), p).tolist() == [20.0, 30.0, 10.0]
    q = P.random_permutation(31, 5)
    assert P.compose(q, P.inverse(q)) == P.identity_permutation(31)
    assert P.inverse(P.inverse(q)) == q
    h = P.histogram_2d(ident, 3, 3)
    assert h.counts.tolist() == [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    assert P.histogram_2d(P.CooMatrix(4, 4, np.arange(4), np.arange(4), np.ones(4)), 2, 2).counts.tolist() == [[2, 0], [0, 2]]
    assert P.row_histogram(P.CooMatrix(10, 1, [9], [0], [1.0]), 3).counts.tolist() == [0, 0, 1]
    m7 = P.CooMatrix(100, 100, [0] * 7, list(range(7)), np.ones(7))
    assert P.row_histogram(m7, 10).counts.tolist() == [7] + [0] * 9
    assert P.col_histogram(P.CooMatrix(4, 4, [0, 1, 2, 3], [0, 0, 0, 3], np.ones(4)), 4).counts.tolist() == [3, 0, 0, 1]


def test_reference_error_behaviour(dev):
    with pytest.raises(ValueError, match="duplicate entry at \\(0, 1\\)"):
        P.CooMatrix(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="duplicate entry at \\(3, 7\\)"):
        P.CooMatrix(10, 10, [5, 3, 3, 5, 1], [2, 7, 7, 2, 0], np.ones(5))
    with pytest.raises(ValueError, match="row index outside"):
        P.CooMatrix(2, 2, [0, 2], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="column index outside"):
        P.CooMatrix(2, 2, [0, 1], [0, -1], [1.0, 1.0])
    with pytest.raises(ValueError, match="identical length"):
        P.CooMatrix(2, 2, [0, 1], [0], [1.0, 1.0])
    with pytest.raises(ValueError, match="bijection"):
        P.Permutation([0, 0, 1])
    with pytest.raises(ValueError, match="bijection"):
        P.Permutation([0, 3, 1])
    with pytest.raises(ValueError, match="strictly increasing"):
        P.CsrMatrix(1, 3, [0, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="start at 0"):
        P.CsrMatrix(1, 3, [1, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="non-decreasing"):
        P.CsrMatrix(2, 3, [0, 2, 1], [0], [1.0])
    with pytest.raises(ValueError, match="column index outside"):
        P.CsrMatrix(1, 3, [0, 1], [3], [1.0])
    with pytest.raises(ValueError, match="n_rows \\+ 1"):
        P.CsrMatrix(2, 3, [0, 1], [0], [1.0])
    m = P.CooMatrix(4, 5, [0, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        P.spmv_coo(m, np.zeros(4))
    with pytest.raises(ValueError):
        P.spmv_csr(P.coo_to_csr(m), np.zeros(6))
    with pytest.raises(ValueError):
        P.spmv_csr_parallel(P.coo_to_csr(m), np.zeros(5), 0)
    with pytest.raises(ValueError):
        P.permute_vector(np.zeros(2), P.identity_permutation(3))
    with pytest.raises(ValueError):
        P.histogram_2d(m, 5, 2)


def test_duplicate_reported_in_row_major_order_like_lexsort(dev, rng):
    for _ in range(20):
        n = int(rng.integers(2, 40))
        k = int(rng.integers(2, 3 * n))
        rows = rng.integers(0, n, k)
        cols = rng.integers(0, n, k)
        dup = O.find_duplicate(rows, cols)
        if dup is None:
            P.CooMatrix(n, n, rows, cols, np.ones(k))
        else:
            with pytest.raises(ValueError, match=f"duplicate entry at \\({dup[0]}, {dup[1]}\\)"):
                P.CooMatrix(n, n, rows, cols, np.ones(k))


# ---------------------------------------------------------------------------
# random matrices against the oracle (seeded), incl. ragged rows and f32
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (300, 200), (2000, 3000), (5000, 5000)])
def test_random_pipeline_vs_oracle(dev, rng, shape):
    n_rows, n_cols = shape
    dens = min(1.0, 20.0 / n_cols)
    rows, cols = np.nonzero(rng.random(shape) < dens)
    vals = rng.random(rows.size) * 2 - 1
    order = rng.permutation(rows.size)
    rows, cols, vals = rows[order], cols[order], vals[order]
    p_r, p_c = O.random_permutation(n_rows, 1), O.random_permutation(n_cols, 2)
    m = P.CooMatrix(n_rows, n_cols, rows, cols, vals)
    csr = P.coo_to_csr(P.permute_matrix(m, P.Permutation(p_r), P.Permutation(p_c)))
    pr2, pc2 = O.permute_coo(rows, cols, p_r, p_c)
    optr, ocol, oval = O.coo_to_csr(n_rows, pr2, pc2, vals)
    assert np.array_equal(csr.row_ptr, optr) and np.array_equal(csr.col_idx, ocol)
    assert np.array_equal(bits(csr.values), bits(oval))
    x = O.input_vector(0, n_cols)
    xp = O.permute_vector(x, p_c)
    want = O.spmv_csr(optr, ocol, oval, xp)
    for kernel in ("vector", "merge", "stream"):
        assert O.relative_error(P.spmv_csr(csr, xp, kernel), want) <= F64_TOL
    assert np.array_equal(bits(P.spmv_csr(csr, xp, "exact")), bits(want))
    br, bc = min(128, n_rows), min(128, n_cols)
    assert np.array_equal(P.histogram_2d(csr, br, bc).counts, O.histogram_2d_counts(pr2, pc2, n_rows, n_cols, br, bc))


def test_power_law_rows_merge_kernel(dev, rng):
    """Ragged rows (0 .. 20000 nnz, many empty) exercise merge tiles spanning rows and the fix-up."""
    n_rows, n_cols = 3000, 50000
    lens = np.minimum((rng.pareto(1.2, n_rows) * 3).astype(np.int64), 20000)
    lens[rng.random(n_rows) < 0.3] = 0
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens if L] or [np.zeros(0, int)])
    val = rng.random(col.size) * 2 - 1
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    x = rng.random(n_cols)
    want = O.spmv_csr(ptr, col, val, x)
    for kernel in ("vector", "merge", "stream"):
        assert O.relative_error(P.spmv_csr(m, x, kernel), want) <= F64_TOL, kernel
    # accumulate mode: y += A x
    xd = torch.from_numpy(x).to(dev)
    for kernel in ("merge", "stream", "vector"):
        y = torch.ones(n_rows, dtype=torch.float64, device=dev)
        spmv_into(m, xd, y, kernel, accumulate=True)
        assert O.relative_error(y.cpu().numpy(), want + 1.0) <= F64_TOL, kernel
    # permuted with long rows (> 4096: chunked merge sort path)
    p_r, p_c = O.random_permutation(n_rows, 3), O.random_permutation(n_cols, 4)
    pm = P.permute_csr(m, P.Permutation(p_r), P.Permutation(p_c))
    rows = O.csr_to_coo_rows(ptr)
    pr2, pc2 = O.permute_coo(rows, col, p_r, p_c)
    optr, ocol, oval = O.coo_to_csr(n_rows, pr2, pc2, val)
    assert np.array_equal(pm.row_ptr, optr) and np.array_equal(pm.col_idx, ocol)
    assert np.array_equal(bits(pm.values), bits(oval))


def test_f32_spmv_within_1e5(dev, rng):
    n = 4000
    rows, cols = np.nonzero(rng.random((n, n)) < 0.01)
    vals = (rng.random(rows.size) * 2 - 1).astype(np.float32)
    x = rng.random(n).astype(np.float32)
    m = P.CooMatrix(n, n, rows, cols, vals, dtype=np.float32)
    csr = P.coo_to_csr(m)
    assert csr.dtype == torch.float32
    optr, ocol, oval = O.coo_to_csr(n, rows, cols, vals.astype(np.float64))
    want = O.spmv_csr(optr, ocol, oval, x.astype(np.float64))
    xd = torch.from_numpy(x).to(dev)
    for kernel in ("vector", "merge", "stream"):
        y = P.spmv_csr(csr, xd, kernel)
        assert y.dtype == torch.float32
        assert O.relative_error(y.double().cpu().numpy(), want) <= F32_TOL, kernel


# ---------------------------------------------------------------------------
# generators and large-size properties (C2 / C4 shapes at reduced scale)
# ---------------------------------------------------------------------------
def test_laplacian_generator_matches_oracle(dev):
    for g in (1, 2, 3, 17, 200):
        m = synth.laplacian5(g)
        ptr, col, val = O.laplacian5(g)
        assert np.array_equal(m.row_ptr, ptr) and np.array_equal(m.col_idx, col)
        assert np.array_equal(m.values, val)


def test_random_rows_generator_matches_oracle(dev):
    m = synth.random_rows(100_000, 1_000_000, 20, seed=99)
    sample = np.r_[0, 1, 2, 777, 50_000, 99_999]
    cols, vals = O.random_rows(sample, 1_000_000, 20, 99)
    for i, r in enumerate(sample):
        a = 20 * r
        assert np.array_equal(m.col_idx[a : a + 20], cols[i])
        assert np.array_equal(bits(m.values[a : a + 20]), bits(vals[i]))
    small = synth.random_rows(50, 25, 20, seed=7)  # several draw rounds
    cols, _ = O.random_rows(np.arange(50), 25, 20, 7)
    assert np.array_equal(small.col_idx.reshape(50, 20), cols)


def test_c2_scale_properties(dev):
    """C2 at full size: permute round trip (Eq. 1), kernel agreement, histogram totals,
    entropy gain, and the permuted CSR on sampled rows vs the oracle."""
    A = synth.laplacian5(2000)
    n = A.n_rows
    x = torch.from_numpy(O.input_vector(0, n)).to(dev)
    p_r, p_c = P.random_permutation(n, 11), P.random_permutation(n, 12)
    B = P.permute_csr(A, p_r, p_c)
    y0 = P.spmv_csr(A, x, "merge")
    y = P.spmv_csr(B, P.permute_vector(x, p_c), "merge")
    assert P.relative_error(y, P.permute_vector(y0, p_r)) <= F64_TOL
    assert P.relative_error(P.spmv_csr(B, P.permute_vector(x, p_c), "vector"), y) <= F64_TOL
    hA, hB = P.histogram_2d(A, 128, 128), P.histogram_2d(B, 128, 128)
    assert hA.total == hB.total == A.nnz
    assert P.shannon_entropy(hB) > P.shannon_entropy(hA) + 5.0
    rows = np.r_[0, 1, 12345, n // 2, n - 1]
    ptr, col, val = O.laplacian5(2000)
    want = O.permute_csr_rows(ptr, col, val, p_r.forward, p_c.forward, rows)
    bptr = B.row_ptr
    for r, (c, v) in zip(rows, want):
        assert np.array_equal(B.col_idx[bptr[r] : bptr[r + 1]], c)
        assert np.array_equal(B.values[bptr[r] : bptr[r + 1]], v)
    # the CSR-vector kernel is row-partition invariant -> shards are bitwise equal
    par = P.spmv_csr_parallel(B, P.permute_vector(x, p_c), 7)
    assert torch.equal(par, P.spmv_csr(B, P.permute_vector(x, p_c), "vector"))


def test_virtual_rowshard_bitwise_equals_single_gpu(dev):
    A = synth.random_rows(200_003, 200_003, 20, seed=5)
    x = torch.from_numpy(O.input_vector(0, A.n_cols)).to(dev)
    ref = P.spmv_csr(A, x, "vector")
    for world in (2, 3, 8):
        shards = rowshard.virtual_ranks(A, world)
        assert sum(s.nnz for s in shards) == A.nnz
        assert torch.equal(rowshard.virtual_step(shards, x), ref), world
    shards = rowshard.virtual_ranks(A, 4, kernel="merge")
    assert P.relative_error(rowshard.virtual_step(shards, x), ref) <= F64_TOL


def test_rowshard_remap_kernel_matches_oracle(dev):
    from paper_2308_00106_b200 import _lib
    from paper_2308_00106_b200._cuda import ptr, stream

    n, parts = 1_000_003, 8
    pad = -(-n // parts)
    col = torch.arange(n, dtype=torch.int32, device=dev)
    out = torch.empty_like(col)
    _lib.call("sme_rowshard_remap_cols", n, n, parts, pad, ptr(col), ptr(out), stream())
    assert np.array_equal(out.cpu().numpy(), O.rowshard_remap_cols(np.arange(n), n, parts, pad))


def test_gpu_kernelspecs_plug_into_protocol(dev, golden):
    from paper_2308_00106_b200.bench import PermutedOperands, gpu_kernels, time_kernel

    g = gcase(golden, "c1")
    n = int(g("shape")[0])
    csr = P.CsrMatrix(n, n, g("csr_ptr"), g("csr_col"), g("csr_val"))
    ops = PermutedOperands(None, csr)
    for spec in gpu_kernels(max_workers=3):
        secs, y = time_kernel(spec.fn, ops, g("x_perm"), 3)
        assert secs > 0
        assert O.relative_error(np.asarray(y), g("y_expected")) <= F64_TOL, spec.kernel_id


@pytest.mark.parametrize("n_panels", [1, 2, 3, 7])
def test_panel_layout_matches_oracle(dev, rng, n_panels):
    from paper_2308_00106_b200.panels import PanelCsr

    n_rows, n_cols = 3000, 5000
    lens = rng.integers(0, 60, n_rows)
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens])
    val = rng.random(col.size) * 2 - 1
    m = P.CsrMatrix(n_rows, n_cols, ptr, col, val)
    pc = PanelCsr(m, n_panels)
    assert pc.nnz == m.nnz
    b = [p * n_cols // n_panels for p in range(n_panels + 1)]
    for p, a in enumerate(pc.panels):
        # each panel is the column slice of every row, columns still ascending
        rows = O.csr_to_coo_rows(ptr)
        sel = (col >= b[p]) & (col < b[p + 1])
        optr, ocol, oval = O.coo_to_csr(n_rows, rows[sel], col[sel], val[sel])
        assert np.array_equal(a.row_ptr, optr) and np.array_equal(a.col_idx, ocol)
        assert np.array_equal(bits(a.values), bits(oval))
    x = rng.random(n_cols)
    m._cache["n_panels"] = n_panels
    want = O.spmv_csr(ptr, col, val, x)
    assert O.relative_error(P.spmv_csr(m, x, "panel"), want) <= F64_TOL


@pytest.mark.parametrize("fuse_last", [False, True])
@pytest.mark.parametrize("slice_cols", [1 << 30, 20_000, 7_001, 997])
def test_permute_csr_premap_path_is_bit_identical(dev, rng, slice_cols, fuse_last):
    """K4 with the column pre-map forced on (sme_map_cols_sliced_partial: 1, 1, 3 and 21
    slices, i.e. the single pass and the first / middle / last in-place flagged passes,
    with the last slice mapped by its own pass or by the row sort, which then also clears
    the flags) builds the same permuted CSR, bit for bit, as the in-sort gather, and the
    same as the oracle."""
    import paper_2308_00106_b200.permute as PM

    n = 20_000
    mask = rng.random((400, n)) < 0.01
    rows, cols = np.nonzero(mask)
    m = P.coo_to_csr(P.CooMatrix(400, n, rows, cols, rng.random(rows.size)))
    p_r, p_c = P.random_permutation(400, 3), P.random_permutation(n, 4)
    saved = PM.PREMAP, PM.PREMAP_SLICE_BYTES, PM.PREMAP_FUSE_LAST
    try:
        PM.PREMAP, PM.PREMAP_SLICE_BYTES, PM.PREMAP_FUSE_LAST = True, slice_cols * 4, fuse_last
        assert PM._premap_slices(m) == -(-n // slice_cols)
        a = P.permute_csr(m, p_r, p_c)
        PM.PREMAP = False
        b = P.permute_csr(m, p_r, p_c)
    finally:
        PM.PREMAP, PM.PREMAP_SLICE_BYTES, PM.PREMAP_FUSE_LAST = saved
    pr, pc = O.permute_coo(rows, cols, p_r.forward, p_c.forward)
    optr, ocol, _ = O.coo_to_csr(400, pr, pc, np.zeros(rows.size))  # structure only; values: a == b above
    assert np.array_equal(a.row_ptr, optr) and np.array_equal(a.col_idx, ocol)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
