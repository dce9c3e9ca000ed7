"""2-D histogram kernels (hist.cu) against the oracle's bincount (entropy.py:91-101):
the lane-private-counter kernel (default), the shared-atomic window kernel and the
one-CTA test mode, on shapes that hit every path (row-bin edges inside a warp
iteration, ragged tails, unaligned col_idx, bins_c > 128 fallback, u16 flushes)."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib
from paper_2308_00106_b200.matio import CsrMatrix

pytestmark = pytest.mark.gpu


@pytest.fixture
def hist_mode():
    yield lambda m: _lib.call("sme_hist2d_set_mode", m)
    _lib.call("sme_hist2d_set_mode", 0)
    _lib.call("sme_hist2d_set_variant", 0)


@pytest.mark.parametrize("variant", range(8))
def test_hist2d_lane_kernel_tilings(variant, hist_mode):
    rng = np.random.default_rng(21)
    rows, cols, ptr = _random_csr(rng, 30000, 9000, 400_003, skew=True)
    m = P.CsrMatrix(30000, 9000, ptr, cols, np.ones(cols.size))
    _lib.call("sme_hist2d_set_variant", variant)
    for br, bc in ((128, 128), (3000, 100), (1, 7)):
        got = P.histogram_2d(m, br, bc).counts
        assert np.array_equal(got, O.histogram_2d_counts(rows, cols, 30000, 9000, br, bc)), (variant, br, bc)


def _random_csr(rng, n_rows, n_cols, nnz_target, skew=False):
    if skew:  # a few long rows spanning many row-bin edges' worth of positions
        lens = np.minimum(rng.zipf(1.6, n_rows), n_cols).astype(np.int64)
    else:
        lens = rng.poisson(max(1e-9, nnz_target / n_rows), n_rows).clip(0, n_cols)
    rows = np.repeat(np.arange(n_rows), lens)
    cols = np.concatenate([np.sort(rng.choice(n_cols, int(k), replace=False)) for k in lens]) if lens.sum() else \
        np.zeros(0, dtype=np.int64)
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    return rows, cols.astype(np.int64), ptr


CASES = [  # n_rows, n_cols, nnz, bins_r, bins_c, skew
    (1000, 900, 20_003, 1, 1, False),
    (1000, 900, 20_003, 3, 5, False),
    (5000, 4000, 100_001, 128, 128, False),
    (5000, 4000, 100_001, 7, 31, True),
    (3000, 20000, 60_000, 200, 64, False),
    (3000, 20000, 60_000, 17, 129, False),  # bins_c > 128: window kernel
    (20000, 300, 150_000, 128, 128, True),
    (64, 64, 5, 64, 64, False),
]


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("case", CASES)
def test_hist2d_csr_matches_oracle(case, mode, hist_mode):
    n_rows, n_cols, nnz, br, bc, skew = case
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    rows, cols, ptr = _random_csr(rng, n_rows, n_cols, nnz, skew)
    m = P.CsrMatrix(n_rows, n_cols, ptr, cols, rng.random(cols.size))
    hist_mode(mode)
    got = P.histogram_2d(m, br, bc).counts
    assert np.array_equal(got, O.histogram_2d_counts(rows, cols, n_rows, n_cols, br, bc))


@pytest.mark.parametrize("mode", [0, 2])
def test_hist2d_unaligned_col_idx(mode, hist_mode):
    rng = np.random.default_rng(8)
    rows, cols, ptr = _random_csr(rng, 4000, 5000, 90_001)
    dev = torch.device("cuda")
    big = torch.zeros(cols.size + 1, dtype=torch.int32, device=dev)
    big[1:] = torch.from_numpy(cols.astype(np.int32)).to(dev)
    m = CsrMatrix._from_device(4000, 5000, torch.from_numpy(ptr.astype(np.int32)).to(dev), big[1:],
                               torch.ones(cols.size, dtype=torch.float64, device=dev))
    assert m.d_col_idx.data_ptr() % 16 != 0
    hist_mode(mode)
    got = P.histogram_2d(m, 50, 128).counts
    assert np.array_equal(got, O.histogram_2d_counts(rows, cols, 4000, 5000, 50, 128))


@pytest.mark.parametrize("target", [0, 1])
def test_hist2d_u16_counters_flush_before_overflow(hist_mode, target):
    """40M nonzeros in ONE bin on one CTA: every lane's u16 counter would overflow ~20
    times without the periodic flush.  Bins 0 and 1 share a counter word (low / high
    half), so an overflow of either would show in the other or be lost."""
    dev = torch.device("cuda")
    n_rows, k, n_cols = 40_000, 1000, 128_000  # width 1000: every column lies in bin `target`
    row_ptr = (torch.arange(n_rows + 1, device=dev, dtype=torch.int64) * k).to(torch.int32)
    col = (torch.arange(k, device=dev, dtype=torch.int32) + target * k).repeat(n_rows)
    m = CsrMatrix._from_device(n_rows, n_cols, row_ptr, col, torch.ones(n_rows * k, dtype=torch.float64,
                                                                          device=dev))
    for mode in (2, 0):
        hist_mode(mode)
        got = P.histogram_2d(m, 1, 128).counts
        assert int(got[0, target]) == n_rows * k and int(got.sum()) == n_rows * k
