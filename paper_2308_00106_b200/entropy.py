"""Binned nonzero histograms and their Shannon entropy, on the GPU.

Drop-in for the hot half of `spmv_entropy.entropy` (reference
/root/reference/pkg/src/spmv_entropy/entropy.py:18-119): same bin rule
(width = n // bins, the last bin absorbs the remainder), same int64 counts,
same entropy definition.  Counts come from hist.cu (bit-exact: they are
integers); the entropy is one deterministic block reduction (k_entropy),
equal to the reference within 1e-12 relative (log2 rounding differs in the
last ulp; exact for the reference's exact cases: uniform, delta, [1,1,2]).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .matio import CooMatrix, CsrMatrix

DEFAULT_BINS_1D = 512
DEFAULT_BINS_2D = 128
DEFAULT_LEVELS = (2, 4, 8)


class BinnedHistogram:
    """Nonzero counts over equal-width bins; 1-D (counts[B]) or 2-D (counts[Br, Bc]) (entropy.py:23-55).

    `counts` is a host int64 array (lazy copy of `d_counts` when the histogram
    was produced on the GPU); `edges[d][b]` is the first index of bin b.
    """

    def __init__(self, counts, edges):
        if isinstance(counts, torch.Tensor):
            self.d_counts = counts.to(torch.int64)
            self._counts = None
            shape = tuple(counts.shape)
        else:
            arr = np.asarray(counts, dtype=np.int64)
            self._counts = arr
            self.d_counts = None
            shape = arr.shape
        self.edges = tuple(np.asarray(e, dtype=np.int64) for e in edges)
        if len(shape) not in (1, 2):
            raise ValueError("counts must be 1-D or 2-D")
        if len(self.edges) != len(shape):
            raise ValueError("one edge array required per counts axis")
        for axis, e in enumerate(self.edges):
            if e.size != shape[axis] + 1:
                raise ValueError("edges must have bin-count + 1 offsets")
        if self._counts is not None and self._counts.size and self._counts.min() < 0:
            raise ValueError("counts must be non-negative")

    @property
    def counts(self) -> np.ndarray:
        if self._counts is None:
            self._counts = _cuda.to_host(self.d_counts, np.int64)
        return self._counts

    def device_counts(self) -> torch.Tensor:
        if self.d_counts is None:
            dev = _cuda.require_cuda()
            self.d_counts = torch.from_numpy(np.ascontiguousarray(self._counts)).to(dev)
        return self.d_counts

    @property
    def total(self) -> int:
        return int(self.counts.sum())

    @property
    def n_bins(self) -> int:
        return int(self.counts.size)


def _bin_edges(n: int, bins: int) -> np.ndarray:
    width = n // bins
    edges = np.arange(bins + 1, dtype=np.int64) * width
    edges[-1] = n
    return edges


def _check_bins(bins: int, n: int, what: str) -> None:
    if bins < 1:
        raise ValueError(f"{what} bin count must be >= 1")
    if bins > n:
        raise ValueError(f"{what} bin count {bins} exceeds dimension {n}")


def _zeros(n: int) -> torch.Tensor:
    return torch.zeros(n, dtype=torch.int64, device=_cuda.require_cuda())


@_cuda.nvtx("histogram_2d")
def histogram_2d(m, bins_r: int, bins_c: int) -> BinnedHistogram:
    """Count nonzeros on a bins_r x bins_c grid (entropy.py:91-101).

    CsrMatrix input uses the row-bin-segmented streaming kernel (reads col_idx
    only); CooMatrix input uses its cached CSR when present, else the COO
    kernel over the triplets.
    """
    _check_bins(bins_r, m.n_rows, "row")
    _check_bins(bins_c, m.n_cols, "column")
    counts = _zeros(bins_r * bins_c)
    csr = m if isinstance(m, CsrMatrix) else getattr(m, "_csr", None)
    if csr is not None:
        _lib.call_rp("sme_hist2d_csr", csr.d_row_ptr, csr.n_rows, csr.n_cols, csr.nnz, ptr(csr.d_row_ptr),
                     ptr(csr.d_col_idx), bins_r, bins_c, ptr(counts), stream())
    elif isinstance(m, CooMatrix):
        _lib.call("sme_hist2d_coo", m.n_rows, m.n_cols, m.nnz, ptr(m.d_row_idx), ptr(m.d_col_idx), bins_r,
                  bins_c, ptr(counts), stream())
    else:
        raise TypeError("histogram_2d expects a CooMatrix or CsrMatrix of this package")
    return BinnedHistogram(counts.view(bins_r, bins_c), (_bin_edges(m.n_rows, bins_r), _bin_edges(m.n_cols, bins_c)))


def row_histogram(m, bins: int) -> BinnedHistogram:
    """Count nonzeros per row bin (entropy.py:77-81): differences of row_ptr at the bin edges."""
    _check_bins(bins, m.n_rows, "row")
    csr = m if isinstance(m, CsrMatrix) else _csr_of(m)
    counts = _zeros(bins)
    _lib.call_rp("sme_row_hist_csr", csr.d_row_ptr, csr.n_rows, ptr(csr.d_row_ptr), bins, ptr(counts), stream())
    return BinnedHistogram(counts, (_bin_edges(m.n_rows, bins),))


def col_histogram(m, bins: int) -> BinnedHistogram:
    """Count nonzeros per column bin (entropy.py:84-88): the 2-D kernel with one row bin."""
    _check_bins(bins, m.n_cols, "column")
    if m.n_rows == 0 or m.nnz == 0:  # the reference checks column bins only (a 0-row matrix is legal)
        return BinnedHistogram(_zeros(bins), (_bin_edges(m.n_cols, bins),))
    h = histogram_2d(m, 1, bins)
    return BinnedHistogram(h.device_counts().view(bins), (_bin_edges(m.n_cols, bins),))


def _csr_of(m: CooMatrix) -> CsrMatrix:
    from .matio import coo_to_csr

    return coo_to_csr(m)


@_cuda.nvtx("shannon_entropy")
def shannon_entropy(h: BinnedHistogram, base: float = 2.0) -> float:
    """-sum p_i log(p_i) over nonzero bins, p_i = count_i / total (entropy.py:104-119).

    Any base the reference accepts works (base 2: log2; otherwise ln / ln(base), so a
    base in (0, 1) gives a negative value); the reference's errors are kept, in its
    order: an empty histogram is a ValueError, then base 1 divides by ln 1 = 0
    (ZeroDivisionError) and base <= 0 fails math.log (ValueError)."""
    base = float(base)
    valid = base > 0.0 and base != 1.0
    d = h.device_counts().reshape(-1).contiguous()
    out = torch.empty(1, dtype=torch.float64, device=d.device)
    total = torch.empty(1, dtype=torch.int64, device=d.device)
    _lib.call("sme_entropy", d.numel(), ptr(d), base if valid else 2.0, ptr(out), ptr(total), stream())
    if int(total.item()) == 0:
        raise ValueError("histogram is empty (total = 0)")
    if base == 1.0:
        raise ZeroDivisionError("float division by zero")
    if base <= 0.0:
        raise ValueError("math domain error")
    return float(out.item())
