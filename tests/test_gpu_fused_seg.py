"""K4 with the seg layout built by the same row sort (sme_permute_csr_seg).

The fused build must give the permuted CSR bit for bit (permute_csr's contract,
permute.py:98-102 + matio.py:281-294) AND the same segmented-chunk layout, word for word,
as SegLayout on that CSR (the separate count + fill of spmv_seg.cu), for every panel
count, empty rows, f64 / f32, the column pre-map and int64 row_ptr; rows longer than 32
fall back to the plain K4.
"""

import contextlib

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _cuda, synth
from paper_2308_00106_b200 import permute as PM
from paper_2308_00106_b200.seg import SegLayout

pytestmark = pytest.mark.gpu


def short_rows_csr(seed, n_rows=3000, n_cols=9000, max_len=32, dtype=np.float64):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, n_rows)
    lens[rng.random(n_rows) < 0.1] = 0  # empty rows: explicit zeros in panel 0 / even rows
    ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, int(L), replace=False)) for L in lens if L])
    val = (rng.random(col.size) * 2 - 1).astype(dtype)
    return ptr, col, val, n_cols


@contextlib.contextmanager
def fused(panels):
    old = PM._fused_seg_panels
    PM._fused_seg_panels = (lambda m: panels) if panels else (lambda m: 0)
    try:
        yield
    finally:
        PM._fused_seg_panels = old


def same_layout(a: SegLayout, b: SegLayout):
    assert np.array_equal(a.entries, b.entries) and np.array_equal(a.offsets, b.offsets)
    assert torch.equal(a.pk, b.pk), "pk words differ"
    assert torch.equal(a.val.view(torch.uint8), b.val.view(torch.uint8)), "values differ"
    assert torch.equal(a.hdr, b.hdr) and torch.equal(a.plans, b.plans)


def build_both(A, p_r, p_c, panels):
    with fused(panels):
        Bf = P.permute_csr(A, p_r, p_c)
    with fused(0):
        Bp = P.permute_csr(A, p_r, p_c)
    return Bf, Bp


@pytest.mark.parametrize("panels", [1, 3, 8, 32])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fused_layout_equals_separate_build(panels, dtype):
    ptr, col, val, n = short_rows_csr(panels, dtype=dtype)
    A = P.CsrMatrix(len(ptr) - 1, n, ptr, col, val, dtype=dtype)
    p_r, p_c = P.random_permutation(A.n_rows, 5), P.random_permutation(n, 6)
    Bf, Bp = build_both(A, p_r, p_c, panels)
    assert Bf == Bp
    key = ("seg", panels, False)
    assert key in Bf._cache and key not in Bp._cache
    same_layout(Bf._cache[key], SegLayout(Bp, panels))
    # and it computes y = B x
    Bf._cache["seg_panels"] = panels
    x = O.input_vector(2, n).astype(dtype)
    y = np.asarray(P.spmv_csr(Bf, x, "seg"), dtype=np.float64)
    xp = x.astype(np.float64)
    ref = O.spmv_csr(Bp.row_ptr, Bp.col_idx, Bp.values, xp)
    assert O.relative_error(y, ref) <= (1e-12 if dtype == np.float64 else 1e-5)


def test_fused_with_column_premap(monkeypatch):
    monkeypatch.setattr(PM, "_premap_slices", lambda m: 4)
    ptr, col, val, n = short_rows_csr(11)
    A = P.CsrMatrix(len(ptr) - 1, n, ptr, col, val)
    p_r, p_c = P.random_permutation(A.n_rows, 1), P.random_permutation(n, 2)
    Bf, Bp = build_both(A, p_r, p_c, 5)
    assert Bf == Bp
    same_layout(Bf._cache[("seg", 5, False)], SegLayout(Bp, 5))
    monkeypatch.setattr(PM, "PREMAP_FUSE_LAST", True)  # the sort maps the last slice itself
    Bf2, _ = build_both(A, p_r, p_c, 5)
    assert Bf2 == Bp
    same_layout(Bf2._cache[("seg", 5, False)], SegLayout(Bp, 5))


def test_fused_identity_rows_and_columns():
    ptr, col, val, n = short_rows_csr(12)
    A = P.CsrMatrix(len(ptr) - 1, n, ptr, col, val)
    Bf, Bp = build_both(A, None, None, 4)
    assert Bf == Bp == A
    same_layout(Bf._cache[("seg", 4, False)], SegLayout(Bp, 4))


def test_rows_longer_than_32_fall_back():
    ptr, col, val, n = short_rows_csr(13, max_len=40)
    A = P.CsrMatrix(len(ptr) - 1, n, ptr, col, val)
    p_r, p_c = P.random_permutation(A.n_rows, 3), P.random_permutation(n, 4)
    Bf, Bp = build_both(A, p_r, p_c, 4)
    assert Bf == Bp
    assert ("seg", 4, False) not in Bf._cache  # the plain K4 ran


def test_fused_wide_row_ptr():
    ptr, col, val, n = short_rows_csr(14)
    old = _cuda.FORCE_WIDE_ROW_PTR
    _cuda.FORCE_WIDE_ROW_PTR = True
    try:
        A = P.CsrMatrix(len(ptr) - 1, n, ptr, col, val)
        p_r, p_c = P.random_permutation(A.n_rows, 7), P.random_permutation(n, 8)
        Bf, Bp = build_both(A, p_r, p_c, 6)
    finally:
        _cuda.FORCE_WIDE_ROW_PTR = old
    assert Bf.wide and Bf == Bp
    same_layout(Bf._cache[("seg", 6, False)], SegLayout(Bp, 6))


def test_fused_triggers_on_large_x():
    """No override: a 12M x 12M random matrix (x = 96 MB > 60 % of L2, 20-entry rows) gets
    its layout from K4, equal to the one built on first use."""
    n = 12_000_000
    A = synth.random_rows(n, n, 20)
    p_r, p_c = P.random_permutation(n, 21), P.random_permutation(n, 22)
    assert PM._fused_seg_panels(A) >= 2
    B = P.permute_csr(A, p_r, p_c)
    keys = [k for k in B._cache if isinstance(k, tuple) and k[0] == "seg"]
    assert len(keys) == 1
    with fused(0):
        Bp = P.permute_csr(A, p_r, p_c)
    assert B == Bp
    same_layout(B._cache[keys[0]], SegLayout(Bp, keys[0][1]))
