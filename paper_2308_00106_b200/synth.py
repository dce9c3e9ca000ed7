"""Synthetic matrices of the BASELINE.json configs, generated on the device.

Benchmark / test inputs, not part of the reference path:
  C1  uniform random 10k x 10k, 100k nnz  -> make_random_coo (host numpy,
      the reference test generator's algorithm, tests/conftest.py:10-16)
  C2  5-point Laplacian 2000^2             -> laplacian5(2000)
  C4  50M rows x 20 distinct random cols   -> random_rows(50_000_000, 50_000_000, 20)
  C5  5-point Laplacian 2828^2             -> laplacian5(2828)
The device generators (synth.cu) have bit-identical numpy restatements in
oracle/spmv_entropy_oracle.py (laplacian5, random_rows) used by the tests.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .matio import CooMatrix, CsrMatrix

C4_SEED = 0x5EED_C4


def _vdt(dtype) -> torch.dtype:
    return torch.float32 if dtype in (np.float32, torch.float32, "f32", "float32") else torch.float64


def laplacian5(g: int, dtype=np.float64) -> CsrMatrix:
    """5-point Laplacian on a g x g grid (g*g rows, 5g^2 - 4g nnz), CSR on the device."""
    dev = _cuda.require_cuda()
    n, nnz = g * g, 5 * g * g - 4 * g
    vdt = _vdt(dtype)
    row_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=vdt, device=dev)
    _lib.call("sme_synth_laplacian5", _cuda.sme_dtype(val), g, ptr(row_ptr), ptr(col), ptr(val), stream())
    return CsrMatrix._from_device(n, n, row_ptr, col, val)


def random_rows(n_rows: int, n_cols: int, k: int, seed: int = C4_SEED, dtype=np.float64) -> CsrMatrix:
    """k distinct uniform random columns per row, sorted, values U[-1, 1) (C4's structure)."""
    dev = _cuda.require_cuda()
    vdt = _vdt(dtype)
    nnz = n_rows * k
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=vdt, device=dev)
    if _cuda.wide_row_ptr(nnz):  # int64 row_ptr (nnz >= 2^31 - 1): row r starts at r * k
        row_ptr = torch.arange(n_rows + 1, dtype=torch.int64, device=dev) * k
        _lib.call("sme_synth_random_rows", _cuda.sme_dtype(val), n_rows, n_cols, k, seed, None, ptr(col),
                  ptr(val), stream())
    else:
        row_ptr = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
        _lib.call("sme_synth_random_rows", _cuda.sme_dtype(val), n_rows, n_cols, k, seed, ptr(row_ptr), ptr(col),
                  ptr(val), stream())
    return CsrMatrix._from_device(n_rows, n_cols, row_ptr, col, val)


def random_rows_select(rows: torch.Tensor, n_cols: int, k: int, seed: int = C4_SEED, dtype=np.float64) -> CsrMatrix:
    """Rows `rows` (device int32, any order) of random_rows(., n_cols, k, seed): output
    row i is generator row rows[i].  A row shard of the permuted C4 generates only
    the original rows inverse(p_r)[lo:hi] it owns."""
    dev = _cuda.require_cuda()
    vdt = _vdt(dtype)
    rows = rows.to(dev, torch.int32).contiguous()
    n_sel = rows.numel()
    row_ptr = torch.empty(n_sel + 1, dtype=torch.int32, device=dev)
    col = torch.empty(n_sel * k, dtype=torch.int32, device=dev)
    val = torch.empty(n_sel * k, dtype=vdt, device=dev)
    _lib.call("sme_synth_random_rows_sel", _cuda.sme_dtype(val), n_sel, ptr(rows), n_cols, k, seed, ptr(row_ptr),
              ptr(col), ptr(val), stream())
    return CsrMatrix._from_device(n_sel, n_cols, row_ptr, col, val)


C3_SEED = 0x5EED_C3
RMAT_ABC = (0.57, 0.19, 0.19)


def rmat(scale: int, edge_factor: int = 16, abc=RMAT_ABC, seed: int = C3_SEED, cap: int = 1024,
         dtype=np.float32) -> CsrMatrix:
    """R-MAT graph (C3: scale 24, edge factor 16, (0.57, 0.19, 0.19), f32): edges from
    the device generator, deduplicated and degree-capped to `cap` (the smallest
    columns of a row are kept: "no dense rows") by the CSR builder, values
    U[-1, 1) per (row, slot)."""
    dev = _cuda.require_cuda()
    n, E = 1 << scale, edge_factor << scale
    a, b, c = abc
    vdt = _vdt(dtype)
    row = torch.empty(E, dtype=torch.int32, device=dev)
    col = torch.empty(E, dtype=torch.int32, device=dev)
    _lib.call("sme_synth_rmat_edges", E, scale, a, b, c, seed, ptr(row), ptr(col), stream())
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    row_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ws = _cuda.workspace(_lib.query_size("sme_row_ptr_workspace_size", n))
    _lib.call("sme_coo_row_ptr", n, n, E, ptr(row), ptr(col), None, ptr(row_ptr), ptr(ws), ws.numel(), ptr(flag),
              stream())
    long_t = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call("sme_long_row_nnz", n, ptr(row_ptr), ptr(long_t), stream())
    long_nnz = int(long_t.item())
    zeros = torch.zeros(E, dtype=vdt, device=dev)
    col_s = torch.empty(E, dtype=torch.int32, device=dev)
    val_s = torch.empty(E, dtype=vdt, device=dev)
    ws2 = _cuda.workspace(_lib.query_size("sme_coo_to_csr_workspace_size", n, E, long_nnz))
    _lib.call("sme_coo_to_csr_dedup", _cuda.sme_dtype(zeros), n, n, E, ptr(row), ptr(col), ptr(zeros), ptr(row_ptr),
              ptr(col_s), ptr(val_s), ptr(ws2), ws2.numel(), long_nnz, ptr(flag), stream())
    del ws2, zeros, row, col
    out_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ws3 = _cuda.workspace(_lib.query_size("sme_row_ptr_workspace_size", n))
    _lib.call("sme_csr_compact_row_ptr", n, ptr(row_ptr), ptr(col_s), cap, ptr(out_ptr), ptr(ws3), ws3.numel(),
              stream())
    nnz = int(out_ptr[n].item())
    col_c = torch.empty(nnz, dtype=torch.int32, device=dev)
    val_c = torch.empty(nnz, dtype=vdt, device=dev)
    _lib.call("sme_csr_compact", _cuda.sme_dtype(val_s), n, ptr(row_ptr), ptr(col_s), ptr(val_s), cap, ptr(out_ptr),
              ptr(col_c), ptr(val_c), stream())
    _lib.call("sme_synth_row_values", _cuda.sme_dtype(val_c), n, ptr(out_ptr), seed, ptr(val_c), stream())
    return CsrMatrix._from_device(n, n, out_ptr, col_c, val_c)


def make_random_coo(rng: np.random.Generator, n_rows: int, n_cols: int, density: float) -> CooMatrix:
    """Random COO with `density` fill, values in [-1, 1), shuffled entry order
    (the reference test generator, pkg/tests/conftest.py:10-16; C1 = (default_rng(0), 10000, 10000, 0.001))."""
    total = n_rows * n_cols
    nnz = int(round(density * total))
    cells = rng.choice(total, size=nnz, replace=False)
    values = rng.random(nnz) * 2.0 - 1.0
    return CooMatrix(n_rows, n_cols, cells // n_cols, cells % n_cols, values)
