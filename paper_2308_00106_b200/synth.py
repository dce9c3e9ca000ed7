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
    row_ptr = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=vdt, device=dev)
    _lib.call("sme_synth_random_rows", _cuda.sme_dtype(val), n_rows, n_cols, k, seed, ptr(row_ptr), ptr(col),
              ptr(val), stream())
    return CsrMatrix._from_device(n_rows, n_cols, row_ptr, col, val)


def make_random_coo(rng: np.random.Generator, n_rows: int, n_cols: int, density: float) -> CooMatrix:
    """Random COO with `density` fill, values in [-1, 1), shuffled entry order
    (the reference test generator, pkg/tests/conftest.py:10-16; C1 = (default_rng(0), 10000, 10000, 0.001))."""
    total = n_rows * n_cols
    nnz = int(round(density * total))
    cells = rng.choice(total, size=nnz, replace=False)
    values = rng.random(nnz) * 2.0 - 1.0
    return CooMatrix(n_rows, n_cols, cells // n_cols, cells % n_cols, values)
