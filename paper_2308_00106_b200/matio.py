"""Device-resident COO / CSR storage and the COO<->CSR conversions.

Drop-in for the storage half of `spmv_entropy.matio` (reference
/root/reference/pkg/src/spmv_entropy/matio.py): same class names, constructor
arguments, validation rules and error messages, but the arrays live in HBM as
int32 indices and f64 (default, like the reference) or f32 values.  row_ptr is
int32 while nnz < 2^31 - 1 and int64 above (the reference's int64 everywhere,
matio.py:97-99; those CSRs go through the `_i64` entry points of include/sme.h).  The
reference attribute names (`row_idx`, `col_idx`, `values`, `row_ptr`) return
host numpy copies widened to int64 / float64 (made lazily, cached), so code and
tests written against the reference keep working; the device tensors are the
`d_*` attributes.

Validation runs on the GPU:
  * CooMatrix.__post_init__ (matio.py:41-64): range check + duplicate check.
    The reference sorts with lexsort to find duplicates; here the duplicate
    check is a by-product of building the CSR (counting sort + segmented
    column sort, csr_build.cu), which is cached so that coo_to_csr() is free.
  * CsrMatrix.__post_init__ (matio.py:96-122): k_csr_validate.
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import DeviceFlags, ptr, stream


def _value_dtype(values, dtype) -> torch.dtype:
    if dtype is not None:
        d = np.dtype(dtype) if not isinstance(dtype, torch.dtype) else dtype
        if d in (np.float32, torch.float32):
            return torch.float32
        if d in (np.float64, torch.float64):
            return torch.float64
        raise ValueError(f"unsupported value dtype {dtype}")
    if isinstance(values, torch.Tensor) and values.dtype == torch.float32:
        return torch.float32
    return torch.float64


def _check_dims(n_rows: int, n_cols: int) -> None:
    if n_rows < 0 or n_cols < 0:
        raise ValueError("matrix dimensions must be non-negative")
    if n_rows >= _cuda.INT32_MAX or n_cols >= _cuda.INT32_MAX:
        raise ValueError("matrix dimensions exceed the int32 index range of the GPU layout")


def _numel(a) -> int:
    return int(a.numel()) if isinstance(a, torch.Tensor) else int(np.asarray(a).size)


def _ndim(a) -> int:
    return int(a.dim()) if isinstance(a, torch.Tensor) else int(np.asarray(a).ndim)


class CsrMatrix:
    """Compressed sparse row matrix in HBM (reference: matio.py:82-137).

    row_ptr has n_rows + 1 entries; columns are strictly increasing within each
    row.  Immutable by convention, like the reference.
    """

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col_idx, values, *, dtype=None, _trusted: bool = False):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        _check_dims(self.n_rows, self.n_cols)
        if not _trusted:
            if _ndim(row_ptr) != 1 or _numel(row_ptr) != self.n_rows + 1:
                raise ValueError("row_ptr must have n_rows + 1 entries")
            if _numel(col_idx) != _numel(values):
                raise ValueError("col_idx and values must have identical length")
        vdt = _value_dtype(values, dtype)
        self.d_row_ptr = _cuda.as_row_ptr_tensor(row_ptr, _numel(values))
        self.d_col_idx = _cuda.as_index_tensor(col_idx, "col_idx")
        self.d_values = _cuda.as_value_tensor(values, vdt)
        self._host: dict[str, np.ndarray] = {}
        self._cache: dict = {}
        if not _trusted:
            self._validate()

    # ---- construction helpers ------------------------------------------
    @classmethod
    def _from_device(cls, n_rows, n_cols, d_row_ptr, d_col_idx, d_values) -> "CsrMatrix":
        m = cls.__new__(cls)
        m.n_rows, m.n_cols = int(n_rows), int(n_cols)
        m.d_row_ptr, m.d_col_idx, m.d_values = d_row_ptr, d_col_idx, d_values
        m._host, m._cache = {}, {}
        return m

    def _validate(self) -> None:
        fl = DeviceFlags()
        _lib.call_rp("sme_csr_validate", self.d_row_ptr, self.n_rows, self.n_cols, self.nnz, ptr(self.d_row_ptr),
                     ptr(self.d_col_idx), fl.flag_ptr, stream())
        bits, _ = fl.read()
        if bits & _lib.FLAG_ROWPTR:
            first, last = int(self.d_row_ptr[0]), int(self.d_row_ptr[-1])
            if first != 0 or last != self.nnz:
                raise ValueError("row_ptr must start at 0 and end at nnz")
            raise ValueError("row_ptr must be non-decreasing")
        if bits & _lib.FLAG_RANGE:
            raise ValueError("column index outside [0, n_cols)")
        if bits & _lib.FLAG_UNSORTED:
            raise ValueError("columns must be strictly increasing within each row")

    # ---- reference-compatible views ---------------------------------------
    @property
    def nnz(self) -> int:
        return int(self.d_values.numel())

    @property
    def dtype(self) -> torch.dtype:
        return self.d_values.dtype

    @property
    def wide(self) -> bool:
        """int64 row_ptr (nnz >= 2^31 - 1, or forced by _cuda.FORCE_WIDE_ROW_PTR)."""
        return self.d_row_ptr.dtype == torch.int64

    def _h(self, key: str, t: torch.Tensor, dt) -> np.ndarray:
        if key not in self._host:
            arr = _cuda.to_host(t, dt)
            arr.flags.writeable = False
            self._host[key] = arr
        return self._host[key]

    @property
    def row_ptr(self) -> np.ndarray:
        return self._h("row_ptr", self.d_row_ptr, np.int64)

    @property
    def col_idx(self) -> np.ndarray:
        return self._h("col_idx", self.d_col_idx, np.int64)

    @property
    def values(self) -> np.ndarray:
        return self._h("values", self.d_values, np.float64)

    def __eq__(self, other) -> bool:
        if not isinstance(other, CsrMatrix):
            return NotImplemented
        return (
            self.n_rows == other.n_rows
            and self.n_cols == other.n_cols
            and self.dtype == other.dtype
            and torch.equal(self.d_row_ptr, other.d_row_ptr)
            and torch.equal(self.d_col_idx, other.d_col_idx)
            and torch.equal(self.d_values, other.d_values)
        )

    __hash__ = object.__hash__

    def __repr__(self) -> str:
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, {self.dtype}, device)"

    def long_row_nnz(self) -> int:
        """Sum of lengths of rows longer than SME_SORT_SMEM_MAX (scratch sizing)."""
        if "long_nnz" not in self._cache:
            out = torch.zeros(1, dtype=torch.int64, device=self.d_row_ptr.device)
            _lib.call_rp("sme_long_row_nnz", self.d_row_ptr, self.n_rows, ptr(self.d_row_ptr), ptr(out), stream())
            self._cache["long_nnz"] = int(out.item())
        return self._cache["long_nnz"]


class CooMatrix:
    """Coordinate-list sparse matrix in HBM (reference: matio.py:26-79).

    Entries may be stored in any order but (row, col) pairs must be unique;
    duplicates are rejected at construction (on the GPU).
    """

    def __init__(self, n_rows: int, n_cols: int, row_idx, col_idx, values, *, dtype=None, _trusted: bool = False):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        _check_dims(self.n_rows, self.n_cols)
        if not _trusted:
            if not (_ndim(row_idx) == _ndim(col_idx) == _ndim(values) == 1):
                raise ValueError("row_idx, col_idx, values must be 1-D arrays")
            if not (_numel(row_idx) == _numel(col_idx) == _numel(values)):
                raise ValueError("row_idx, col_idx, values must have identical length")
        vdt = _value_dtype(values, dtype)
        self.d_row_idx = _cuda.as_index_tensor(row_idx, "row index")
        self.d_col_idx = _cuda.as_index_tensor(col_idx, "column index")
        self.d_values = _cuda.as_value_tensor(values, vdt)
        self._host: dict[str, np.ndarray] = {}
        self._cache: dict = {}  # per-matrix plans (kernels.coo_entry_order)
        self._csr: CsrMatrix | None = None
        self._csr_thunk: Callable[[], CsrMatrix] | None = None
        if not _trusted:
            self._csr = _coo_build_csr(self, None, None, check=True)

    @classmethod
    def _from_device(cls, n_rows, n_cols, d_row, d_col, d_val, csr_thunk=None, csr=None) -> "CooMatrix":
        m = cls.__new__(cls)
        m.n_rows, m.n_cols = int(n_rows), int(n_cols)
        m.d_row_idx, m.d_col_idx, m.d_values = d_row, d_col, d_val
        m._host, m._csr, m._csr_thunk = {}, csr, csr_thunk
        m._cache = {}
        return m

    @property
    def nnz(self) -> int:
        return int(self.d_values.numel())

    @property
    def dtype(self) -> torch.dtype:
        return self.d_values.dtype

    def _h(self, key: str, t: torch.Tensor, dt) -> np.ndarray:
        if key not in self._host:
            arr = _cuda.to_host(t, dt)
            arr.flags.writeable = False
            self._host[key] = arr
        return self._host[key]

    @property
    def row_idx(self) -> np.ndarray:
        return self._h("row_idx", self.d_row_idx, np.int64)

    @property
    def col_idx(self) -> np.ndarray:
        return self._h("col_idx", self.d_col_idx, np.int64)

    @property
    def values(self) -> np.ndarray:
        return self._h("values", self.d_values, np.float64)

    def __eq__(self, other) -> bool:
        if not isinstance(other, CooMatrix):
            return NotImplemented
        return (
            self.n_rows == other.n_rows
            and self.n_cols == other.n_cols
            and self.dtype == other.dtype
            and torch.equal(self.d_row_idx, other.d_row_idx)
            and torch.equal(self.d_col_idx, other.d_col_idx)
            and torch.equal(self.d_values, other.d_values)
        )

    __hash__ = object.__hash__

    def __repr__(self) -> str:
        return f"CooMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, {self.dtype}, device)"


def _coo_build_csr(m: CooMatrix, row_map, col_map, check: bool, row_ptr_dtype=None) -> CsrMatrix:
    """GPU counting sort + segmented column sort (csr_build.cu).  row_ptr is int32 while
    nnz < 2^31 - 1, else int64 (row_ptr_dtype overrides: internal plans)."""
    dev = _cuda.require_cuda()
    n_rows, n_cols, nnz = m.n_rows, m.n_cols, m.nnz
    fl = DeviceFlags()
    row_ptr = torch.empty(n_rows + 1, dtype=row_ptr_dtype or _cuda.row_ptr_dtype(nnz), device=dev)
    ws1 = _cuda.workspace(_lib.query_size("sme_row_ptr_workspace_size", n_rows))
    _lib.call_rp("sme_coo_row_ptr", row_ptr, n_rows, n_cols, nnz, ptr(m.d_row_idx), ptr(m.d_col_idx), ptr(row_map),
                 ptr(row_ptr), ptr(ws1), ws1.numel(), fl.flag_ptr, stream())
    if check:
        bits, _ = fl.read()
        if bits & _lib.FLAG_RANGE:
            _raise_range(m)
    long_t = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call_rp("sme_long_row_nnz", row_ptr, n_rows, ptr(row_ptr), ptr(long_t), stream())
    long_nnz = int(long_t.item())
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=m.dtype, device=dev)
    ws2 = _cuda.workspace(_lib.query_size("sme_coo_to_csr_workspace_size", n_rows, nnz, long_nnz))
    _lib.call_rp("sme_coo_to_csr", row_ptr, _cuda.sme_dtype(m.d_values), n_rows, n_cols, nnz, ptr(m.d_row_idx),
                 ptr(m.d_col_idx), ptr(m.d_values), ptr(row_map), ptr(col_map), ptr(row_ptr), ptr(col), ptr(val),
                 ptr(ws2), ws2.numel(), long_nnz, fl.flag_ptr, fl.dup_ptr, stream())
    if check:
        bits, dup = fl.read()
        if bits & _lib.FLAG_DUPLICATE:
            raise ValueError(f"duplicate entry at ({dup >> 32}, {dup & 0xFFFFFFFF})")
    csr = CsrMatrix._from_device(n_rows, n_cols, row_ptr, col, val)
    csr._cache["long_nnz"] = long_nnz
    return csr


def _raise_range(m: CooMatrix) -> None:
    # error path only: find which index array is out of range for the message
    r, c = m.d_row_idx, m.d_col_idx
    if bool(((r < 0) | (r >= m.n_rows)).any()):
        raise ValueError("row index outside [0, n_rows)")
    if bool(((c < 0) | (c >= m.n_cols)).any()):
        raise ValueError("column index outside [0, n_cols)")
    raise ValueError("index outside the matrix")


@_cuda.nvtx("coo_to_csr")
def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Convert COO to CSR; values reordered (row-major, columns ascending) but
    otherwise bit-identical.  Duplicates are an error (reference: matio.py:281-294)."""
    if not isinstance(m, CooMatrix):
        raise TypeError("coo_to_csr expects a CooMatrix")
    if m._csr is None:
        m._csr = m._csr_thunk() if m._csr_thunk is not None else _coo_build_csr(m, None, None, check=True)
        m._csr_thunk = None
    return m._csr


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    """Expand CSR back to COO; coo_to_csr(csr_to_coo(m)) reproduces m exactly (matio.py:297-300)."""
    row = torch.empty(m.nnz, dtype=torch.int32, device=m.d_row_ptr.device)
    _lib.call_rp("sme_csr_expand_rows", m.d_row_ptr, m.n_rows, ptr(m.d_row_ptr), ptr(row), stream())
    return CooMatrix._from_device(m.n_rows, m.n_cols, row, m.d_col_idx.clone(), m.d_values.clone(), csr=m)


def from_reference(m):
    """Upload a reference `spmv_entropy` CooMatrix / CsrMatrix (duck-typed) to the device."""
    if hasattr(m, "row_ptr"):
        return CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)
    return CooMatrix(m.n_rows, m.n_cols, m.row_idx, m.col_idx, m.values)
