"""Torch plumbing for the C-ABI: device tensors, the current stream, scratch.

PyTorch provides device memory (its caching allocator), streams and host<->
device copies; every computation on the path is a libsme.so kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

INT32_MAX = 2**31 - 1


def nvtx(name: str):
    """Decorator: an NVTX range around a public API call (visible in nsys / ncu
    --nvtx timelines; a no-op cost of ~1 us otherwise).  Per-launch timing stays
    with CUDA events; this only labels the phases (tracing)."""
    import functools

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **k):
            torch.cuda.nvtx.range_push(f"sme.{name}")
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()

        return inner

    return wrap


_PRELOADED: set[int] = set()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "a CUDA device is required: the max_E SpMV path runs only as sm_100a kernels "
            "(no CPU fallback)"
        )
    _lib.load()
    dev = torch.cuda.current_device()
    if dev not in _PRELOADED:  # once per device: load libsme's kernel modules up front
        _PRELOADED.add(dev)
        torch.zeros(1, device=f"cuda:{dev}")  # the context exists
        # an optimisation only: a module that fails here fails loudly at its first launch
        _lib.load().sme_preload()
    return torch.device("cuda", dev)


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def sme_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return _lib.SME_F64
    if t.dtype == torch.float32:
        return _lib.SME_F32
    if t.dtype == torch.int32:
        return _lib.SME_I32
    raise ValueError(f"unsupported dtype {t.dtype}")


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=require_cuda())


def as_index_tensor(a, what: str, n_max: int | None = None) -> torch.Tensor:
    """1-D int32 device tensor from numpy / list / torch input (values are range-checked
    on the device by the caller; here only representability in int32 is checked)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.int32:
            return a.to(dev).contiguous()
        a64 = a.to(torch.int64)
        if a64.numel() and (int(a64.min()) < -INT32_MAX or int(a64.max()) > INT32_MAX):
            raise ValueError(f"{what} outside int32 range")
        return a64.to(dev, torch.int32).contiguous()
    arr = np.asarray(a, dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError(f"{what} must be a 1-D array")
    if arr.size and (arr.min() < -INT32_MAX or arr.max() > INT32_MAX):
        raise ValueError(f"{what} outside int32 range")
    return torch.from_numpy(arr.astype(np.int32)).to(dev)


# Test hook: give every CSR built from now on an int64 row_ptr, whatever its nnz, so
# the `_i64` entry points are exercised on matrices the oracle can check.
FORCE_WIDE_ROW_PTR = False


def wide_row_ptr(nnz: int) -> bool:
    """int64 row_ptr for nnz >= 2^31 - 1 (int32 offsets below that)."""
    return int(nnz) >= INT32_MAX or FORCE_WIDE_ROW_PTR


def row_ptr_dtype(nnz: int) -> torch.dtype:
    return torch.int64 if wide_row_ptr(nnz) else torch.int32


def as_row_ptr_tensor(a, nnz: int) -> torch.Tensor:
    """1-D device row_ptr: int32 while nnz < 2^31 - 1, int64 above (or when forced)."""
    if not wide_row_ptr(nnz):
        return as_index_tensor(a, "row_ptr")
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(dev, torch.int64).contiguous()
    arr = np.asarray(a, dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError("row_ptr must be a 1-D array")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev)


def as_value_tensor(a, dtype: torch.dtype) -> torch.Tensor:
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(dev, dtype).contiguous()
    arr = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev, dtype)


class DeviceFlags:
    """An int32 validation flag word plus a uint64 'first duplicate' key on the device."""

    def __init__(self):
        dev = require_cuda()
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.dup = torch.full((1,), -1, dtype=torch.int64, device=dev)  # 0xFFFF...FFFF

    @property
    def flag_ptr(self) -> int:
        return self.flag.data_ptr()

    @property
    def dup_ptr(self) -> int:
        return self.dup.data_ptr()

    def read(self) -> tuple[int, int]:
        """Synchronising read: (flag bits, duplicate key as unsigned)."""
        f = int(self.flag.item())
        d = int(self.dup.item()) & 0xFFFFFFFFFFFFFFFF
        return f, d


def to_host(t: torch.Tensor, dtype) -> np.ndarray:
    return t.detach().to("cpu").numpy().astype(dtype, copy=False)
