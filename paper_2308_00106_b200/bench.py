"""The measurement protocol's plugin boundary with GPU kernels registered.

Mirrors the reference `spmv_entropy.bench` boundary (reference
/root/reference/pkg/src/spmv_entropy/bench.py:32-171): `KernelSpec`,
`PermutedOperands`, `gflops`, `time_kernel`, `choose_iterations`,
`derived_seed`, `input_vector` keep their names and meaning, and
`gpu_kernels()` returns KernelSpecs that drop into the reference's own
`run_experiment` next to its `default_kernels`.

The three boundary gotchas of SURVEY.md §8b are handled here:
 (1) `fn` receives a host x on every call -> the matrix's device copy is
     memoised per operands object; x crosses PCIe each call (honest e2e);
 (2) the reference `time_kernel` has no device sync -> every GPU `fn`
     synchronises its stream before returning;
 (3) y goes through np.asarray -> `fn` returns a host float64 array.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from .kernels import spmv_csr, spmv_csr_parallel, spmv_into
from .matio import CooMatrix, CsrMatrix, from_reference

ITERATIONS_MIN = 1000
ITERATIONS_MAX = 5000
CORRECTNESS_RTOL = 1e-12  # bench.py:34 (f64); the north star's f32 bar is 1e-5
CORRECTNESS_RTOL_F32 = 1e-5
PILOT_CALLS = 10
_X_STREAM = 0
_REPEAT_STREAM = 1


@dataclass(frozen=True)
class PermutedOperands:
    """The permuted matrix in both storage formats (bench.py:41-46)."""

    coo: object
    csr: object


@dataclass(frozen=True)
class KernelSpec:
    """A timeable kernel: id, optional worker count, fn(operands, x) -> y (bench.py:49-55)."""

    kernel_id: str
    fn: Callable
    workers: int | None = None


def choose_iterations(estimated_seconds_per_call: float, target_total: float = 2.0) -> int:
    """bench.py:131-135."""
    if estimated_seconds_per_call <= 0:
        raise ValueError("estimated seconds per call must be positive")
    return int(min(ITERATIONS_MAX, max(ITERATIONS_MIN, round(target_total / estimated_seconds_per_call))))


def gflops(nnz: int, seconds_per_call: float) -> float:
    """2 * nnz / s / 1e9 (bench.py:138-144)."""
    if seconds_per_call <= 0:
        raise ValueError("seconds per call must be positive")
    if nnz == 0:
        return 0.0
    return 2 * nnz / seconds_per_call / 1e9


def spmv_bytes(n_rows: int, n_cols: int, nnz: int, value_bytes: int = 8, index_bytes: int = 4) -> int:
    """Algorithmic bytes of one CSR SpMV: values + col_idx once,
    row_ptr once, x read once, y written once."""
    ptr_bytes = 4 if nnz < 2**31 - 1 else 8
    return nnz * (value_bytes + index_bytes) + (n_rows + 1) * ptr_bytes + n_cols * value_bytes + n_rows * value_bytes


def time_kernel(kernel: Callable, m, x, iterations: int):
    """Mean wall seconds per call over `iterations` calls plus the last output
    (bench.py:147-158); the device is synchronised before the clock stops."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    t0 = time.perf_counter()
    for _ in range(iterations):
        y = kernel(m, x)
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iterations, y


def derived_seed(master_seed: int, repeat: int) -> int:
    """bench.py:161-165."""
    return int(np.random.SeedSequence(master_seed, spawn_key=(_REPEAT_STREAM, repeat)).generate_state(1, np.uint64)[0])


def input_vector(master_seed: int, n: int) -> np.ndarray:
    """Deterministic x in [0, 1) (bench.py:168-171) — host numpy, bit-identical."""
    seq = np.random.SeedSequence(master_seed, spawn_key=(_X_STREAM,))
    return np.random.Generator(np.random.PCG64(seq)).random(n)


# ---------------------------------------------------------------------------
# GPU KernelSpecs
# ---------------------------------------------------------------------------
# device copies of reference matrices, keyed by object identity: the reference's
# CsrMatrix defines __eq__ without __hash__ (unhashable), so the entry is dropped by a
# weakref finalizer when the reference object dies
_device_csr: dict[int, CsrMatrix] = {}


def device_csr(ops) -> CsrMatrix:
    """The operands' CSR on the device, uploaded once per reference CsrMatrix object."""
    csr = ops.csr if isinstance(ops, PermutedOperands) or hasattr(ops, "csr") else ops
    if isinstance(csr, CsrMatrix):
        return csr
    if isinstance(csr, CooMatrix):
        from .matio import coo_to_csr

        return coo_to_csr(csr)
    key = id(csr)
    d = _device_csr.get(key)
    if d is None:
        d = _device_csr[key] = from_reference(csr)
        weakref.finalize(csr, _device_csr.pop, key, None)
    return d


def _host_call(kernel: str) -> Callable:
    def fn(ops, x):
        return spmv_csr(device_csr(ops), x, kernel)  # H2D x, kernel, D2H y (synchronous)

    return fn


def _parallel_call(workers: int) -> Callable:
    def fn(ops, x):
        return spmv_csr_parallel(device_csr(ops), x, workers)

    return fn


class _ResidentX:
    """Memoises the device copy of x by object identity (gotcha 1 for the resident kernel)."""

    def __init__(self):
        self._key = None
        self._dev: torch.Tensor | None = None

    def get(self, x, dtype, device) -> torch.Tensor:
        if self._key is not x:
            self._dev = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(device, dtype)
            self._key = x
        return self._dev


def _resident_call(kernel: str) -> Callable:
    cache = _ResidentX()

    def fn(ops, x):
        m = device_csr(ops)
        xd = cache.get(x, m.dtype, m.d_row_ptr.device)
        y = torch.empty(m.n_rows, dtype=m.dtype, device=m.d_row_ptr.device)
        spmv_into(m, xd, y, kernel)
        torch.cuda.current_stream().synchronize()
        return _LazyHost(y)

    return fn


class _LazyHost:
    """A device result that becomes a host float64 array only when numpy asks (gotcha 3)."""

    def __init__(self, t: torch.Tensor):
        self._t = t

    def __array__(self, dtype=None, copy=None):
        a = self._t.to("cpu").numpy().astype(np.float64, copy=False)
        return a if dtype is None else a.astype(dtype, copy=False)

    @property
    def shape(self):
        return tuple(self._t.shape)


def gpu_kernels(max_workers: int = 1) -> list[KernelSpec]:
    """GPU KernelSpecs for the reference protocol (ids recognised by the report as raw ids)."""
    specs = [
        # "auto": the kernel bench.py measures (seg column panels for large permuted
        # matrices, CSR-vector for banded ones; kernels.auto_kernel)
        KernelSpec("gpu_csr_auto", _host_call("auto")),
        KernelSpec("gpu_csr_auto_resident", _resident_call("auto")),
        KernelSpec("gpu_csr_vector", _host_call("vector")),
        KernelSpec("gpu_csr_merge", _host_call("merge")),
        KernelSpec("gpu_csr_merge_resident", _resident_call("merge")),
        KernelSpec("gpu_csr_vector_resident", _resident_call("vector")),
    ]
    for w in range(2, max_workers + 1):
        specs.append(KernelSpec("gpu_par", _parallel_call(w), workers=w))
    return specs


KERNEL_LABELS = {
    "gpu_csr_auto": "GPU AUTO",
    "gpu_csr_auto_resident": "GPU AUTO-RES",
    "gpu_csr_vector": "GPU CSR",
    "gpu_csr_merge": "GPU CSR-MRG",
    "gpu_csr_merge_resident": "GPU MRG-RES",
    "gpu_csr_vector_resident": "GPU CSR-RES",
    "gpu_par": "GPU PAR",
}
