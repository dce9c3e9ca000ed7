"""SpMV on the GPU: CSR (CSR-vector and merge-path), row-partitioned CSR, COO.

Drop-in for `spmv_entropy.kernels` (reference
/root/reference/pkg/src/spmv_entropy/kernels.py).  All kernels are pure and
deterministic (the opt-in COO kernel="atomic" excepted).

Input/output convention: a host array x gives a host numpy float64 y (H2D of
x, kernel, D2H of y — the reference-facing call); a CUDA tensor x gives a CUDA
tensor y of the matrix's dtype with nothing crossing PCIe (the resident path
used by repeated SpMV).

Kernels (spmv.cu):
  "vector"  CSR-vector, `lanes` threads per row (default: next power of two of
            the mean row length, at most 32).  Row-partition invariant, so
            spmv_csr_parallel is bitwise equal to spmv_csr, as in the reference.
  "merge"   merge-path tiles balanced over rows + nonzeros; the load-balanced
            kernel for ragged / power-law rows.  Per-matrix plan cached.
  "exact"   numpy add.reduceat association restated on the GPU (f64): bitwise
            equal to the reference spmv_csr; a parity tool, not a fast path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _cuda, _lib, hostio
from ._cuda import ptr, stream
from .matio import CooMatrix, CsrMatrix

KERNELS = ("auto", "seg", "stream", "panel", "vector", "merge", "exact")
# kernels with int64 row_ptr twins (CSRs of nnz >= 2^31 - 1; auto_kernel only picks these)
WIDE_KERNELS = ("seg", "vector")


@dataclass(frozen=True, eq=False)
class RowPartition:
    """Even split of [0, n_rows) into `workers` contiguous ranges (kernels.py:20-35)."""

    boundaries: np.ndarray
    workers: int

    def __post_init__(self):
        b = np.asarray(self.boundaries, dtype=np.int64)
        object.__setattr__(self, "boundaries", b)
        if b.size != self.workers + 1 or b[0] != 0 or np.any(np.diff(b) < 0):
            raise ValueError("boundaries must be a non-decreasing array of workers + 1 offsets starting at 0")


def make_row_partition(n_rows: int, workers: int) -> RowPartition:
    """Split rows evenly: the first n_rows % workers parts get one extra row (kernels.py:38-49)."""
    if workers < 1:
        raise ValueError("worker count must be >= 1")
    if workers > n_rows:
        raise ValueError(f"worker count {workers} exceeds row count {n_rows}")
    base, extra = divmod(n_rows, workers)
    sizes = np.full(workers, base, dtype=np.int64)
    sizes[:extra] += 1
    boundaries = np.zeros(workers + 1, dtype=np.int64)
    np.cumsum(sizes, out=boundaries[1:])
    return RowPartition(boundaries, workers)


def default_lanes(m: CsrMatrix) -> int:
    """Threads per row of the CSR-vector kernel: the largest power of two with
    lanes * 5 <= mean_row_length (each lane handles >= ~2.5 elements), in [1, 32].
    Measured on B200 (tools/vector_lanes_ab.py): C2 (4.998 nnz/row -> 1 lane) permuted
    0.1017 ms at 1 lane, 0.1004 at 2, 0.110 at 4, 0.151 at 8; unpermuted 0.0592 at 1,
    0.0615 at 2 (C5 unpermuted: 0.123 / 0.125) — 1 and 2 lanes are within 1-4 %."""
    if "lanes" not in m._cache:
        mean = m.nnz / max(1, m.n_rows)
        lanes = 1
        while lanes < 32 and lanes * 2 * 2.5 <= mean:
            lanes <<= 1
        m._cache["lanes"] = lanes
    return m._cache["lanes"]


def auto_kernel(m: CsrMatrix) -> str:
    """Kernel policy (measured on B200, profiles/round1/kernel_compare.txt):
    * 'seg' (column panels in the segmented-chunk layout, seg.py) when x exceeds
      60 % of L2 — random gathers would miss to DRAM (62 G gathers/s at 400 MB vs
      287 G/s L2-resident, tools/gather_roofline.py); C4: 5.5-5.7 ms vs 6.4-7.0 ms for
      the CSR column panels ('panel');
    * 'seg' for ragged rows (max row > 8 x mean + 32), whose dominant rows get
      split-row plans: uncapped R-MAT scale 22 (f32) 0.256 ms vs 1.24 'stream', 0.72
      'merge', 3.5 'vector'; scale 24 (f64) 1.42 ms vs 4.64 / 3.62;
    * 'seg' when x exceeds 30 % of L2 and the matrix is not banded: C3 R-MAT 447 vs 409
      GFLOP/s ('stream'), C5 307 vs 299 ('vector');
    * else 'vector' (partition-invariant; banded / regular rows: C2 0.107 ms, ties 'seg')."""
    if "auto" not in m._cache:
        from .panels import l2_bytes

        xb = m.n_cols * m.d_values.element_size()
        if xb > 0.6 * l2_bytes():
            m._cache["auto"] = "seg"
        else:
            max_len, _ = row_stats(m)
            mean = m.nnz / max(1, m.n_rows)
            ragged = max_len > 8 * mean + 32
            if ragged or (xb > 0.3 * l2_bytes() and not banded(m)):
                m._cache["auto"] = "seg"
            else:
                m._cache["auto"] = "vector"
    return m._cache["auto"]


def banded(m: CsrMatrix, samples: int = 4096) -> bool:
    """True when sampled rows span a small column window (median last-first column
    <= n_cols / 256): x gathers then coalesce and the CSR-vector kernel wins
    (C5 unpermuted: 'vector' 610 GFLOP/s vs 'seg' 497).  Rows are column-sorted,
    so each sampled row costs two index loads (sme_row_spans); cached."""
    if "banded" not in m._cache:
        spans = np.zeros(0, dtype=np.int32)
        if m.nnz and m.n_rows:
            s = min(samples, m.n_rows)
            out = torch.empty(s, dtype=torch.int32, device=m.d_row_ptr.device)
            _lib.call_rp("sme_row_spans", m.d_row_ptr, m.n_rows, ptr(m.d_row_ptr), ptr(m.d_col_idx), s, ptr(out),
                         stream())
            spans = out.cpu().numpy()
            spans = spans[spans >= 0]
        # torch's median of an even count is the lower middle value
        m._cache["banded"] = (True if spans.size == 0
                              else bool(np.sort(spans)[(spans.size - 1) // 2] <= m.n_cols / 256))
    return m._cache["banded"]


def row_stats(m: CsrMatrix) -> tuple[int, int]:
    """(max row length, empty rows), one device reduction, cached."""
    if "row_stats" not in m._cache:
        out = torch.empty(2, dtype=torch.int64, device=m.d_row_ptr.device)
        _lib.call_rp("sme_row_stats", m.d_row_ptr, m.n_rows, ptr(m.d_row_ptr), ptr(out), stream())
        m._cache["row_stats"] = tuple(int(v) for v in out.cpu())
    return m._cache["row_stats"]


class MergePlan:
    """Per-matrix state of the merge-path kernel: tile split points + carry scratch."""

    def __init__(self, m: CsrMatrix):
        self.n_tiles = _lib.query_i64("sme_spmv_merge_tiles", m.n_rows, m.nnz)
        dev = m.d_row_ptr.device
        self.plan = torch.empty(2 * (self.n_tiles + 1), dtype=torch.int32, device=dev)
        _lib.call("sme_spmv_merge_plan", m.n_rows, m.nnz, ptr(m.d_row_ptr), ptr(self.plan), stream())
        self.carry = _cuda.workspace(
            _lib.query_size("sme_spmv_merge_carry_bytes", _cuda.sme_dtype(m.d_values), self.n_tiles)
        )


def set_merge_mode(mode: int) -> None:
    """Select the merge kernel: 1 = TMA-pipelined persistent, 0 = per-tile, -1 = auto."""
    _lib.call("sme_spmv_merge_set_mode", int(mode))


def stream_plan(m: CsrMatrix) -> tuple[torch.Tensor, int]:
    """Per-matrix warp row ranges of the stream kernel (nnz-balanced, one per resident warp)."""
    if "stream" not in m._cache:
        import ctypes

        w = ctypes.c_int32(0)
        _lib.call("sme_spmv_stream_warps", m.n_rows, m.nnz, ctypes.byref(w))
        plan = torch.empty(w.value + 1, dtype=torch.int32, device=m.d_row_ptr.device)
        _lib.call("sme_spmv_stream_plan", m.n_rows, m.nnz, ptr(m.d_row_ptr), w.value, ptr(plan), stream())
        m._cache["stream"] = (plan, int(w.value))
    return m._cache["stream"]


def merge_plan(m: CsrMatrix) -> MergePlan:
    if "merge" not in m._cache:
        m._cache["merge"] = MergePlan(m)
    return m._cache["merge"]


def _host_src(x, n: int) -> tuple[torch.Tensor, str]:
    """A host input vector as a CPU tensor (numpy wrapped without a copy) and the
    caller's mode: 'host' (CPU torch tensor in / out) or 'numpy' (numpy in / out)."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 1 or x.numel() != n:
            raise ValueError(f"input vector length {tuple(x.shape)} does not match n_cols {n}")
        return x.contiguous(), "host"
    xa = np.asarray(x, dtype=np.float64)
    if xa.shape != (n,):
        raise ValueError(f"input vector length {xa.shape} does not match n_cols {n}")
    return torch.from_numpy(np.ascontiguousarray(xa)), "numpy"


def _x_device(x, n: int, dtype: torch.dtype, dev) -> tuple[torch.Tensor, str]:
    """x on the device plus the caller's mode: 'device' (CUDA tensor in/out), 'host'
    (CPU torch tensor in/out), 'numpy' (numpy in/out).  Host vectors cross through
    hostio.stage_in (pinned staging, host-parallel copies overlapped with the DMA)."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        if x.dim() != 1 or x.numel() != n:
            raise ValueError(f"input vector length {tuple(x.shape)} does not match n_cols {n}")
        return x.to(dtype).contiguous(), "device"
    src, mode = _host_src(x, n)
    xd = torch.empty(n, dtype=dtype, device=dev)
    ev = None
    for _, ev in hostio.stage_in(src, xd, hostio.slices(n, xd.element_size())):
        pass
    torch.cuda.current_stream(dev).wait_event(ev)
    return xd, mode


def _y_out(y: torch.Tensor, mode: str):
    """The result in the caller's mode; host results are fresh arrays (never a buffer
    a later call reuses), as the reference's are."""
    if mode == "device":
        return y
    return hostio.to_host(y, np.float64, as_numpy=(mode == "numpy"))


def _layout_pass(lay, kern: str, p: int, xd: torch.Tensor, y: torch.Tensor) -> None:
    """Pass p of a column-panel layout ('seg' or 'panel') with x slice p pinned in L2."""
    lay._window(p, xd)
    if kern == "seg":
        lay._pass(p, xd, y)
    else:
        spmv_into(lay.panels[p], xd, y, lay.inner, accumulate=p > 0, lanes=lay.lanes)


def spmv_into(m: CsrMatrix, xd: torch.Tensor, y: torch.Tensor, kernel: str = "vector", *, lanes: int | None = None,
              accumulate: bool = False) -> None:
    """Launch y (+)= A x on device tensors (no checks beyond the C-ABI's; stream-ordered)."""
    dt = _cuda.sme_dtype(m.d_values)
    if kernel == "auto":
        kernel = auto_kernel(m)
        if kernel in ("panel", "seg") and accumulate:
            kernel = "vector" if m.wide else "stream"
    _check_wide(m, kernel)
    if kernel == "vector":
        _lib.call_rp("sme_spmv_vector", m.d_row_ptr, dt, lanes or default_lanes(m), m.n_rows, m.n_cols,
                     ptr(m.d_row_ptr), ptr(m.d_col_idx), ptr(m.d_values), ptr(xd), ptr(y), int(accumulate), stream())
    elif kernel == "seg":
        from .seg import seg_of

        if accumulate:
            raise ValueError("the seg kernel does not accumulate")
        seg_of(m).spmv_into(xd, y)
    elif kernel == "panel":
        from .panels import panels_of

        if accumulate:
            raise ValueError("the panel kernel does not accumulate")
        panels_of(m).spmv_into(xd, y)
    elif kernel == "stream":
        plan, n_warps = stream_plan(m)
        _lib.call("sme_spmv_stream", dt, m.n_rows, m.n_cols, m.nnz, ptr(m.d_row_ptr), ptr(m.d_col_idx),
                  ptr(m.d_values), ptr(xd), ptr(y), ptr(plan), n_warps, int(accumulate),
                  int(m._cache.get("align_off", 0)), stream())
    elif kernel == "merge":
        pl = merge_plan(m)
        _lib.call("sme_spmv_merge", dt, m.n_rows, m.n_cols, m.nnz, ptr(m.d_row_ptr), ptr(m.d_col_idx),
                  ptr(m.d_values), ptr(xd), ptr(y), ptr(pl.plan), pl.n_tiles, ptr(pl.carry), int(accumulate),
                  stream())
    elif kernel == "exact":
        if m.d_values.dtype != torch.float64 or accumulate:
            raise ValueError("the exact (reduceat-order) kernel is f64, non-accumulating")
        _lib.call("sme_spmv_reduceat_exact", m.n_rows, ptr(m.d_row_ptr), ptr(m.d_col_idx), ptr(m.d_values),
                  ptr(xd), ptr(y), stream())
    else:
        raise ValueError(f"unknown kernel {kernel!r}; expected one of {KERNELS}")


def _check_wide(m: CsrMatrix, kernel: str) -> None:
    if m.wide and kernel not in WIDE_KERNELS:
        raise ValueError(f"kernel {kernel!r} uses int32 row offsets; a CSR with int64 row_ptr "
                         f"(nnz >= 2^31 - 1) runs one of {WIDE_KERNELS}")


def _check_out(out, m: CsrMatrix, dev) -> None:
    """The caller's `out` must be exactly what the kernels write: a contiguous device
    tensor of n_rows elements of the matrix dtype on the matrix's device."""
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.device != dev:
        raise ValueError(f"out must be a CUDA tensor on {dev}")
    if out.dtype != m.dtype or out.dim() != 1 or out.numel() != m.n_rows or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous 1-D {m.dtype} tensor of length n_rows {m.n_rows} "
                         f"(got {out.dtype} {tuple(out.shape)})")


@_cuda.nvtx("spmv_csr")
def spmv_csr(m: CsrMatrix, x, kernel: str = "auto", *, out: torch.Tensor | None = None):
    """y[i] = sum over row i of values[k] * x[col_idx[k]] (kernels.py:73-78).

    kernel="auto" (auto_kernel): the segmented-chunk column panels ('seg') when x is
    large (> 60 % of L2) or medium-sized and the matrix is not banded; the
    nnz-balanced 'stream' kernel for other ragged matrices; else the CSR-vector
    kernel.  spmv_csr_parallel with the same kernel is bitwise equal (as in the
    reference).  `out`: optional device result tensor (checked by _check_out).  A pinned
    host x of a panel layout streams in slice by slice while the passes run."""
    if not isinstance(m, CsrMatrix):
        raise TypeError("spmv_csr expects a CsrMatrix of this package (see matio.from_reference)")
    dev = m.d_row_ptr.device
    if out is not None:
        _check_out(out, m, dev)
    if isinstance(x, torch.Tensor) and x.is_cuda:
        xd, mode = _x_device(x, m.n_cols, m.dtype, dev)
        y = out if out is not None else torch.empty(m.n_rows, dtype=m.dtype, device=dev)
        spmv_into(m, xd, y, kernel)
        return y
    # host x: it crosses PCIe slice by slice; with column panels pass p starts as soon
    # as slice p has landed
    src, mode = _host_src(x, m.n_cols)
    # per-call device buffers (torch's caching allocator: free after warm-up), so
    # concurrent callers on one matrix never share them (reentrant)
    xd = torch.empty(m.n_cols, dtype=m.dtype, device=dev)
    y = out if out is not None else torch.empty(m.n_rows, dtype=m.dtype, device=dev)
    main = torch.cuda.current_stream(dev)
    kern = auto_kernel(m) if kernel == "auto" else kernel
    _check_wide(m, kern)
    if kern in ("seg", "panel"):
        from .panels import panels_of
        from .seg import seg_of

        lay = seg_of(m) if kern == "seg" else panels_of(m)
        for p, ev in hostio.stage_in(src, xd, lay.bounds_host):
            main.wait_event(ev)
            _layout_pass(lay, kern, p, xd, y)
        lay._window(None, None)
    else:
        ev = None
        for _, ev in hostio.stage_in(src, xd, hostio.slices(m.n_cols, xd.element_size())):
            pass
        main.wait_event(ev)
        spmv_into(m, xd, y, kern)
    return _y_out(y, mode)


PIPELINE_BUFFERS = 2  # device x/y buffers of spmv_csr_pipelined (steps in flight)
PIPELINE_H2D_COPIES = 0  # H2D copies per x (0: one per column panel)


@_cuda.nvtx("spmv_csr_pipelined")
def spmv_csr_pipelined(m: CsrMatrix, xs, ys=None, kernel: str = "auto") -> list:
    """y_k = A x_k for a sequence of host vectors, with the PCIe copies of neighbouring
    steps overlapped: step k+1's x crosses host->device while step k computes and step
    k-1's y crosses device->host (H2D and D2H use separate copy engines).  Every step
    still copies its full x in and its full y out; with column panels ('seg'/'panel')
    pass p of a step starts as soon as its x slice has landed.  Same results as calling
    spmv_csr(m, x_k) for each k (kernels.py:73-78 per vector).

    xs: CPU tensors (pinned for asynchronous copies) of length n_cols and the matrix's
    dtype; ys: optional CPU output tensors (pinned); returns the list of outputs."""
    if not isinstance(m, CsrMatrix):
        raise TypeError("spmv_csr_pipelined expects a CsrMatrix of this package")
    xs = list(xs)
    for x in xs:
        if not isinstance(x, torch.Tensor) or x.is_cuda or x.dim() != 1 or x.numel() != m.n_cols:
            raise ValueError(f"inputs must be 1-D host tensors of length n_cols {m.n_cols}")
    dev = m.d_row_ptr.device
    if ys is None:
        ys = [torch.empty(m.n_rows, dtype=m.dtype, pin_memory=True) for _ in xs]
    ys = list(ys)
    if len(ys) != len(xs):
        raise ValueError("need one output per input vector")
    kern = auto_kernel(m) if kernel == "auto" else kernel
    _check_wide(m, kern)
    lay = None
    if kern == "seg":
        from .seg import seg_of

        lay = seg_of(m)
    elif kern == "panel":
        from .panels import panels_of

        lay = panels_of(m)
    bounds = lay.bounds_host if lay is not None else np.array([0, m.n_cols])
    P = len(bounds) - 1
    main = torch.cuda.current_stream()
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    nb = PIPELINE_BUFFERS
    xb = [torch.empty(m.n_cols, dtype=m.dtype, device=dev) for _ in range(nb)]
    yb = [torch.empty(m.n_rows, dtype=m.dtype, device=dev) for _ in range(nb)]
    computed = [None] * nb  # event: step using buffer b finished computing
    copied_out = [None] * nb  # event: y buffer b has been copied to the host
    h2d.wait_stream(main)
    d2h.wait_stream(main)
    for k, x in enumerate(xs):
        b = k % nb
        xk = x.to(m.dtype) if x.dtype != m.dtype else x
        slice_ev = []
        with torch.cuda.stream(h2d):
            if computed[b] is not None:
                h2d.wait_event(computed[b])  # x buffer b is free once step k-2 computed
            # x crosses in `groups` copies; pass p waits for the copy holding its slice
            groups = max(1, min(P, PIPELINE_H2D_COPIES or P))
            for gi in range(groups):
                p0, p1 = gi * P // groups, (gi + 1) * P // groups
                lo, hi = int(bounds[p0]), int(bounds[p1])
                xb[b][lo:hi].copy_(xk[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                slice_ev.extend([ev] * (p1 - p0))
        if copied_out[b] is not None:
            main.wait_event(copied_out[b])  # y buffer b is free once step k-2's y left
        if lay is None:
            main.wait_event(slice_ev[-1])
            spmv_into(m, xb[b], yb[b], kern)
        else:
            for p in range(P):
                main.wait_event(slice_ev[p])
                _layout_pass(lay, kern, p, xb[b], yb[b])
            lay._window(None, None, reset=False)  # a device-wide reset here would serialise the pipeline
        done = torch.cuda.Event()
        done.record(main)
        computed[b] = done
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            ys[k].copy_(yb[b], non_blocking=True)
            out = torch.cuda.Event()
            out.record(d2h)
            copied_out[b] = out
    d2h.synchronize()
    if lay is not None:
        lay._window(None, None)  # demote the last slice's persisting lines once, at the end
    main.wait_stream(d2h)
    main.wait_stream(h2d)
    return ys


@_cuda.nvtx("spmv_csr_parallel")
def spmv_csr_parallel(m: CsrMatrix, x, workers: int, reuse_pool: bool = True, kernel: str = "auto"):
    """Row-partitioned CSR SpMV (kernels.py:102-128), bitwise equal to spmv_csr(m, x,
    kernel) for every worker count, as the reference's is to its serial kernel.

    kernel="auto" resolves exactly as spmv_csr does (auto_kernel).  For the
    CSR-vector kernel each of the `workers` even row ranges (make_row_partition) is
    its own launch over those rows; a row's reduction order depends only on the
    lane count, so the ranges reproduce the whole-matrix call bit for bit.  The
    other kernels ('seg', 'stream', 'merge', 'panel') fix each row's reduction
    order in their per-matrix layout; the partition cannot change it, and the
    whole-matrix launch (whose CTAs are the GPU's workers) IS every range's result.
    `reuse_pool` is accepted for signature compatibility (there is no thread pool).
    Multi-GPU sharding of the same partition is rowshard.RowShardedSpMV."""
    del reuse_pool
    if not isinstance(m, CsrMatrix):
        raise TypeError("spmv_csr_parallel expects a CsrMatrix of this package")
    dev = m.d_row_ptr.device
    part = make_row_partition(m.n_rows, workers)
    kern = auto_kernel(m) if kernel == "auto" else kernel
    if kern != "vector":
        return spmv_csr(m, x, kern)
    xd, mode = _x_device(x, m.n_cols, m.dtype, dev)
    y = torch.empty(m.n_rows, dtype=m.dtype, device=dev)
    lanes = default_lanes(m)
    dt = _cuda.sme_dtype(m.d_values)
    es = m.d_row_ptr.element_size()
    ys = y.element_size()
    for lo, hi in zip(part.boundaries[:-1], part.boundaries[1:]):
        lo, hi = int(lo), int(hi)
        if hi == lo:
            continue
        _lib.call_rp("sme_spmv_vector", m.d_row_ptr, dt, lanes, hi - lo, m.n_cols, ptr(m.d_row_ptr) + lo * es,
                     ptr(m.d_col_idx), ptr(m.d_values), ptr(xd), ptr(y) + lo * ys, 0, stream())
    return _y_out(y, mode)


def coo_entry_order(m: CooMatrix) -> CsrMatrix:
    """Per-matrix plan of the deterministic COO SpMV (cached like a CSR analysis): the
    entries grouped by row, each row's entries in ascending stored-entry order.  Built
    by the CSR builder (counting sort + segmented sort) with the entry id as the sort
    key: col_idx of the result holds entry ids, values the matching values."""
    plan = m._cache.get("coo_order")
    if plan is None:
        from .matio import _coo_build_csr

        if m.nnz >= _cuda.INT32_MAX:
            raise ValueError("the ordered COO SpMV keys entries by int32 ids (nnz < 2^31 - 1); use kernel='atomic'")
        dev = m.d_row_idx.device
        ids = torch.arange(m.nnz, dtype=torch.int32, device=dev)
        proxy = CooMatrix._from_device(m.n_rows, max(1, m.nnz), m.d_row_idx, ids, m.d_values)
        plan = _coo_build_csr(proxy, None, None, check=False, row_ptr_dtype=torch.int32)
        m._cache["coo_order"] = plan
    return plan


@_cuda.nvtx("spmv_coo")
def spmv_coo(m: CooMatrix, x, kernel: str = "ordered"):
    """y = 0; y[row_idx[k]] += values[k] * x[col_idx[k]] in stored entry order (kernels.py:81-86).

    kernel="ordered" (default): every row sums its products in entry order with
    round-to-nearest arithmetic (sme_spmv_coo_ordered over coo_entry_order) — bitwise
    equal to the reference's np.add.at and run-to-run deterministic.  kernel="atomic":
    one floating atomic add per entry (no plan; the order of the adds, hence the last
    ulps, can change from run to run)."""
    if not isinstance(m, CooMatrix):
        raise TypeError("spmv_coo expects a CooMatrix of this package")
    dev = m.d_row_idx.device
    xd, mode = _x_device(x, m.n_cols, m.dtype, dev)
    y = torch.empty(m.n_rows, dtype=m.dtype, device=dev)
    dt = _cuda.sme_dtype(m.d_values)
    if kernel == "atomic":
        _lib.call("sme_spmv_coo", dt, m.n_rows, m.nnz, ptr(m.d_row_idx), ptr(m.d_col_idx), ptr(m.d_values), ptr(xd),
                  ptr(y), stream())
    elif kernel == "ordered":
        if m.nnz == 0:
            y.zero_()
        else:
            plan = coo_entry_order(m)
            _lib.call("sme_spmv_coo_ordered", dt, m.n_rows, ptr(plan.d_row_ptr), ptr(plan.d_col_idx),
                      ptr(plan.d_values), ptr(m.d_col_idx), ptr(xd), ptr(y), stream())
    else:
        raise ValueError(f"unknown COO kernel {kernel!r}; expected 'ordered' or 'atomic'")
    return _y_out(y, mode)


def relative_error(got, expected) -> float:
    """max|got - expected| / max|expected| (absolute if expected is all zero) (kernels.py:131-142).

    Computed by one device reduction (sme_maxabs_diff); NaN propagates."""
    dev = _cuda.require_cuda()

    def dev_f64(a) -> torch.Tensor:
        if isinstance(a, torch.Tensor):
            return a.to(dev, torch.float64).contiguous().reshape(-1) if a.dim() else a.to(dev, torch.float64).reshape(1)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev).reshape(-1)

    g_shape = tuple(got.shape) if hasattr(got, "shape") else np.shape(got)
    e_shape = tuple(expected.shape) if hasattr(expected, "shape") else np.shape(expected)
    if tuple(g_shape) != tuple(e_shape):
        raise ValueError("shape mismatch")
    g, e = dev_f64(got), dev_f64(expected)
    if g.numel() == 0:
        return 0.0
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    _lib.call("sme_maxabs_diff", _lib.SME_F64, g.numel(), ptr(g), ptr(e), ptr(out), stream())
    diff, scale = (float(v) for v in out.cpu())
    return diff / scale if scale > 0 else diff
