"""Column-panel layout of a CSR matrix for L2-resident x gathers (panel.cu).

For a matrix whose x does not fit in L2 (C4: 400 MB of x against 126 MB of
L2) random gathers miss to DRAM; splitting the columns into P panels and
running P accumulating SpMV passes (y = A_0 x_0; y += A_p x_p) keeps each
pass's x slice resident.  Each panel is an ordinary CsrMatrix sharing one
col/val buffer, so every SpMV kernel runs on it unchanged.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .matio import CsrMatrix

CHUNK = 128  # panel offsets keep the global 128-element chunk alignment


def device_info() -> dict:
    import ctypes

    _cuda.require_cuda()
    out = (ctypes.c_int64 * 6)()
    _lib.call("sme_device_info", ctypes.cast(out, ctypes.c_void_p))
    keys = ("l2", "max_persisting_l2", "max_window", "sms", "smem_per_sm", "smem_per_block")
    return dict(zip(keys, (int(v) for v in out)))


def l2_bytes() -> int:
    return device_info()["l2"]


def auto_panels(m: CsrMatrix, l2_fraction: float = 0.38) -> int:
    """Smallest P whose x slice fits in `l2_fraction` of L2 (0.38 of the 132.6 MB
    B200 L2 = 50 MB slices: C4 P=8 measured 6.36 ms vs P=7 6.41, P=6 6.56)."""
    xb = m.n_cols * m.d_values.element_size()
    return max(1, math.ceil(xb / (l2_bytes() * l2_fraction)))


class PanelCsr:
    """P column panels of a CsrMatrix (bounds b_p = p * n_cols // P)."""

    def __init__(self, m: CsrMatrix, n_panels: int):
        if n_panels < 1 or n_panels > max(1, m.n_cols):
            raise ValueError("panel count must lie in [1, n_cols]")
        dev = m.d_row_ptr.device
        P, n = int(n_panels), m.n_rows
        self.n_rows, self.n_cols, self.n_panels = m.n_rows, m.n_cols, P
        bounds = np.array([p * m.n_cols // P for p in range(P + 1)], dtype=np.int32)
        self.bounds_host = bounds
        self.bounds = torch.from_numpy(bounds).to(dev)
        self.panel_ptr = torch.empty(P * (n + 1), dtype=torch.int32, device=dev)
        ws = _cuda.workspace(_lib.query_size("sme_panel_count_workspace_size", n, P))
        _lib.call("sme_panel_row_ptrs", n, ptr(m.d_row_ptr), ptr(m.d_col_idx), P, ptr(self.bounds),
                  ptr(self.panel_ptr), ptr(ws), ws.numel(), stream())
        nnz_p = self.panel_ptr.view(P, n + 1)[:, -1].to(torch.int64).cpu().numpy()
        offs = np.zeros(P + 1, dtype=np.int64)
        for p in range(P):
            offs[p + 1] = offs[p] + -(-int(nnz_p[p]) // CHUNK) * CHUNK
        total = int(offs[-1])
        self.col = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        self.val = torch.empty(max(total, 1), dtype=m.dtype, device=dev)
        d_offs = torch.from_numpy(offs[:P].copy()).to(dev)
        _lib.call("sme_panel_scatter", _cuda.sme_dtype(m.d_values), n, ptr(m.d_row_ptr), ptr(m.d_col_idx),
                  ptr(m.d_values), P, ptr(self.bounds), ptr(self.panel_ptr), ptr(d_offs), ptr(self.col),
                  ptr(self.val), stream())
        self.panels = []
        for p in range(P):
            a, k = int(offs[p]), int(nnz_p[p])
            rp = self.panel_ptr[p * (n + 1) : (p + 1) * (n + 1)]
            self.panels.append(CsrMatrix._from_device(n, m.n_cols, rp, self.col[a : a + k], self.val[a : a + k]))
        self.nnz = int(nnz_p.sum())
        self.offsets = offs

    persist: bool = False  # pin each pass's x slice with an L2 access-policy window

    inner: str = "stream"  # kernel of each pass
    lanes: int | None = None  # CSR-vector lanes when inner == "vector"

    def _window(self, p: int | None, xd: torch.Tensor | None, reset: bool = True) -> None:
        """Pin x slice p in L2 (access-policy window) or clear the window (p None; with
        `reset` also demote the persisting lines, which waits for the device)."""
        if not self.persist:
            return
        if p is None:
            _lib.call("sme_l2_window", None, 0, 0.0, stream())
            if reset:
                _lib.call("sme_l2_reset_persisting")
            return
        vb = xd.element_size()
        lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
        _lib.call("sme_l2_window", ptr(xd) + lo * vb, (hi - lo) * vb, 1.0, stream())

    def spmv_into(self, xd: torch.Tensor, y: torch.Tensor, kernel: str | None = None) -> None:
        from .kernels import spmv_into

        kernel = kernel or self.inner
        vb = xd.element_size()
        for p, a in enumerate(self.panels):
            if self.persist:
                lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
                _lib.call("sme_l2_window", ptr(xd) + lo * vb, (hi - lo) * vb, 1.0, stream())
            spmv_into(a, xd, y, kernel, accumulate=p > 0, lanes=self.lanes)
        if self.persist:
            _lib.call("sme_l2_window", None, 0, 0.0, stream())
            _lib.call("sme_l2_reset_persisting")

    def spmv_host(self, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor,
                  kernel: str | None = None) -> None:
        """y_host = A x_host with host (pinned) vectors: the H2D copy of x slice p+1
        runs on a copy stream while pass p computes (each pass needs only its
        own slice), then y comes back in one D2H.  Synchronous on return."""
        from .kernels import spmv_into

        kernel = kernel or self.inner
        main = torch.cuda.current_stream()
        cs = self._copy_stream = getattr(self, "_copy_stream", None) or torch.cuda.Stream(device=x_dev.device)
        cs.wait_stream(main)  # x_dev may still be read by the previous call
        events = []
        with torch.cuda.stream(cs):
            for p in range(self.n_panels):
                lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
                x_dev[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                events.append(ev)
        vb = x_dev.element_size()
        for p, a in enumerate(self.panels):
            main.wait_event(events[p])
            if self.persist:
                lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
                _lib.call("sme_l2_window", ptr(x_dev) + lo * vb, (hi - lo) * vb, 1.0, stream())
            spmv_into(a, x_dev, y_dev, kernel, accumulate=p > 0, lanes=self.lanes)
        if self.persist:
            _lib.call("sme_l2_window", None, 0, 0.0, stream())
            _lib.call("sme_l2_reset_persisting")
        y_host.copy_(y_dev, non_blocking=True)
        main.synchronize()

    def enable_persistence(self, on: bool = True) -> None:
        """Reserve persisting L2 for one x slice (device limit) and pin it per pass."""
        if on:
            info = device_info()
            slice_bytes = int(max(np.diff(self.bounds_host))) * self.val.element_size()
            _lib.call("sme_l2_set_persisting", min(info["max_persisting_l2"], slice_bytes))
        self.persist = on

    def algorithmic_extra_bytes(self) -> int:
        """Bytes the panel passes add to one SpMV: (P-1) y read+write and P-1 more row_ptr arrays."""
        vb = self.val.element_size()
        return (self.n_panels - 1) * (2 * self.n_rows * vb + (self.n_rows + 1) * 4)


def panels_of(m: CsrMatrix, n_panels: int | None = None) -> PanelCsr:
    """The cached panel layout of m (built on first use)."""
    if m.wide:
        raise ValueError("the CSR column panels use int32 row offsets; a CSR with int64 row_ptr runs 'seg'")
    P = n_panels or m._cache.get("n_panels") or auto_panels(m)
    key = ("panels", P)
    if key not in m._cache:
        pc = PanelCsr(m, P)
        # pin each pass's x slice when it fits the persisting carve-out (measured on
        # B200 C4: P=6 7.57 -> 7.12 ms; larger slices thrash the carve-out)
        slice_bytes = int(max(np.diff(pc.bounds_host))) * m.d_values.element_size()
        if P > 1 and slice_bytes <= device_info()["max_persisting_l2"]:
            pc.enable_persistence(True)
        m._cache[key] = pc
    return m._cache[key]
