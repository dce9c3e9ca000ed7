"""Segmented-chunk SpMV layout (spmv_seg.cu): column panels without row_ptr.

The replacement of spmv_csr (kernels.py:59-78) for randomly permuted matrices.
The columns are split into P panels whose x slices stay L2-resident (see
panels.py for why); each panel stores its entries in CSR order as 32-bit
words (column within the panel, row offset within the 128-entry chunk) plus
one header row per chunk, so a pass streams 4 + sizeof(value) bytes per entry
and nothing per row.  SpMV = one non-accumulating pass (panel 0, which holds
an explicit zero for every row it has no entry of) and P-1 accumulating ones.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .matio import CsrMatrix

CHUNK = 128
MAX_PANEL_COLS = (1 << 23) - 2  # 23-bit column field, all-ones reserved for explicit zeros


def seg_warps() -> int:
    w = ctypes.c_int32(0)
    _lib.call("sme_spmv_seg_warps", ctypes.byref(w))
    return int(w.value)


def auto_seg_panels(m: CsrMatrix, l2_fraction: float = 0.38) -> int:
    """P: the x slice fits `l2_fraction` of L2 (50 MB slices of the 132.6 MB B200 L2)
    and every panel is narrower than the 23-bit column field."""
    from .panels import l2_bytes

    xb = m.n_cols * m.d_values.element_size()
    p = max(1, math.ceil(xb / (l2_bytes() * l2_fraction)))
    # int32 slot positions per panel: keep every panel near 2^30 slots at most (nnz >= 2^31)
    p = max(p, math.ceil((m.nnz + m.n_rows) / (1 << 30)))
    return max(p, math.ceil(m.n_cols / MAX_PANEL_COLS))


class SegLayout:
    """P column panels of a CsrMatrix in the segmented-chunk layout."""

    def __init__(self, m: CsrMatrix, n_panels: int, n_warps: int | None = None, full_last: bool = False,
                 split_rows: bool | None = None):
        P, n = self._geometry(m, n_panels, full_last)
        s = stream()
        ws = _cuda.workspace(_lib.query_size("sme_seg_workspace_size", n, P))
        pos = torch.empty(P * (n + 1), dtype=torch.int32, device=self.bounds.device)
        _lib.call_rp("sme_seg_positions", m.d_row_ptr, n, ptr(m.d_row_ptr), ptr(m.d_col_idx), P, ptr(self.bounds),
                     int(full_last), ptr(pos), ptr(ws), ws.numel(), s)
        h_offs, d_offs = self._allocate(pos)
        _lib.call_rp("sme_seg_fill", m.d_row_ptr, _cuda.sme_dtype(m.d_values), n, ptr(m.d_row_ptr),
                     ptr(m.d_col_idx), ptr(m.d_values), P, ptr(self.bounds), ptr(pos), ptr(d_offs),
                     ctypes.cast(h_offs, ctypes.c_void_p), ptr(self.pk), ptr(self.val), ptr(self.hdr), ptr(ws), s)
        self._finish(m, pos, n_warps, split_rows)

    # -- construction pieces ------------------------------------------------------
    def _geometry(self, m: CsrMatrix, n_panels: int, full_last: bool) -> tuple[int, int]:
        P, n = int(n_panels), m.n_rows
        if P < 1 or P > max(1, m.n_cols):
            raise ValueError("panel count must lie in [1, n_cols]")
        bounds = np.array([p * m.n_cols // P for p in range(P + 1)], dtype=np.int32)
        if np.diff(bounds).max(initial=0) > MAX_PANEL_COLS:
            raise ValueError(f"panels of {int(np.diff(bounds).max())} columns exceed the 23-bit column field; "
                             f"use at least {math.ceil(m.n_cols / MAX_PANEL_COLS)} panels")
        self.n_rows, self.n_cols, self.n_panels, self.dtype = n, m.n_cols, P, m.dtype
        self.bounds_host = bounds
        self.bounds = torch.from_numpy(bounds).to(m.d_col_idx.device)
        self.full_last = bool(full_last)
        return P, n

    def _allocate(self, pos: torch.Tensor):
        """Panel sizes from the positions (one host sync), pk / val / hdr, tail padding."""
        P, n, dev = self.n_panels, self.n_rows, pos.device
        ent = pos.view(P, n + 1)[:, -1].cpu().numpy().astype(np.int64)
        if (ent < 0).any():  # int32 slot positions wrapped: a panel of >= 2^31 slots
            raise ValueError(f"a column panel holds >= 2^31 entries; use more than {P} panels")
        offs = np.zeros(P + 1, dtype=np.int64)
        for p in range(P):
            offs[p + 1] = offs[p] + -(-int(ent[p]) // CHUNK) * CHUNK
        total = max(int(offs[-1]), CHUNK)
        self.entries = ent
        self.offsets = offs
        # the fill writes every entry slot and every chunk header; only each panel's tail
        # padding (< CHUNK slots) is set here, as explicit zeros
        self.pk = torch.empty(total, dtype=torch.int32, device=dev)
        self.val = torch.empty(total, dtype=self.dtype, device=dev)
        self.hdr = torch.zeros(total // CHUNK, dtype=torch.int32, device=dev) if total == CHUNK else \
            torch.empty(total // CHUNK, dtype=torch.int32, device=dev)
        for p in range(P):
            lo, hi = int(offs[p] + ent[p]), int(offs[p + 1])
            if hi > lo:
                self.pk[lo:hi] = -1
                self.val[lo:hi] = 0
        if total > int(offs[-1]):  # an all-empty layout: one chunk of explicit zeros
            self.pk[int(offs[-1]):] = -1
            self.val[int(offs[-1]):] = 0
        h_offs = (ctypes.c_int64 * P)(*[int(o) for o in offs[:P]])
        d_offs = torch.from_numpy(offs[:P].copy()).to(dev)
        return h_offs, d_offs

    def _finish(self, m: CsrMatrix, pos: torch.Tensor, n_warps: int | None, split_rows: bool | None) -> None:
        P, n, dev, s = self.n_panels, self.n_rows, pos.device, stream()
        ent = self.entries
        self.n_warps = int(n_warps or seg_warps())
        self.plans = torch.empty(P * (self.n_warps + 1), dtype=torch.int32, device=dev)
        # split-row plans when one row would dominate a warp's share (power-law rows): ranges
        # then end mid-row and an ordered fix-up adds the open partials; the fused epilogue
        # then runs as its own row pass (sme_rows_epi) after the passes
        if split_rows is None:
            from .kernels import row_stats

            max_len, _ = row_stats(m)
            split_rows = max_len > max(256, 0.25 * m.nnz / max(1, self.n_warps))
        self.split_rows = bool(split_rows)
        for p in range(P):
            if self.split_rows:
                _lib.call("sme_seg_plan_split", int(ent[p]), self.n_warps, ptr(self.plans) + p * (self.n_warps + 1) * 4,
                          s)
            else:
                _lib.call("sme_seg_plan", n, ptr(pos) + p * (n + 1) * 4, self.n_warps,
                          ptr(self.plans) + p * (self.n_warps + 1) * 4, s)
        if self.split_rows:
            self.carry_val = torch.empty(self.n_warps, dtype=m.dtype, device=dev)
            self.carry_row = torch.empty(self.n_warps, dtype=torch.int32, device=dev)
        # partials scratch of the fused epilogue: per warp (in-pass) or per block (row pass)
        self.epi_partials_len = (max(self.n_warps, _lib.query_i64("sme_rows_epi_blocks", n)) if self.split_rows
                                 else self.n_warps)
        torch.cuda.current_stream().synchronize()  # pos / ws are freed on return
        self.nnz = m.nnz
        self.persist = False
        self.hit_ratio = 1.0  # access-policy window hit ratio of the pinned x slice
        self.warm = False  # L2 prefetch sweep of each pass's x slice (experiment knob)

    # -- passes --------------------------------------------------------------
    def _pass(self, p: int, xd: torch.Tensor, y: torch.Tensor) -> None:
        vb = self.val.element_size()
        o = int(self.offsets[p])
        if self.warm:  # sweep the pass's x slice into L2 before its random gathers
            lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
            _lib.call("sme_l2_prefetch", ptr(xd) + vb * lo, (hi - lo) * vb, stream())
        if self.split_rows:
            _lib.call("sme_spmv_seg_split", _cuda.sme_dtype(self.val), self.n_warps, ptr(self.pk) + 4 * o,
                      ptr(self.val) + vb * o, ptr(self.hdr) + 4 * (o // CHUNK),
                      ptr(self.plans) + 4 * p * (self.n_warps + 1), ptr(xd) + vb * int(self.bounds_host[p]), ptr(y),
                      int(p > 0), ptr(self.carry_val), ptr(self.carry_row), stream())
            return
        _lib.call("sme_spmv_seg", _cuda.sme_dtype(self.val), self.n_warps, ptr(self.pk) + 4 * o, ptr(self.val) + vb * o,
                  ptr(self.hdr) + 4 * (o // CHUNK), ptr(self.plans) + 4 * p * (self.n_warps + 1),
                  ptr(xd) + vb * int(self.bounds_host[p]), ptr(y), int(p > 0), stream())

    def epi_pass(self, xd: torch.Tensor, y: torch.Tensor, out: torch.Tensor, qinv: torch.Tensor | None,
                 scal: torch.Tensor, partials: torch.Tensor, ticket: torch.Tensor, result: torch.Tensor) -> None:
        """Passes 0..P-2 into y, then the last pass with the fused iteration epilogue
        (sme_spmv_seg_epi): out[qinv[r]] = scal[0] * (A x)[r], result = {1/||out||, ||out||^2}."""
        if not self.full_last:
            raise ValueError("the fused epilogue needs a layout built with full_last=True")
        P = self.n_panels
        if self.split_rows:  # passes end mid-row: all passes into y, then the epilogue as a row pass
            self.spmv_into(xd, y)
            _lib.call("sme_rows_epi", self.n_rows, ptr(y), ptr(out), ptr(qinv), ptr(scal), None, ptr(partials),
                      ptr(ticket), ptr(result), 0, stream())
            return
        for p in range(P - 1):
            self._window(p, xd)
            self._pass(p, xd, y)
        self._window(P - 1, xd)
        vb = self.val.element_size()
        o = int(self.offsets[P - 1])
        _lib.call("sme_spmv_seg_epi", _cuda.sme_dtype(self.val), self.n_warps, ptr(self.pk) + 4 * o,
                  ptr(self.val) + vb * o, ptr(self.hdr) + 4 * (o // CHUNK),
                  ptr(self.plans) + 4 * (P - 1) * (self.n_warps + 1), ptr(xd) + vb * int(self.bounds_host[P - 1]),
                  ptr(y), int(P > 1), ptr(out), ptr(qinv), ptr(scal), ptr(partials), ptr(ticket), ptr(result),
                  stream())
        self._window(None, None)

    def epi_cg_pass(self, p: torch.Tensor, y: torch.Tensor, out: torch.Tensor, partials: torch.Tensor,
                    ticket: torch.Tensor, scal: torch.Tensor) -> None:
        """out = A p with p.Ap reduced in the last pass and alpha = scal[0] / p.Ap -> scal[1]
        (sme_spmv_seg_epi_cg)."""
        if not self.full_last:
            raise ValueError("the fused epilogue needs a layout built with full_last=True")
        P = self.n_panels
        if self.split_rows:
            self.spmv_into(p, y)
            _lib.call("sme_rows_epi", self.n_rows, ptr(y), ptr(out), None, None, ptr(p), ptr(partials), ptr(ticket),
                      ptr(scal), 1, stream())
            return
        for q in range(P - 1):
            self._window(q, p)
            self._pass(q, p, y)
        self._window(P - 1, p)
        vb = self.val.element_size()
        o = int(self.offsets[P - 1])
        _lib.call("sme_spmv_seg_epi_cg", _cuda.sme_dtype(self.val), self.n_warps, ptr(self.pk) + 4 * o,
                  ptr(self.val) + vb * o, ptr(self.hdr) + 4 * (o // CHUNK),
                  ptr(self.plans) + 4 * (P - 1) * (self.n_warps + 1), ptr(p) + vb * int(self.bounds_host[P - 1]),
                  ptr(p), ptr(y), int(P > 1), ptr(out), ptr(partials), ptr(ticket), ptr(scal), stream())
        self._window(None, None)

    def _window(self, p: int | None, xd: torch.Tensor | None, reset: bool = True) -> None:
        """Pin x slice p in L2 (access-policy window), or clear the window (p None) and,
        with `reset`, demote the persisting lines.  The reset waits for the whole device,
        so a pipeline of steps (spmv_csr_pipelined) clears without it and resets once."""
        if not self.persist:
            return
        if p is None:
            _lib.call("sme_l2_window", None, 0, 0.0, stream())
            if reset:
                _lib.call("sme_l2_reset_persisting")
            return
        vb = xd.element_size()
        lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
        _lib.call("sme_l2_window", ptr(xd) + lo * vb, (hi - lo) * vb, float(self.hit_ratio), stream())

    def spmv_into(self, xd: torch.Tensor, y: torch.Tensor) -> None:
        """y = A x on device tensors: P stream-ordered launches."""
        for p in range(self.n_panels):
            self._window(p, xd)
            self._pass(p, xd, y)
        self._window(None, None)

    def spmv_host(self, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor) -> None:
        """y_host = A x_host with pinned host vectors: the H2D copy of x slice p+1 overlaps
        pass p (each pass reads only its slice); y returns in one D2H.  Synchronous."""
        main = torch.cuda.current_stream()
        cs = self._copy_stream = getattr(self, "_copy_stream", None) or torch.cuda.Stream(device=x_dev.device)
        cs.wait_stream(main)
        events = []
        with torch.cuda.stream(cs):
            for p in range(self.n_panels):
                lo, hi = int(self.bounds_host[p]), int(self.bounds_host[p + 1])
                x_dev[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                events.append(ev)
        for p in range(self.n_panels):
            main.wait_event(events[p])
            self._window(p, x_dev)
            self._pass(p, x_dev, y_dev)
        self._window(None, None)
        y_host.copy_(y_dev, non_blocking=True)
        main.synchronize()

    def enable_persistence(self, on: bool = True) -> None:
        """Reserve persisting L2 for one x slice and pin each pass's slice with an access-policy window."""
        if on:
            from .panels import device_info

            info = device_info()
            slice_bytes = int(max(np.diff(self.bounds_host))) * self.val.element_size()
            _lib.call("sme_l2_set_persisting", min(info["max_persisting_l2"], slice_bytes))
        self.persist = on

    # -- accounting ------------------------------------------------------------
    def stream_bytes(self) -> int:
        """DRAM bytes one SpMV streams: entries (pk + val), headers, x once, y written
        once plus (P-1) read+write passes."""
        vb = self.val.element_size()
        ent = int(self.entries.sum())
        return (ent * (4 + vb) + int(self.hdr.numel()) * 4 + self.n_cols * vb
                + self.n_rows * vb * (2 * self.n_panels - 1))

    def launches(self) -> int:
        return self.n_panels


def seg_of(m: CsrMatrix, n_panels: int | None = None, full_last: bool = False,
           split_rows: bool | None = None) -> SegLayout:
    """The cached segmented-chunk layout of m (built on first use)."""
    P = n_panels or m._cache.get("seg_panels") or auto_seg_panels(m)
    key = ("seg", P, bool(full_last)) if split_rows is None else ("seg", P, bool(full_last), bool(split_rows))
    if key not in m._cache:
        install(m, key, SegLayout(m, P, full_last=full_last, split_rows=split_rows))
    return m._cache[key]


def install(m: CsrMatrix, key, lay: SegLayout) -> None:
    """Cache `lay` as m's layout `key` (pinning each pass's x slice in L2 when it fits
    the persisting carve-out)."""
    from .panels import device_info

    slice_bytes = int(max(np.diff(lay.bounds_host))) * m.d_values.element_size()
    if lay.n_panels > 1 and slice_bytes <= device_info()["max_persisting_l2"]:
        lay.enable_persistence(True)
    m._cache[key] = lay
