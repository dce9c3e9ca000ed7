"""On-disk cache of permuted CSR matrices and their seg layouts.

The reference persists a permuted matrix through `cmd_permute` -> `write_matrix_market`
(cli.py:173-230, matio.py:262-278): text, re-parsed and re-sorted on every load.  Here
a permuted matrix is stored as a versioned binary image of its device arrays —
`row_ptr`, `col_idx`, `values` and, optionally, the segmented-chunk column-panel
layout the SpMV runs on (seg.py) — so a reload is one read per array straight into
pinned memory and one DMA each, with no sort and no layout build.  A cache entry is
keyed by the content hashes (sme_hash64) of the source matrix and of both
permutations, so `permute_csr_cached` returns exactly what `permute_csr` would.

File layout (little endian):
  b"SMECACHE" | u32 version | u32 header bytes | header (JSON, utf-8) | pad to 4096
  | each array's raw bytes at the 4096-aligned offset the header records.
The header holds the kind, shape, dtype, key, per-array {dtype, count, offset,
hash64} and the layout's scalar fields.  load() checks the magic, the version and
(with verify=True) every array's hash after upload.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
from pathlib import Path

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .matio import CsrMatrix

MAGIC = b"SMECACHE"
VERSION = 1
ALIGN = 4096
_DT = {"int32": torch.int32, "int64": torch.int64, "float64": torch.float64, "float32": torch.float32}


def hash64(t: torch.Tensor, seed: int = 0) -> int:
    """Content hash of a device tensor's bytes (sme_hash64)."""
    t = t.contiguous()
    out = torch.empty(1, dtype=torch.int64, device=t.device)
    _lib.call("sme_hash64", ptr(t), t.numel() * t.element_size(), seed, ptr(out), stream())
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF


def matrix_key(m: CsrMatrix, p_r=None, p_c=None) -> str:
    """Cache key of permute_csr(m, p_r, p_c): shape, dtype and the content hashes of
    m's arrays and of both permutations (None = identity)."""
    parts = [m.n_rows, m.n_cols, m.nnz, str(m.dtype).replace("torch.", ""),
             hash64(m.d_row_ptr, 1), hash64(m.d_col_idx, 2), hash64(m.d_values, 3)]
    for k, p in ((4, p_r), (5, p_c)):
        parts.append(0 if p is None else hash64(p.d_forward, k))
    return hashlib.sha256(json.dumps(parts).encode()).hexdigest()[:32]


def _np_dtype(t: torch.Tensor) -> str:
    return str(t.dtype).replace("torch.", "")


def _layout_arrays(lay) -> dict[str, torch.Tensor]:
    return {"seg.pk": lay.pk, "seg.val": lay.val, "seg.hdr": lay.hdr, "seg.plans": lay.plans,
            "seg.bounds": lay.bounds}


def save(path, m: CsrMatrix, *, layout=None, key: str | None = None, meta: dict | None = None) -> Path:
    """Write m (and optionally one SegLayout of it) to `path` atomically (tmp + rename)."""
    path = Path(path)
    arrays = {"row_ptr": m.d_row_ptr, "col_idx": m.d_col_idx, "values": m.d_values}
    head = {"kind": "csr", "n_rows": m.n_rows, "n_cols": m.n_cols, "nnz": m.nnz, "dtype": _np_dtype(m.d_values),
            "key": key, "meta": meta or {}, "arrays": {}}
    if layout is not None:
        arrays.update(_layout_arrays(layout))
        head["seg"] = {"n_panels": layout.n_panels, "n_warps": layout.n_warps, "full_last": layout.full_last,
                       "split_rows": layout.split_rows, "entries": [int(v) for v in layout.entries],
                       "offsets": [int(v) for v in layout.offsets], "bounds": [int(v) for v in layout.bounds_host],
                       "epi_partials_len": int(layout.epi_partials_len)}
    off = 0
    order = list(arrays)
    for name in order:
        t = arrays[name]
        nb = t.numel() * t.element_size()
        head["arrays"][name] = {"dtype": _np_dtype(t), "count": int(t.numel()), "offset": off,
                                "hash64": "%016x" % hash64(t, 7)}
        off += -(-nb // ALIGN) * ALIGN
    hb = json.dumps(head, sort_keys=True).encode()
    pre = MAGIC + struct.pack("<II", VERSION, len(hb)) + hb
    base = -(-len(pre) // ALIGN) * ALIGN
    tmp = path.with_name(path.name + f".tmp{os.getpid()}")
    bufs = _pinned_pair()
    with open(tmp, "wb") as f:
        f.write(pre + b"\0" * (base - len(pre)))
        for name in order:
            _write_array(f, arrays[name], bufs)
    os.replace(tmp, path)
    return path


def read_header(path) -> tuple[dict, int]:
    """(header, data base offset); raises ValueError on a foreign or newer file."""
    with open(path, "rb") as f:
        pre = f.read(16)
        if len(pre) < 16 or pre[:8] != MAGIC:
            raise ValueError(f"{path}: not an sme cache file")
        ver, hlen = struct.unpack("<II", pre[8:16])
        if ver != VERSION:
            raise ValueError(f"{path}: cache version {ver}, this build reads {VERSION}")
        head = json.loads(f.read(hlen).decode())
    return head, -(-(16 + hlen) // ALIGN) * ALIGN


CHUNK_BYTES = 64 << 20  # file <-> device moves in pinned chunks (two in flight)


def _pinned_pair() -> list[torch.Tensor]:
    return [torch.empty(CHUNK_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]


def _read_array(f, base: int, spec: dict, dev, bufs) -> torch.Tensor:
    """Read one array into a new device tensor: file -> pinned chunk -> DMA, the read
    of chunk k+1 overlapping the copy of chunk k."""
    dt = _DT[spec["dtype"]]
    n = int(spec["count"])
    out = torch.empty(n, dtype=dt, device=dev)
    nbytes = n * out.element_size()
    if nbytes == 0:
        return out
    raw = out.view(torch.uint8) if out.dim() else out
    f.seek(base + int(spec["offset"]))
    cs = torch.cuda.current_stream(dev)
    done = [None, None]
    pos, k = 0, 0
    while pos < nbytes:
        b = k & 1
        if done[b] is not None:
            done[b].synchronize()  # the DMA out of this pinned chunk has finished
        step = min(CHUNK_BYTES, nbytes - pos)
        mv = memoryview(bufs[b].numpy())[:step]
        got = f.readinto(mv)
        if got != step:
            raise ValueError(f"truncated cache file: array needs {nbytes} bytes, read {pos + got}")
        raw[pos:pos + step].copy_(bufs[b][:step], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cs)
        done[b] = ev
        pos += step
        k += 1
    return out


def _write_array(f, t: torch.Tensor, bufs) -> None:
    """Device -> pinned chunk -> file, the DMA of chunk k+1 overlapping the write of k."""
    raw = t.contiguous().view(torch.uint8) if t.numel() else t
    nbytes = t.numel() * t.element_size()
    cs = torch.cuda.current_stream(t.device)
    pending = []
    pos, k = 0, 0
    while pos < nbytes or pending:
        if pos < nbytes:
            step = min(CHUNK_BYTES, nbytes - pos)
            b = k & 1
            bufs[b][:step].copy_(raw[pos:pos + step], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            pending.append((ev, b, step))
            pos += step
            k += 1
        if len(pending) == 2 or (pos >= nbytes and pending):
            ev, b, step = pending.pop(0)
            ev.synchronize()
            f.write(memoryview(bufs[b].numpy())[:step])
    f.write(b"\0" * (-nbytes % ALIGN))


def load(path, device=None, *, with_layout: bool = True, verify: bool = False) -> CsrMatrix:
    """Read a cached matrix back to the device (bit-identical); its seg layout, if stored
    and built for this device's warp count, is installed in the matrix's plan cache so
    the first SpMV skips the layout build."""
    dev = torch.device(device) if device is not None else _cuda.require_cuda()
    head, base = read_header(path)
    arrs = {}
    want = ["row_ptr", "col_idx", "values"]
    if with_layout and "seg" in head:
        want += [n for n in head["arrays"] if n.startswith("seg.")]
    bufs = _pinned_pair()
    with open(path, "rb") as f:
        for name in want:
            arrs[name] = _read_array(f, base, head["arrays"][name], dev, bufs)
    torch.cuda.current_stream(dev).synchronize()
    if verify:
        for name, t in arrs.items():
            if "%016x" % hash64(t, 7) != head["arrays"][name]["hash64"]:
                raise ValueError(f"{path}: array {name} does not match its recorded hash")
    m = CsrMatrix._from_device(head["n_rows"], head["n_cols"], arrs["row_ptr"], arrs["col_idx"], arrs["values"])
    if with_layout and "seg" in head:
        _install_layout(m, head["seg"], arrs)
    return m


def _install_layout(m: CsrMatrix, s: dict, arrs: dict) -> None:
    from .panels import device_info
    from .seg import SegLayout, seg_warps

    if int(s["n_warps"]) != seg_warps():  # plans are per device shape: rebuild lazily instead
        return
    lay = SegLayout.__new__(SegLayout)
    lay.n_rows, lay.n_cols, lay.n_panels, lay.dtype = m.n_rows, m.n_cols, int(s["n_panels"]), m.dtype
    lay.bounds_host = np.asarray(s["bounds"], dtype=np.int32)
    lay.bounds = arrs["seg.bounds"]
    lay.full_last = bool(s["full_last"])
    lay.entries = np.asarray(s["entries"], dtype=np.int64)
    lay.offsets = np.asarray(s["offsets"], dtype=np.int64)
    lay.pk, lay.val, lay.hdr, lay.plans = arrs["seg.pk"], arrs["seg.val"], arrs["seg.hdr"], arrs["seg.plans"]
    lay.n_warps = int(s["n_warps"])
    lay.split_rows = bool(s["split_rows"])
    dev = m.d_row_ptr.device
    if lay.split_rows:
        lay.carry_val = torch.empty(lay.n_warps, dtype=m.dtype, device=dev)
        lay.carry_row = torch.empty(lay.n_warps, dtype=torch.int32, device=dev)
    lay.epi_partials_len = int(s["epi_partials_len"])
    lay.nnz = m.nnz
    lay.persist, lay.hit_ratio, lay.warm = False, 1.0, False
    slice_bytes = int(max(np.diff(lay.bounds_host))) * m.d_values.element_size()
    if lay.n_panels > 1 and slice_bytes <= device_info()["max_persisting_l2"]:
        lay.enable_persistence(True)
    m._cache[("seg", lay.n_panels, lay.full_last)] = lay
    m._cache["seg_panels"] = lay.n_panels


def permute_csr_cached(m: CsrMatrix, p_r, p_c, cache_dir, *, layout: bool = True, verify: bool = False) -> CsrMatrix:
    """permute_csr(m, p_r, p_c) through the on-disk cache: a hit loads the stored result
    (and its seg layout); a miss computes it, builds the layout the SpMV would use, and
    stores both.  Returns the same bits either way."""
    from .permute import _as_perm, permute_csr

    p_r = None if p_r is None else _as_perm(p_r)
    p_c = None if p_c is None else _as_perm(p_c)
    key = matrix_key(m, p_r, p_c)
    path = Path(cache_dir) / f"permuted-{key}.smecache"
    if path.exists():
        head, _ = read_header(path)
        if head.get("key") == key:
            return load(path, m.d_row_ptr.device, with_layout=layout, verify=verify)
    B = permute_csr(m, p_r, p_c)
    lay = None
    if layout:
        from .kernels import auto_kernel
        from .seg import seg_of

        if auto_kernel(B) == "seg":
            lay = seg_of(B)
    Path(cache_dir).mkdir(parents=True, exist_ok=True)
    save(path, B, layout=lay, key=key)
    return B
