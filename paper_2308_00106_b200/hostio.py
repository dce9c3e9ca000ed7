"""Host <-> device vector movement for the reference-shaped calls.

The reference API takes numpy vectors and returns fresh numpy arrays (kernels.py:73-78,
SURVEY.md §8b gotchas 1 and 3: a KernelSpec receives the host x_perm on every call).
Moving a 400 MB vector naively costs far more than the SpMV: a pageable H2D copy is
staged by the driver, and a fresh 400 MB numpy result is ~100k first-touch page faults
(C4, tools/numpy_path_probe.py: 35 ms in, 185 ms out, against a 5.3 ms SpMV).  Here:

* inputs cross in slices through a reused pinned buffer: the host-parallel copy
  (torch copy_) of slice p+1 overlaps the DMA of slice p, and the caller can start
  work on slice p as soon as its event fires (column panels: pass p);
* outputs land in FRESH host memory (never an alias of a live array): anonymous
  mappings that are page-locked once and recycled through a pool when the caller
  drops the array, so a result crosses PCIe in one DMA straight into it (a dtype
  change goes through a pinned stage in chunks, copied out while the next crosses).

Calls are synchronous on return and reentrant: the pinned staging buffers and the
copy streams are per thread, the result pool is guarded by a lock (the reference
contract: pure functions, safe to call from concurrent workers)."""
from __future__ import annotations

import mmap
import threading

import numpy as np
import torch

_TLS = threading.local()  # per-thread pinned staging buffers and copy streams

#: bytes below which vectors move in one piece (chunking only pays for large vectors)
CHUNK_MIN_BYTES = 8 << 20
#: D2H chunks of an output vector
OUT_CHUNKS = 8


def pinned(shape, dtype, tag: str = "") -> torch.Tensor:
    """A reusable pinned host buffer (page-locking 400 MB costs tens of ms per call);
    `tag` keeps the input and output staging buffers of one call apart."""
    pins = _TLS.__dict__.setdefault("pinned", {})
    key = (tuple(shape), dtype, tag)
    buf = pins.get(key)
    if buf is None:
        buf = pins[key] = torch.empty(shape, dtype=dtype, pin_memory=True)
    return buf


def copy_stream(dev: torch.device) -> torch.cuda.Stream:
    """This thread's copy stream on `dev`."""
    streams = _TLS.__dict__.setdefault("streams", {})
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    s = streams.get(idx)
    if s is None:
        s = streams[idx] = torch.cuda.Stream(device=dev)
    return s


#: released host mappings kept for reuse, per size (a reused mapping is already faulted
#: in and page-locked); at most POOL_PER_SIZE per size and POOL_MAX_BYTES in all, the
#: least recently released evicted (unregistered and unmapped) first
_POOL: dict[int, list["_Mapping"]] = {}
_POOL_LRU: list["_Mapping"] = []
_POOL_LOCK = threading.Lock()
POOL_PER_SIZE = 3
POOL_MAX_BYTES = 4 << 30


def pool_bytes() -> int:
    with _POOL_LOCK:
        return sum(len(m.mm) for m in _POOL_LRU)


def _pool_put(m: "_Mapping") -> None:
    with _POOL_LOCK:
        free = _POOL.setdefault(len(m.mm), [])
        evict = []
        if len(free) >= POOL_PER_SIZE:
            evict.append(m)
        else:
            free.append(m)
            _POOL_LRU.append(m)
            total = sum(len(q.mm) for q in _POOL_LRU)
            while total > POOL_MAX_BYTES and _POOL_LRU:
                old = _POOL_LRU.pop(0)
                _POOL[len(old.mm)].remove(old)
                total -= len(old.mm)
                evict.append(old)
    for q in evict:
        q.close()


def pool_clear() -> None:
    """Unregister and unmap every pooled mapping."""
    with _POOL_LOCK:
        evict = list(_POOL_LRU)
        _POOL_LRU.clear()
        _POOL.clear()
    for q in evict:
        q.close()


def _pool_take(nbytes: int) -> "_Mapping | None":
    with _POOL_LOCK:
        free = _POOL.get(nbytes)
        if not free:
            return None
        m = free.pop()
        _POOL_LRU.remove(m)
        return m


class _Mapping:
    """An anonymous host mapping (MADV_HUGEPAGE), page-locked with cudaHostRegister when
    CUDA is up, so device->host copies land in it directly at the full PCIe rate."""

    def __init__(self, nbytes: int):
        self.mm = mmap.mmap(-1, nbytes)
        try:
            self.mm.madvise(mmap.MADV_HUGEPAGE)
        except (AttributeError, OSError, ValueError):
            pass
        probe = np.frombuffer(self.mm, dtype=np.uint8)
        self.addr = probe.ctypes.data
        del probe
        self.registered = False
        if torch.cuda.is_available():
            self.registered = torch.cuda.cudart().cudaHostRegister(self.addr, nbytes, 0) == 0

    def close(self) -> None:
        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.addr)
            self.registered = False
        self.mm.close()


class _PooledMapping:
    """Buffer owner of one mapping: when the last array viewing it is gone (numpy
    releases the buffer), the mapping goes back to the pool instead of being unmapped,
    so the next result of that size skips ~100k first-touch page faults and the
    page-locking."""

    def __init__(self, m: _Mapping):
        self._m = m

    def __buffer__(self, flags):
        return memoryview(self._m.mm)

    def __release_buffer__(self, view):
        view.release()
        try:
            _pool_put(self._m)
        except (AttributeError, TypeError):  # interpreter shutdown: module globals are gone
            return


def _fresh(n: int, dtype) -> tuple[np.ndarray, bool]:
    """(array, page_locked): a new writable host array of n elements that aliases no
    live array.  Large ones are pooled mappings (see _PooledMapping)."""
    dt = np.dtype(dtype)
    nbytes = n * dt.itemsize
    if nbytes < CHUNK_MIN_BYTES:
        return np.empty(n, dtype=dt), False
    m = _pool_take(nbytes) or _Mapping(nbytes)
    return np.frombuffer(_PooledMapping(m), dtype=dt, count=n), m.registered


def fresh_host(n: int, dtype) -> np.ndarray:
    return _fresh(n, dtype)[0]


def stage_in(src: torch.Tensor, dst: torch.Tensor, bounds):
    """Copy the CPU vector src into the device vector dst slice by slice (bounds: slice
    edges), yielding (p, event) once slice p's copy is enqueued; the event fires when it
    has landed.  A pinned src of dst's dtype is copied directly; anything else is
    staged through a reused pinned buffer by a host-parallel copy, which for slice p+1
    runs while slice p crosses PCIe.  The copy stream first waits for the current
    stream (dst may still be read by earlier work)."""
    dev = dst.device
    cs = copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    direct = src.is_pinned() and src.dtype == dst.dtype
    if not direct and dst.numel() * dst.element_size() < CHUNK_MIN_BYTES:
        # small: one pageable copy (no staging buffer per shape); every slice is in with it
        with torch.cuda.stream(cs):
            dst.copy_(src.to(dst.dtype))
            ev = torch.cuda.Event()
            ev.record(cs)
        for p in range(len(bounds) - 1):
            yield p, ev
        return
    stage = None if direct else pinned((dst.numel(),), dst.dtype, "in")
    for p in range(len(bounds) - 1):
        lo, hi = int(bounds[p]), int(bounds[p + 1])
        if direct:
            part = src[lo:hi]
        else:
            part = stage[lo:hi]
            part.copy_(src[lo:hi])  # host-parallel (and converting) copy into pinned memory
        with torch.cuda.stream(cs):
            dst[lo:hi].copy_(part, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        yield p, ev


def slices(n: int, itemsize: int, parts: int = 4) -> list[int]:
    """Slice edges for moving an n-element vector (one piece when it is small)."""
    if n * itemsize < CHUNK_MIN_BYTES:
        return [0, n]
    return [n * q // parts for q in range(parts + 1)]


def to_host(yd: torch.Tensor, out_dtype, as_numpy: bool):
    """A fresh host copy of the device vector yd (numpy array of out_dtype, or a CPU
    tensor of yd's dtype), after the current stream's work on yd: chunked D2H into a
    reused pinned buffer, each chunk copied out while the next crosses."""
    dev = yd.device
    n = yd.numel()
    if n * yd.element_size() < CHUNK_MIN_BYTES:
        h = yd.to("cpu")  # a new tensor, after the current stream's work
        return h.numpy().astype(out_dtype, copy=False) if as_numpy else h
    np_dtype = np.dtype(out_dtype) if as_numpy else torch.empty(0, dtype=yd.dtype).numpy().dtype
    out, locked = _fresh(n, np_dtype)
    dst = torch.from_numpy(out)
    cs = copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    if locked and dst.dtype == yd.dtype:
        # page-locked result of the same dtype: one DMA straight into it
        with torch.cuda.stream(cs):
            dst.copy_(yd, non_blocking=True)
        cs.synchronize()
        torch.cuda.current_stream(dev).wait_stream(cs)
        return out if as_numpy else dst
    edges = slices(n, yd.element_size(), OUT_CHUNKS)
    stage = pinned((n,), yd.dtype, "out")
    events = []
    with torch.cuda.stream(cs):
        for lo, hi in zip(edges[:-1], edges[1:]):
            stage[lo:hi].copy_(yd[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)
    for (lo, hi), ev in zip(zip(edges[:-1], edges[1:]), events):
        ev.synchronize()
        dst[lo:hi].copy_(stage[lo:hi])  # host-parallel
    torch.cuda.current_stream(dev).wait_stream(cs)  # later users of yd / the stage see the copies ordered
    return out if as_numpy else dst
