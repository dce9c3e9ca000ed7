"""Row/column permutations: generation on the host, application on the GPU.

Drop-in for `spmv_entropy.permute` (reference
/root/reference/pkg/src/spmv_entropy/permute.py).  Permutation GENERATION
(random_permutation, the riffle strategies, build_strategy) stays on the host
with numpy's PCG64, exactly as in the reference, so permutation vectors are
bit-identical by construction (SURVEY.md §7 design principles).  Everything
that APPLIES a permutation — the bijection check / inverse, compose,
permute_vector, permute_rows/cols/matrix and the fused permuted-CSR build —
is an sm_100a kernel (perm.cu, csr_build.cu).
"""

from __future__ import annotations

import threading
from enum import Enum

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import DeviceFlags, ptr, stream
from .matio import CooMatrix, CsrMatrix


class Permutation:
    """A bijection on [0, n): forward[i] is the new position of index i (permute.py:23-50).

    The bijection check runs on the GPU (sme_perm_inverse) and leaves the
    inverse behind, cached for inverse() and for the row-gather of permute_csr.
    """

    def __init__(self, forward, *, _trusted: bool = False, _host: np.ndarray | None = None):
        if isinstance(forward, torch.Tensor):
            if forward.dim() != 1 or forward.numel() == 0:
                raise ValueError("forward must be a non-empty 1-D array")
            self.d_forward = _cuda.as_index_tensor(forward, "forward")
            self._fwd_host = _host
        else:
            fwd = np.asarray(forward, dtype=np.int64)
            if fwd.ndim != 1 or fwd.size == 0:
                raise ValueError("forward must be a non-empty 1-D array")
            if fwd.min() < 0 or fwd.max() >= fwd.size:
                raise ValueError("forward is not a bijection on [0, n)")
            self.d_forward = _cuda.as_index_tensor(fwd, "forward")
            self._fwd_host = fwd
        self._d_inverse: torch.Tensor | None = None
        if not _trusted:
            self._compute_inverse(check=True)

    def _compute_inverse(self, check: bool) -> torch.Tensor:
        inv = torch.empty_like(self.d_forward)
        fl = DeviceFlags()
        _lib.call("sme_perm_inverse", self.n, ptr(self.d_forward), ptr(inv), fl.flag_ptr, stream())
        if check:
            bits, _ = fl.read()
            if bits & (_lib.FLAG_RANGE | _lib.FLAG_NOT_BIJECTION):
                raise ValueError("forward is not a bijection on [0, n)")
        self._d_inverse = inv
        return inv

    @property
    def d_inverse(self) -> torch.Tensor:
        return self._d_inverse if self._d_inverse is not None else self._compute_inverse(check=False)

    @property
    def n(self) -> int:
        return int(self.d_forward.numel())

    @property
    def forward(self) -> np.ndarray:
        if self._fwd_host is None:
            self._fwd_host = _cuda.to_host(self.d_forward, np.int64)
            self._fwd_host.flags.writeable = False
        return self._fwd_host

    def inverse(self) -> "Permutation":
        q = Permutation(self.d_inverse, _trusted=True)
        q._d_inverse = self.d_forward
        return q

    def __eq__(self, other) -> bool:
        if not isinstance(other, Permutation):
            return NotImplemented
        if self is other:
            return True
        if self.n != other.n:
            return False
        if self.n == 0:
            return True
        # different content hashes (one libsme pass each) settle the common case; equal
        # hashes are confirmed element by element
        if self._content_hash() != other._content_hash():
            return False
        return torch.equal(self.d_forward, other.d_forward)

    def _content_hash(self) -> int:
        if getattr(self, "_hash", None) is None:
            out = torch.empty(1, dtype=torch.int64, device=self.d_forward.device)
            _lib.call("sme_hash64", ptr(self.d_forward), self.d_forward.numel() * 4, 0x5EED, ptr(out), stream())
            self._hash = int(out.item())
        return self._hash

    __hash__ = object.__hash__

    def __repr__(self) -> str:
        return f"Permutation(n={self.n})"


def _as_perm(p) -> Permutation:
    if isinstance(p, Permutation):
        return p
    fwd = getattr(p, "forward", None)  # a reference spmv_entropy.Permutation
    if fwd is not None:
        return Permutation(fwd)
    return Permutation(p)


def identity_permutation(n: int) -> Permutation:
    if n < 1:
        raise ValueError("permutation size must be >= 1")
    dev = _cuda.require_cuda()
    return Permutation(torch.arange(n, dtype=torch.int32, device=dev), _trusted=True)


def inverse(p: Permutation) -> Permutation:
    """The permutation q with p.forward[q.forward[i]] = i for all i (permute.py:53-55)."""
    return _as_perm(p).inverse()


def compose(after: Permutation, first: Permutation) -> Permutation:
    """Permutation equivalent to applying `first`, then `after` (permute.py:64-68)."""
    after, first = _as_perm(after), _as_perm(first)
    if after.n != first.n:
        raise ValueError("size mismatch")
    out = torch.empty_like(first.d_forward)
    _lib.call("sme_gather", _lib.SME_I32, first.n, ptr(first.d_forward), ptr(after.d_forward), ptr(out), stream())
    return Permutation(out, _trusted=True)


_U64 = (1 << 64) - 1


def _pcg64_words(bitgen: np.random.PCG64) -> np.ndarray:
    """numpy PCG64.state as the six uint64 words sme_host_pcg64_permutation takes."""
    s = bitgen.state
    st, inc = s["state"]["state"], s["state"]["inc"]
    return np.array([st >> 64, st & _U64, inc >> 64, inc & _U64, s["has_uint32"], s["uinteger"]], dtype=np.uint64)


def _set_pcg64_words(bitgen: np.random.PCG64, w: np.ndarray) -> None:
    bitgen.state = {
        "bit_generator": "PCG64",
        "state": {"state": (int(w[0]) << 64) | int(w[1]), "inc": (int(w[2]) << 64) | int(w[3])},
        "has_uint32": int(w[4]),
        "uinteger": int(w[5]),
    }


def pcg64_permutation(bitgen: np.random.PCG64, n: int) -> np.ndarray:
    """Generator(bitgen).permutation(n) as int32, bit-exact, advancing `bitgen` like numpy.

    The native generator (sme_host_pcg64_permutation, pcg64_host.cpp) restates
    numpy's Fisher-Yates shuffle with the swap partners drawn ahead and
    prefetched; it is a host call (ctypes releases the GIL, so the row and
    column permutations of a strategy are generated concurrently).
    """
    if n < 1 or n > 2**31 - 1:
        raise ValueError("permutation size must be in [1, 2^31)")
    words = _pcg64_words(bitgen)
    out = np.empty(n, dtype=np.int32)
    _lib.call("sme_host_pcg64_permutation", words.ctypes.data, n, out.ctypes.data)
    _set_pcg64_words(bitgen, words)
    return out


def pcg64_swap_partners(bitgen: np.random.PCG64, n: int, out: np.ndarray | None = None, threads: int = 0) -> np.ndarray:
    """The swap partners of Generator(bitgen).permutation(n): j[i] for i = n-1..1 in numpy's
    draw order (j[0] = 0), advancing `bitgen` exactly like the full shuffle (host call)."""
    if n < 1 or n > 2**31 - 1:
        raise ValueError("permutation size must be in [1, 2^31)")
    words = _pcg64_words(bitgen)
    j = np.empty(n, dtype=np.uint32) if out is None else out
    _lib.call("sme_host_pcg64_swap_partners", words.ctypes.data, n, j.ctypes.data, int(threads))
    _set_pcg64_words(bitgen, words)
    return j


#: sizes from which the partners are drawn on the GPU (sme_pcg64_swap_partners_gpu)
GPU_PARTNERS_MIN = 1 << 20


_SIDE_STREAMS: dict = {}
_SIDE_LOCK = threading.Lock()


def _side_stream(dev: torch.device, slot) -> torch.cuda.Stream:
    """A long-lived side stream per (device, slot).  Work is stream-ordered, so sharing one
    between callers only serialises them; reusing it lets torch's caching allocator, whose
    blocks belong to the stream that allocated them, hand back the same scratch every call
    (a fresh stream per call meant fresh cudaMallocs: C4 permutation pairs 22-134 ms)."""
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), slot)
    with _SIDE_LOCK:
        st = _SIDE_STREAMS.get(key)
        if st is None:
            st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=dev)
    return st


def pcg64_swap_partners_device(bitgen: np.random.PCG64, n: int, threads: int = 0,
                               out: torch.Tensor | None = None, gpu_min: int | None = None,
                               slot: int = 0) -> torch.Tensor:
    """pcg64_swap_partners straight into a CUDA int32 tensor.  From GPU_PARTNERS_MIN on
    they are drawn on the GPU (sme_pcg64_swap_partners_gpu: parallel PCG64 stream, draws
    decided in parallel inside statistical step windows, the few ambiguous ones in order
    on the host); below it, or if a window check fails, the host replay streams finished
    4 MB slots of a pinned ring to the device while it draws the rest
    (sme_pcg64_swap_partners_to_device).  `bitgen` advances exactly as the full shuffle's."""
    if n < 1 or n > 2**31 - 1:
        raise ValueError("permutation size must be in [1, 2^31)")
    dev = _cuda.require_cuda()
    d_j = torch.empty(n, dtype=torch.int32, device=dev) if out is None else out
    cs = _side_stream(dev, ("partners", slot))
    cs.wait_stream(torch.cuda.current_stream(dev))  # d_j's allocation is ordered before the copies
    words = _pcg64_words(bitgen)
    if n >= (GPU_PARTNERS_MIN if gpu_min is None else gpu_min) and n >= 2:
        # scratch from torch's caching allocator (warm after the matrix build): no
        # driver-level allocation inside the call
        ws = _cuda.workspace(_lib.query_size("sme_pcg64_swap_partners_gpu_workspace_size", n))
        rc = _lib.load().sme_pcg64_swap_partners_gpu(words.ctypes.data, n, ptr(d_j), ptr(ws), ws.numel(),
                                                     cs.cuda_stream)
        ws.record_stream(cs)
        if rc == _lib.SME_OK:
            _set_pcg64_words(bitgen, words)
            torch.cuda.current_stream(dev).wait_stream(cs)
            d_j.record_stream(cs)
            return d_j
        if rc != 1:  # 1: a window check failed -> the host replay below
            raise RuntimeError(f"sme_pcg64_swap_partners_gpu: {_lib.last_error()}")
        words = _pcg64_words(bitgen)
    _lib.call("sme_pcg64_swap_partners_to_device", words.ctypes.data, n, ptr(d_j), int(threads), cs.cuda_stream)
    _set_pcg64_words(bitgen, words)
    torch.cuda.current_stream(dev).wait_stream(cs)
    d_j.record_stream(cs)
    return d_j


def pcg64_permutation_device(bitgen: np.random.PCG64, n: int, threads: int = 0) -> torch.Tensor:
    """Generator(bitgen).permutation(n) as a CUDA int32 tensor, bit-exact: partners drawn on
    the host and uploaded while they are drawn (pcg64_swap_partners_device), swaps applied
    in parallel on the GPU (sme_fy_apply: bucket sort by partner + chain walk instead of n
    dependent swaps)."""
    dev = _cuda.require_cuda()
    d_j = pcg64_swap_partners_device(bitgen, n, threads=threads)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    ws = _cuda.workspace(_lib.query_size("sme_fy_apply_workspace_size", n))
    _lib.call("sme_fy_apply", n, ptr(d_j), ptr(out), ptr(ws), ws.numel(), stream())
    torch.cuda.current_stream().synchronize()  # ws is released on return
    return out


def _check_perm_args(n: int, seed: int) -> None:
    if n < 1:
        raise ValueError("permutation size must be >= 1")
    if seed < 0:
        raise ValueError("seed must be non-negative")


def random_permutation_forward(n: int, seed: int) -> np.ndarray:
    """Host generation, identical to the reference (permute.py:71-81): PCG64 shuffle, int32."""
    _check_perm_args(n, seed)
    return pcg64_permutation(np.random.PCG64(seed), n)


def random_permutation(n: int, seed: int) -> Permutation:
    """Uniform permutation from a seeded PCG64 generator (Fisher-Yates), bit-identical to the reference:
    host draws, GPU swaps (pcg64_permutation_device)."""
    _check_perm_args(n, seed)
    return Permutation(pcg64_permutation_device(np.random.PCG64(seed), n), _trusted=True)


def random_permutations(specs) -> list[Permutation]:
    """random_permutation for several (n, seed) pairs, generated concurrently on host threads."""
    specs = list(specs)
    for n, seed in specs:
        _check_perm_args(n, seed)
    if len(specs) == 1:
        return [random_permutation(*specs[0])]
    # the host draws of all specs run concurrently (ctypes releases the GIL), each with
    # its upload overlapped and its GPU shuffle started as soon as its partners are in
    from concurrent.futures import ThreadPoolExecutor

    dev = _cuda.require_cuda()
    threads = max(1, 8 // len(specs))
    main = torch.cuda.current_stream(dev)
    # buffers come from the caller's stream (its allocator pool); each spec's shuffle then
    # runs on its own stream as soon as its partners are in, overlapping the others' draws
    bufs = [(torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
             _cuda.workspace(_lib.query_size("sme_fy_apply_workspace_size", n))) for n, _ in specs]

    def one(k):
        (n, seed), (d_j, perm, ws) = specs[k], bufs[k]
        s = _side_stream(dev, ("axis", k))
        s.wait_stream(main)
        with torch.cuda.stream(s):
            pcg64_swap_partners_device(np.random.PCG64(seed), n, threads=threads, out=d_j, slot=k)
            _lib.call("sme_fy_apply", n, ptr(d_j), ptr(perm), ptr(ws), ws.numel(), stream())
        s.synchronize()

    with ThreadPoolExecutor(max_workers=len(specs)) as ex:
        list(ex.map(one, range(len(specs))))
    return [Permutation(perm, _trusted=True) for _, perm, _ in bufs]


def permute_rows(m: CooMatrix, p: Permutation) -> CooMatrix:
    """Move entry (i, j, v) to (p.forward[i], j, v) (permute.py:84-88)."""
    p = _as_perm(p)
    if p.n != m.n_rows:
        raise ValueError("permutation size must equal n_rows")
    return _permute_coo(m, p, None)


def permute_cols(m: CooMatrix, p: Permutation) -> CooMatrix:
    """Move entry (i, j, v) to (i, p.forward[j], v) (permute.py:91-95)."""
    p = _as_perm(p)
    if p.n != m.n_cols:
        raise ValueError("permutation size must equal n_cols")
    return _permute_coo(m, None, p)


@_cuda.nvtx("permute_matrix")
def permute_matrix(m: CooMatrix, p_r: Permutation, p_c: Permutation) -> CooMatrix:
    """Apply a (row, column) permutation pair in one pass (permute.py:98-102).

    Returns the COO in the ORIGINAL entry order with remapped indices (one
    remap kernel).  Its CSR (coo_to_csr) is then produced by the fused
    row-gather + segmented-sort kernel from the source's CSR, never by a
    global sort.
    """
    p_r, p_c = _as_perm(p_r), _as_perm(p_c)
    if p_r.n != m.n_rows or p_c.n != m.n_cols:
        raise ValueError("permutation sizes must match matrix dimensions")
    return _permute_coo(m, p_r, p_c)


def _permute_coo(m: CooMatrix, p_r: Permutation | None, p_c: Permutation | None) -> CooMatrix:
    if not isinstance(m, CooMatrix):
        raise TypeError("expected a CooMatrix (use permute_csr for CsrMatrix)")
    dev = m.d_row_idx.device
    row = torch.empty_like(m.d_row_idx) if p_r is not None else m.d_row_idx.clone()
    col = torch.empty_like(m.d_col_idx) if p_c is not None else m.d_col_idx.clone()
    _lib.call("sme_coo_remap", m.nnz, ptr(m.d_row_idx), ptr(m.d_col_idx),
              ptr(p_r.d_forward if p_r is not None else None), ptr(p_c.d_forward if p_c is not None else None),
              ptr(row) if p_r is not None else None, ptr(col) if p_c is not None else None, stream())
    src = m

    def thunk() -> CsrMatrix:
        from .matio import coo_to_csr

        return permute_csr(coo_to_csr(src), p_r, p_c)

    del dev
    return CooMatrix._from_device(m.n_rows, m.n_cols, row, col, m.d_values.clone(), csr_thunk=thunk)


#: K4 relabels the columns in a pre-pass (sme_map_cols_sliced) when p_c is larger than
#: PREMAP_SLICE_BYTES and the matrix has at least PREMAP_MIN_NNZ entries: one pass per
#: PREMAP_SLICE_BYTES slice of p_c, each slice L2-resident while its gathers run.  A random
#: 4-byte gather from a table larger than L2 costs a 64-byte DRAM access
#: (tools/l2fetch_bench.cu: 86-90 G/s from 200 MB, 287 G/s from 50 MB, and 148-160 G/s from
#: 100 MB: the random-gather working set that stays in L2 is about 50-60 MB).  None: auto;
#: True/False force it on/off (tests).  Results are bit-identical either way.
PREMAP: bool | None = None
PREMAP_SLICE_BYTES = 48 << 20
PREMAP_MIN_NNZ = 1 << 24
#: reserve persisting L2 for the slice (access-policy window) during the pre-map passes
PREMAP_PERSIST = False
#: leave the last slice to the row sort (one pass over col fewer)
PREMAP_FUSE_LAST = False
#: gather the source starts once with the permuted lengths (sme_permute_csr_row_ptr_starts)
#: and let the row sort read them in order; False: the sort gathers row_ptr[inv_r[r]]
K4_STARTS = True
def _premap_slices(m: CsrMatrix) -> int:
    """Number of column slices for the pre-map (0: gather p_c inside the row sort)."""
    if PREMAP is False or m.d_col_idx.data_ptr() % 16:
        return 0
    table = m.n_cols * 4
    if PREMAP is None and (m.nnz < PREMAP_MIN_NNZ or table <= PREMAP_SLICE_BYTES):
        return 0
    n = max(1, -(-table // PREMAP_SLICE_BYTES))
    if PREMAP_PERSIST:
        from .panels import device_info

        info = device_info()
        _lib.call("sme_l2_set_persisting", min(info["max_persisting_l2"], -(-table // n)))
    return int(n)


@_cuda.nvtx("permute_csr")
def permute_csr(m: CsrMatrix, p_r: Permutation | None, p_c: Permutation | None) -> CsrMatrix:
    """P_r A P_c directly on CSR (K4): row gather through inverse(p_r), column remap
    through p_c, segmented sort inside each row.  Bit-identical to
    coo_to_csr(permute_matrix(csr_to_coo(m), p_r, p_c))."""
    if p_r is not None:
        p_r = _as_perm(p_r)
        if p_r.n != m.n_rows:
            raise ValueError("permutation sizes must match matrix dimensions")
    if p_c is not None:
        p_c = _as_perm(p_c)
        if p_c.n != m.n_cols:
            raise ValueError("permutation sizes must match matrix dimensions")
    dev = m.d_row_ptr.device
    inv_r = p_r.d_inverse if p_r is not None else None
    row_ptr = torch.empty(m.n_rows + 1, dtype=m.d_row_ptr.dtype, device=dev)  # int64 for nnz >= 2^31 - 1
    # the source start of every new row, gathered once with the lengths: the row sort then
    # reads its sources in order (starts as the source row_ptr, identity rows)
    ws1 = _cuda.workspace(_lib.query_size("sme_row_ptr_workspace_size", m.n_rows))
    if K4_STARTS:
        starts = torch.empty(max(1, m.n_rows), dtype=m.d_row_ptr.dtype, device=dev)
        _lib.call_rp("sme_permute_csr_row_ptr_starts", row_ptr, m.n_rows, ptr(m.d_row_ptr), ptr(inv_r),
                     ptr(row_ptr), ptr(starts), ptr(ws1), ws1.numel(), stream())
        src_ptr, src_inv = starts, None
    else:
        _lib.call_rp("sme_permute_csr_row_ptr", row_ptr, m.n_rows, ptr(m.d_row_ptr), ptr(inv_r), ptr(row_ptr),
                     ptr(ws1), ws1.numel(), stream())
        src_ptr, src_inv = m.d_row_ptr, inv_r
    long_nnz = m.long_row_nnz()
    ws2 = _cuda.workspace(_lib.query_size("sme_permute_csr_workspace_size", m.n_rows, m.nnz, long_nnz))
    col = torch.empty_like(m.d_col_idx)
    val = torch.empty_like(m.d_values)
    fl = DeviceFlags()
    src_col, cmap = m.d_col_idx, (p_c.d_forward if p_c is not None else None)
    n_slices = _premap_slices(m) if cmap is not None else 0
    if n_slices:
        # p_c larger than L2: relabel the columns of all but the last slice first, each
        # pass with its slice of p_c L2-resident; the row sort then gathers only the last
        # slice (L2-resident after the last pass) and clears the relabelled entries' flags
        src_col = torch.empty_like(m.d_col_idx)
        n_passes = n_slices - 1 if (PREMAP_FUSE_LAST and n_slices > 1) else n_slices
        _lib.call("sme_map_cols_sliced_partial", m.nnz, m.n_cols, ptr(m.d_col_idx), ptr(cmap), ptr(src_col),
                  n_slices, n_passes, stream())
        if PREMAP_PERSIST:
            _lib.call("sme_l2_reset_persisting")
        if n_passes == n_slices:
            cmap = None
    _lib.call_rp("sme_permute_csr", row_ptr, _cuda.sme_dtype(m.d_values), m.n_rows, m.n_cols, m.nnz,
                 ptr(src_ptr), ptr(src_col), ptr(m.d_values), ptr(src_inv), ptr(cmap), ptr(row_ptr), ptr(col),
                 ptr(val), ptr(ws2), ws2.numel(), long_nnz, fl.flag_ptr, fl.dup_ptr, stream())
    del src_col, src_ptr
    out = CsrMatrix._from_device(m.n_rows, m.n_cols, row_ptr, col, val)
    out._cache["long_nnz"] = long_nnz
    return out


def permute_vector(x, p: Permutation):
    """Return `out` with out[p.forward[i]] = x[i] (permute.py:105-112).

    Host array in -> host numpy float64 out (one H2D, one scatter kernel, one
    D2H); CUDA tensor in -> CUDA tensor out (device-resident, f64 or f32)."""
    p = _as_perm(p)
    if isinstance(x, torch.Tensor) and x.is_cuda:
        if x.dim() != 1 or x.numel() != p.n:
            raise ValueError("vector length must equal permutation size")
        xs = x.contiguous()
        if xs.dtype not in (torch.float64, torch.float32):
            xs = xs.to(torch.float64)
        out = torch.empty_like(xs)
        _lib.call("sme_permute_vector", _cuda.sme_dtype(xs), p.n, ptr(p.d_forward), ptr(xs), ptr(out), stream())
        return out
    xa = np.asarray(x, dtype=np.float64)
    if xa.shape != (p.n,):
        raise ValueError("vector length must equal permutation size")
    xd = torch.from_numpy(np.ascontiguousarray(xa)).to(p.d_forward.device)
    out = torch.empty_like(xd)
    _lib.call("sme_permute_vector", _lib.SME_F64, p.n, ptr(p.d_forward), ptr(xd), ptr(out), stream())
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# strategies (host-side generation, as in the reference; permute.py:115-250)
# ---------------------------------------------------------------------------
def gradient_pivot(h) -> int:
    """Index of the steepest histogram increase (permute.py:115-126)."""
    counts = np.asarray(h.counts)
    if counts.ndim != 1:
        raise ValueError("gradient pivot requires a 1-D histogram")
    if counts.size < 2:
        raise ValueError("gradient pivot requires at least 2 bins")
    grad = counts[1:] - counts[:-1]
    return int(np.asarray(h.edges[0])[int(np.argmax(grad)) + 1])


def _interleave_forward(n: int, pivot: int) -> np.ndarray:
    a, b = pivot, n - pivot
    short = min(a, b)
    fwd = np.empty(n, dtype=np.int64)
    ka = np.arange(a, dtype=np.int64)
    kb = np.arange(b, dtype=np.int64)
    fwd[:a] = np.where(ka < short, 2 * ka, ka + b)
    fwd[a:] = np.where(kb < short, 2 * kb + 1, kb + a)
    return fwd


def riffle_shuffle_permutation(n: int, pivot: int, seed: int) -> Permutation:
    """Riffle [0, pivot) and [pivot, n) (permute.py:142-157): local PCG64 shuffles, then interleave."""
    if not 0 < pivot < n:
        raise ValueError(f"pivot {pivot} out of range (0, {n})")
    if seed < 0:
        raise ValueError("seed must be non-negative")
    bitgen = np.random.PCG64(seed)  # one generator, two consecutive shuffles (permute.py:154-156)
    local = torch.cat([pcg64_permutation_device(bitgen, pivot), pivot + pcg64_permutation_device(bitgen, n - pivot)])
    return compose(Permutation(_interleave_forward(n, pivot)), Permutation(local, _trusted=True))


class StrategyKind(Enum):
    """The identity baseline plus the four randomization formats (permute.py:160-201)."""

    REGULAR = "regular"
    ROW_PERMUTE = "row_permute"
    ROW_COLUMN_PERMUTE = "row_column_permute"
    ROW_GRADIENT = "row_gradient"
    COLUMN_GRADIENT = "column_gradient"

    @property
    def code(self) -> str:
        return _CODES[self]

    @property
    def label(self) -> str:
        return _LABELS[self]


_CODES = {
    StrategyKind.REGULAR: "reg",
    StrategyKind.ROW_PERMUTE: "r",
    StrategyKind.ROW_COLUMN_PERMUTE: "rc",
    StrategyKind.ROW_GRADIENT: "gr",
    StrategyKind.COLUMN_GRADIENT: "gc",
}
_LABELS = {
    StrategyKind.REGULAR: "Regular",
    StrategyKind.ROW_PERMUTE: "Row-Permute",
    StrategyKind.ROW_GRADIENT: "Row-Gradient",
    StrategyKind.COLUMN_GRADIENT: "Column-Gradient",
    StrategyKind.ROW_COLUMN_PERMUTE: "Row-Column-Permute",
}
TABLE_ORDER = (
    StrategyKind.REGULAR,
    StrategyKind.ROW_PERMUTE,
    StrategyKind.ROW_GRADIENT,
    StrategyKind.COLUMN_GRADIENT,
    StrategyKind.ROW_COLUMN_PERMUTE,
)
_ROW_STREAM, _COL_STREAM = 0, 1


def axis_seed(seed: int, axis: int) -> int:
    """permute.py:206-207: SeedSequence(seed, spawn_key=(axis,)) -> one uint64."""
    return int(np.random.SeedSequence(seed, spawn_key=(axis,)).generate_state(1, np.uint64)[0])


def build_strategy(m, kind: StrategyKind, seed: int, bins: int = 512, column_gradient_both_axes: bool = True):
    """(row, column) permutation pair for a strategy (permute.py:210-250).

    `m` is a CooMatrix or CsrMatrix of this package; the gradient strategies
    take their 1-D histograms from the GPU histogram kernels.
    """
    from .entropy import col_histogram, row_histogram

    if seed < 0:
        raise ValueError("seed must be non-negative")
    row_seed = axis_seed(seed, _ROW_STREAM)
    col_seed = axis_seed(seed, _COL_STREAM)
    if kind is StrategyKind.REGULAR:
        return identity_permutation(m.n_rows), identity_permutation(m.n_cols)
    if kind is StrategyKind.ROW_PERMUTE:
        return random_permutation(m.n_rows, row_seed), identity_permutation(m.n_cols)
    if kind is StrategyKind.ROW_COLUMN_PERMUTE:
        p_r, p_c = random_permutations([(m.n_rows, row_seed), (m.n_cols, col_seed)])
        return p_r, p_c

    def riffled(n: int, histogram, axis_seed_: int) -> Permutation:
        return riffle_shuffle_permutation(n, gradient_pivot(histogram), axis_seed_)

    if kind is StrategyKind.ROW_GRADIENT:
        return riffled(m.n_rows, row_histogram(m, min(bins, m.n_rows)), row_seed), identity_permutation(m.n_cols)
    if kind is StrategyKind.COLUMN_GRADIENT:
        p_c = riffled(m.n_cols, col_histogram(m, min(bins, m.n_cols)), col_seed)
        if not column_gradient_both_axes:
            return identity_permutation(m.n_rows), p_c
        return riffled(m.n_rows, row_histogram(m, min(bins, m.n_rows)), row_seed), p_c
    raise ValueError(f"unknown strategy {kind!r}")
