"""TEST INFRASTRUCTURE — numpy restatement of the reference hot path (see oracle/__init__.py).

All arrays are numpy; indices int64, values float64, as in the reference.
"""

from __future__ import annotations

import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "random_permutation",
    "axis_seed",
    "derived_seed",
    "input_vector",
    "inverse",
    "compose",
    "permute_coo",
    "permute_vector",
    "find_duplicate",
    "coo_to_csr",
    "csr_to_coo_rows",
    "permute_csr_rows",
    "bin_edges",
    "bin_index",
    "histogram_2d_counts",
    "row_histogram_counts",
    "col_histogram_counts",
    "entropy_of_counts",
    "spmv_csr",
    "spmv_csr_parallel",
    "spmv_coo",
    "relative_error",
    "power_iteration",
    "conjugate_gradient",
    "make_row_partition",
    "gflops",
    "rowshard_remap_cols",
    "laplacian5",
    "random_rows",
    "random_rows_fast",
    "rmat_edges",
    "rmat_csr",
    "hash3",
]

# --------------------------------------------------------------------------
# permutations  (reference: permute.py)
# --------------------------------------------------------------------------


def random_permutation(n: int, seed: int) -> np.ndarray:
    """permute.py:71-81 — PCG64 Generator.permutation(n)."""
    return np.random.Generator(np.random.PCG64(seed)).permutation(n).astype(np.int64)


def axis_seed(seed: int, axis: int) -> int:
    """permute.py:206-207."""
    return int(np.random.SeedSequence(seed, spawn_key=(axis,)).generate_state(1, np.uint64)[0])


def derived_seed(master_seed: int, repeat: int) -> int:
    """bench.py:161-165."""
    return int(np.random.SeedSequence(master_seed, spawn_key=(1, repeat)).generate_state(1, np.uint64)[0])


def input_vector(master_seed: int, n: int) -> np.ndarray:
    """bench.py:168-171."""
    seq = np.random.SeedSequence(master_seed, spawn_key=(0,))
    return np.random.Generator(np.random.PCG64(seq)).random(n)


def inverse(fwd: np.ndarray) -> np.ndarray:
    """permute.py:42-45: inv[fwd] = arange(n)."""
    fwd = np.asarray(fwd, dtype=np.int64)
    inv = np.empty(fwd.size, dtype=np.int64)
    inv[fwd] = np.arange(fwd.size, dtype=np.int64)
    return inv


def compose(after: np.ndarray, first: np.ndarray) -> np.ndarray:
    """permute.py:64-68."""
    return np.asarray(after, dtype=np.int64)[np.asarray(first, dtype=np.int64)]


def permute_coo(row, col, p_r, p_c):
    """permute.py:98-102: (p_r[row], p_c[col]) in original entry order."""
    return np.asarray(p_r, dtype=np.int64)[row], np.asarray(p_c, dtype=np.int64)[col]


def permute_vector(x, p) -> np.ndarray:
    """permute.py:105-112: out[p[i]] = x[i]."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    out[np.asarray(p, dtype=np.int64)] = x
    return out


# --------------------------------------------------------------------------
# storage  (reference: matio.py)
# --------------------------------------------------------------------------


def find_duplicate(row, col):
    """matio.py:59-64 / 288-291: first duplicate (row, col) in lexsort order, or None."""
    row = np.asarray(row, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    if row.size == 0:
        return None
    order = np.lexsort((col, row))
    r, c = row[order], col[order]
    dup = np.flatnonzero((r[1:] == r[:-1]) & (c[1:] == c[:-1]))
    if dup.size:
        k = dup[0]
        return int(r[k]), int(c[k])
    return None


def coo_to_csr(n_rows: int, row, col, val):
    """matio.py:281-294: lexsort((col, row)), gather, cumsum(bincount(row))."""
    row = np.asarray(row, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    order = np.lexsort((col, row))
    r, c, v = row[order], col[order], val[order]
    if r.size:
        dup = np.flatnonzero((r[1:] == r[:-1]) & (c[1:] == c[:-1]))
        if dup.size:
            k = dup[0]
            raise ValueError(f"duplicate entry at ({r[k]}, {c[k]})")
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n_rows), out=row_ptr[1:])
    return row_ptr, c, v


def csr_to_coo_rows(row_ptr) -> np.ndarray:
    """matio.py:297-300: np.repeat(arange(n_rows), diff(row_ptr))."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    return np.repeat(np.arange(row_ptr.size - 1, dtype=np.int64), np.diff(row_ptr))


def permute_csr_rows(row_ptr, col, val, p_r, p_c, rows):
    """Rows `rows` of coo_to_csr(permute_matrix(A, p_r, p_c)) without building it
    (SURVEY.md App. A item 4): new row r is old row inv(p_r)[r], columns through
    p_c, sorted.  For sampled checks at sizes the full oracle cannot hold."""
    inv_r = inverse(p_r)
    p_c = np.asarray(p_c, dtype=np.int64)
    out = []
    for r in np.asarray(rows, dtype=np.int64):
        o = inv_r[r]
        a, b = int(row_ptr[o]), int(row_ptr[o + 1])
        c = p_c[np.asarray(col[a:b], dtype=np.int64)]
        order = np.argsort(c, kind="stable")
        out.append((c[order], np.asarray(val[a:b], dtype=np.float64)[order]))
    return out


# --------------------------------------------------------------------------
# histograms and entropy  (reference: entropy.py)
# --------------------------------------------------------------------------


def bin_edges(n: int, bins: int) -> np.ndarray:
    """entropy.py:58-62."""
    width = n // bins
    edges = np.arange(bins + 1, dtype=np.int64) * width
    edges[-1] = n
    return edges


def bin_index(idx, n: int, bins: int) -> np.ndarray:
    """entropy.py:65-67: min(idx // (n // bins), bins - 1)."""
    return np.minimum(np.asarray(idx, dtype=np.int64) // (n // bins), bins - 1)


def histogram_2d_counts(row, col, n_rows, n_cols, bins_r, bins_c) -> np.ndarray:
    """entropy.py:91-101 (_counts_2d)."""
    flat = bin_index(row, n_rows, bins_r) * bins_c + bin_index(col, n_cols, bins_c)
    return np.bincount(flat, minlength=bins_r * bins_c).reshape(bins_r, bins_c).astype(np.int64)


def row_histogram_counts(row, n_rows, bins) -> np.ndarray:
    """entropy.py:77-81."""
    return np.bincount(bin_index(row, n_rows, bins), minlength=bins).astype(np.int64)


def col_histogram_counts(col, n_cols, bins) -> np.ndarray:
    """entropy.py:84-88."""
    return np.bincount(bin_index(col, n_cols, bins), minlength=bins).astype(np.int64)


def entropy_of_counts(counts, base: float = 2.0) -> float:
    """entropy.py:104-119 (_entropy_of_counts; empty histogram -> ValueError)."""
    counts = np.asarray(counts, dtype=np.int64).ravel()
    total = counts.sum()
    if total == 0:
        raise ValueError("histogram is empty (total = 0)")
    p = counts[counts > 0] / total
    if base == 2.0:
        return float(-(p * np.log2(p)).sum())
    return float(-(p * np.log(p)).sum() / math.log(base))


# --------------------------------------------------------------------------
# SpMV  (reference: kernels.py)
# --------------------------------------------------------------------------


def _accumulate_rows(row_ptr, col, val, x, lo, hi, out) -> None:
    """kernels.py:59-70: products then np.add.reduceat over nonempty rows."""
    p0, p1 = int(row_ptr[lo]), int(row_ptr[hi])
    seg = np.zeros(hi - lo)
    if p1 > p0:
        prods = val[p0:p1] * x[col[p0:p1]]
        starts = row_ptr[lo:hi] - p0
        ends = row_ptr[lo + 1 : hi + 1] - p0
        nonempty = ends > starts
        seg[nonempty] = np.add.reduceat(prods, starts[nonempty])
    out[lo:hi] = seg


def spmv_csr(row_ptr, col, val, x) -> np.ndarray:
    """kernels.py:73-78."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n_rows = row_ptr.size - 1
    x = np.asarray(x, dtype=np.float64)
    out = np.empty(n_rows)
    _accumulate_rows(row_ptr, np.asarray(col), np.asarray(val, dtype=np.float64), x, 0, n_rows, out)
    return out


_pools: dict[int, ThreadPoolExecutor] = {}
_pool_lock = threading.Lock()


def make_row_partition(n_rows: int, workers: int) -> np.ndarray:
    """kernels.py:38-49: boundaries of an even split (first n % p parts get +1)."""
    if workers < 1:
        raise ValueError("worker count must be >= 1")
    if workers > n_rows:
        raise ValueError(f"worker count {workers} exceeds row count {n_rows}")
    base, extra = divmod(n_rows, workers)
    sizes = np.full(workers, base, dtype=np.int64)
    sizes[:extra] += 1
    b = np.zeros(workers + 1, dtype=np.int64)
    np.cumsum(sizes, out=b[1:])
    return b


def spmv_csr_parallel(row_ptr, col, val, x, workers: int | None = None) -> np.ndarray:
    """kernels.py:89-128: fork-join over make_row_partition on a cached thread pool
    (numpy releases the GIL inside the vector ops); bitwise equal to spmv_csr."""
    workers = workers or os.cpu_count() or 1
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n_rows = row_ptr.size - 1
    x = np.asarray(x, dtype=np.float64)
    col = np.asarray(col)
    val = np.asarray(val, dtype=np.float64)
    b = make_row_partition(n_rows, workers)
    out = np.empty(n_rows)
    with _pool_lock:
        pool = _pools.get(workers)
        if pool is None:
            pool = _pools[workers] = ThreadPoolExecutor(max_workers=workers)
    futs = [pool.submit(_accumulate_rows, row_ptr, col, val, x, int(lo), int(hi), out) for lo, hi in zip(b[:-1], b[1:])]
    for f in futs:
        f.result()
    return out


def spmv_coo(n_rows: int, row, col, val, x) -> np.ndarray:
    """kernels.py:81-86: np.add.at in entry order."""
    out = np.zeros(n_rows)
    np.add.at(out, np.asarray(row, dtype=np.int64), np.asarray(val) * np.asarray(x)[np.asarray(col, dtype=np.int64)])
    return out


def relative_error(got, expected) -> float:
    """kernels.py:131-142."""
    got = np.asarray(got, dtype=np.float64)
    expected = np.asarray(expected, dtype=np.float64)
    if got.shape != expected.shape:
        raise ValueError("shape mismatch")
    diff = float(np.max(np.abs(got - expected))) if got.size else 0.0
    scale = float(np.max(np.abs(expected))) if expected.size else 0.0
    return diff / scale if scale > 0 else diff


def power_iteration(row_ptr, col, val, x0, steps: int):
    """Reference-style loop over spmv_csr (the paper's reuse premise; no solver exists in
    the reference): x <- A x / ||A x||_2; returns (x, ||A x_last||)."""
    x = np.asarray(x0, dtype=np.float64)
    x = x / np.sqrt(np.dot(x, x))
    lam = 0.0
    for _ in range(steps):
        y = spmv_csr(row_ptr, col, val, x)
        lam = float(np.sqrt(np.dot(y, y)))
        x = y / lam
    return x, lam


def conjugate_gradient(row_ptr, col, val, b, steps: int):
    """Textbook CG from x0 = 0 over spmv_csr; returns (x, r.r)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(np.dot(r, r))
    for _ in range(steps):
        ap = spmv_csr(row_ptr, col, val, p)
        alpha = rr / float(np.dot(p, ap))
        x += alpha * p
        r -= alpha * ap
        rr_new = float(np.dot(r, r))
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, rr


def gflops(nnz: int, seconds_per_call: float) -> float:
    """bench.py:138-144."""
    if seconds_per_call <= 0:
        raise ValueError("seconds per call must be positive")
    return 0.0 if nnz == 0 else 2 * nnz / seconds_per_call / 1e9


# --------------------------------------------------------------------------
# restatements of this build's own host-side plans and input generators
# (not reference functions: they pin the CUDA generators / sharding maps)
# --------------------------------------------------------------------------


def rowshard_remap_cols(col, n_cols: int, parts: int, pad: int) -> np.ndarray:
    """Column id -> slot in the padded all-gathered x (rank k's make_row_partition
    slice lands at k * pad)."""
    b = make_row_partition(n_cols, parts)
    col = np.asarray(col, dtype=np.int64)
    part = np.searchsorted(b, col, side="right") - 1
    return part * pad + (col - b[part])


_M1, _M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def hash3(seed, a, b):
    """synth.cu hash3: mix64(seed*G + mix64(a*K + b + C)) (mod 2^64)."""
    with np.errstate(over="ignore"):
        inner = _mix64(np.asarray(a, dtype=np.uint64) * np.uint64(0xD1B54A32D192ED03)
                       + np.asarray(b, dtype=np.uint64) + np.uint64(0x632BE59BD9B4E019))
        return _mix64(np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + inner)


def laplacian5(g: int):
    """5-point Laplacian on a g x g grid (synth.cu k_laplacian), CSR."""
    n = g * g
    r = np.arange(n, dtype=np.int64)
    i, j = r // g, r % g
    cols = np.stack([r - g, r - 1, r, r + 1, r + g], axis=1)
    vals = np.tile(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), (n, 1))
    ok = np.stack([i > 0, j > 0, np.ones(n, bool), j < g - 1, i < g - 1], axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ok.sum(axis=1), out=row_ptr[1:])
    return row_ptr, cols[ok], vals[ok]


def random_rows(rows, n_cols: int, k: int, seed: int):
    """synth.cu k_random_rows for the given row ids: the first k distinct draws of
    hash3(seed, r, t) -> [0, n_cols), sorted; values U[-1,1) per sorted slot."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.empty((rows.size, k), dtype=np.int64)
    for idx, r in enumerate(rows):
        acc: list[int] = []
        t = 0
        while len(acc) < k:
            h = hash3(seed, np.uint64(r), np.arange(t, t + 32, dtype=np.uint64))
            cand = ((h >> np.uint64(32)) * np.uint64(n_cols)) >> np.uint64(32)
            seen = set(acc)
            for c in cand.tolist():
                if len(acc) == k:
                    break
                if c not in seen:
                    acc.append(c)
                    seen.add(c)
            t += 32
        cols[idx] = np.sort(np.asarray(acc, dtype=np.int64))
    h = hash3(seed ^ 0x5DEECE66D, rows[:, None].astype(np.uint64), np.arange(k, dtype=np.uint64)[None, :])
    vals = (h >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    return cols, vals


def rmat_edges(edge_ids, scale: int, a: float, b: float, c: float, seed: int):
    """synth_rmat.cu k_rmat_edges for the given edge ids."""
    e = np.asarray(edge_ids, dtype=np.uint64)
    r = np.zeros(e.size, dtype=np.int64)
    cc = np.zeros(e.size, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for lvl in range(scale):
        u = (hash3(seed, e, np.uint64(lvl)) >> np.uint64(11)).astype(np.float64) * 2.0**-53
        rb = (u >= ab).astype(np.int64)
        cb = (((u >= a) & (u < ab)) | (u >= abc)).astype(np.int64)
        r = (r << 1) | rb
        cc = (cc << 1) | cb
    return r, cc


def rmat_csr(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, cap: int):
    """Full C3 construction at small scale: edges -> dedupe -> keep the `cap` smallest
    columns per row -> values U[-1,1) per (row, slot) (synth.rmat)."""
    n = 1 << scale
    r, cc = rmat_edges(np.arange(edge_factor * n), scale, a, b, c, seed)
    key = np.unique(r * n + cc)
    r, cc = key // n, key % n
    counts = np.bincount(r, minlength=n)
    starts = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    slot = np.arange(key.size) - starts[r]
    keep = slot < cap
    r, cc, slot = r[keep], cc[keep], slot[keep]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=row_ptr[1:])
    h = hash3(seed ^ 0x5DEECE66D, r.astype(np.uint64), slot.astype(np.uint64))
    vals = (h >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    return row_ptr, cc, vals


def random_rows_fast(rows, n_cols: int, k: int, seed: int):
    """Vectorised random_rows for many rows (first draw round of 32 in numpy; the
    rare rows with < k distinct draws fall back to the loop)."""
    rows = np.asarray(rows, dtype=np.int64)
    t = np.arange(32, dtype=np.uint64)[None, :]
    h = hash3(seed, rows[:, None].astype(np.uint64), t)
    cand = ((h >> np.uint64(32)) * np.uint64(n_cols)) >> np.uint64(32)
    order = np.argsort(cand, axis=1, kind="stable")
    sc = np.take_along_axis(cand, order, axis=1)
    first_sorted = np.ones_like(sc, dtype=bool)
    first_sorted[:, 1:] = sc[:, 1:] != sc[:, :-1]
    first = np.empty_like(first_sorted)
    np.put_along_axis(first, order, first_sorted, axis=1)  # first occurrence, in draw order
    rank = np.cumsum(first, axis=1)
    take = first & (rank <= k)
    ok = take.sum(axis=1) == k
    cols = np.empty((rows.size, k), dtype=np.int64)
    cols[ok] = np.sort(cand[ok][take[ok]].reshape(-1, k), axis=1).astype(np.int64)
    if not ok.all():
        slow, _ = random_rows(rows[~ok], n_cols, k, seed)
        cols[~ok] = slow
    hv = hash3(seed ^ 0x5DEECE66D, rows[:, None].astype(np.uint64), np.arange(k, dtype=np.uint64)[None, :])
    vals = (hv >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    return cols, vals
